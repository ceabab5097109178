O=gpurun_out/r02c; mkdir -p $O
for p in 1 0; do for c in 1 0; do
  timeout 300 python tools/lora_gap.py --profile $p --clocks $c >> $O/lora_gap.jsonl 2>> $O/lora_gap.err
done; done
timeout 300 python tools/lora_gap.py --mode zerocopy --profile 0 --clocks 0 >> $O/lora_gap.jsonl 2>> $O/lora_gap.err
timeout 300 python bench.py --config lora-70b-r32 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_lora.json 2> $O/bench_lora.err
ncu --query-metrics 2>/dev/null | grep -i -E "pcie|nvlrx|nvltx|sysmem" > $O/ncu_pcie_metrics.txt
