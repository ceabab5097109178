O=gpurun_out/r02e; mkdir -p $O
for g in 1 2 0; do for o in 0 1; do
  timeout 300 python tools/lora_gap.py --profile 0 --clocks 1 --gc $g --overlap-free $o --steps 40 >> $O/lora_gap.jsonl 2>> $O/lora_gap.err
done; done
timeout 300 python bench.py --config lora-70b-r32 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_lora.json 2> $O/bench_lora.err
timeout 300 python bench.py --config lora-70b-r32 --mode zerocopy --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_lora_zc.json 2> $O/bench_lora_zc.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
