# r02aw: fine tail on every launch (SLLM_FINE_TAIL=2) vs unbalanced only (default), 2 CTAs/SM
O=gpurun_out/r02aw; mkdir -p $O
M=gpu__time_duration.sum
for rep in 1 2; do for v in 1 2; do
  export SLLM_FINE_TAIL=$v
  timeout 600 ncu --metrics $M --clock-control none --csv -k regex:materialise -c 4 python tools/ncu_kernels.py 2>/dev/null | grep materialise | sed "s/^/ft$v,$rep,/" >> $O/ncu.csv
  SLLM_KTIME=1 timeout 300 python tools/k4_sizes.py --max-gib 4 --reps 5 2>&1 | grep "ktime bytes=4294967296" | sed "s/^/ft$v $rep /" >> $O/k4_live.txt
  timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline | sed "s/^{/{\"variant\": \"ft$v\", \"rep\": $rep, /" >> $O/bench_ce.jsonl 2>> $O/bench.err
  timeout 300 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"variant\": \"ft$v\", \"rep\": $rep, /" >> $O/bench_scatter.jsonl 2>> $O/bench.err
done; done
unset SLLM_FINE_TAIL
