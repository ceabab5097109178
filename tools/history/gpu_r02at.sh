# r02at: 3 ring CTAs per SM (64 KiB) vs 2 (96 KiB)
O=gpurun_out/r02at; mkdir -p $O
M=gpu__time_duration.sum
for rep in 1 2; do for v in r96x2 r64x3; do
  export SLLM_LIB_PATH=build/ab/$v/libsllm.so
  timeout 600 ncu --metrics $M --clock-control none --csv -k regex:materialise -c 4 python tools/ncu_kernels.py 2>/dev/null | grep materialise | sed "s/^/$v,$rep,/" >> $O/ncu.csv
  SLLM_KTIME=1 timeout 300 python tools/k4_sizes.py --max-gib 4 --reps 5 2>&1 | grep "ktime bytes=4294967296" | sed "s/^/$v $rep /" >> $O/k4_live.txt
  timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $O/bench_ce.jsonl 2>> $O/bench.err
  timeout 300 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $O/bench_scatter.jsonl 2>> $O/bench.err
  timeout 300 python bench.py --mode zerocopy --steps 5 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $O/bench_zc.jsonl 2>> $O/bench.err
done; done
unset SLLM_LIB_PATH
