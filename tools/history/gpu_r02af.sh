# r02af: cost of the per-unit consumer barrier (timing-only variant without it)
O=gpurun_out/r02af; mkdir -p $O
M=gpu__time_duration.sum
for rep in 1 2; do for v in base nosync; do
  SLLM_LIB_PATH=build/ab/$v/libsllm.so timeout 600 ncu --metrics $M --clock-control none --csv -k regex:materialise -c 4 python tools/ncu_kernels.py 2>/dev/null | grep materialise | sed "s/^/$v,$rep,/" >> $O/ncu.csv
  SLLM_LIB_PATH=build/ab/$v/libsllm.so SLLM_KTIME=1 timeout 300 python tools/k4_sizes.py --max-gib 4 --reps 5 2>&1 | grep "ktime bytes=4294967296" | sed "s/^/$v $rep /" >> $O/k4_live.txt
done; done
