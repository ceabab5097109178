# r02v: standalone K4/K3 under ncu (duration + DRAM) for the four work-distribution variants, twice
O=gpurun_out/r02v; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed
for rep in 1 2; do
for v in dyn_fine dyn static_fine static; do
  unset SLLM_STATIC_UNITS SLLM_FINE_TAIL
  case $v in dyn) export SLLM_FINE_TAIL=0;; static_fine) export SLLM_STATIC_UNITS=1;; static) export SLLM_STATIC_UNITS=1 SLLM_FINE_TAIL=0;; esac
  timeout 600 ncu --metrics $M --clock-control none --csv -k regex:materialise -c 4 python tools/ncu_kernels.py 2>/dev/null \
     | grep materialise | sed "s/^/$v,$rep,/" >> $O/ncu_variants.csv
  SLLM_KTIME=1 timeout 300 python tools/k4_sizes.py --max-gib 4 --reps 7 2>&1 | grep -E "ktime bytes=4294967296|\"bytes\": 4294967296" | sed "s/^/$v $rep /" >> $O/k4_live.txt
done; done
