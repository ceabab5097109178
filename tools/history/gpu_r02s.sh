# r02s: CE copy-window size A/B (one cudaMemcpyAsync per window), S = 1 / 2
O=gpurun_out/r02s; mkdir -p $O
for rep in 1 2; do
for w in 64 256 1024; do for s in 2 1; do
  SLLM_WINDOW_MIB=$w timeout 300 python bench.py --steps 8 --warmup 3 --streams $s --no-cpu-baseline --no-standalone \
     | sed "s/^{/{\"window_mib\": $w, \"rep\": $rep, /" >> $O/window_sweep.jsonl 2>> $O/window_sweep.err
done; done; done
