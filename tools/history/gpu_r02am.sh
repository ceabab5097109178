O=gpurun_out/r02am; mkdir -p $O
for rep in 1 2; do for w in 1024 2048; do
  SLLM_SCATTER_WINDOW_MIB=$w timeout 300 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"scatter_window_mib\": $w, \"rep\": $rep, /" >> $O/scatter_window.jsonl 2>> $O/err.txt
done; done
