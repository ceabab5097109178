# r01q: N=1 bench lines of C3/C4 partition 0; SCATTER_CE staging-window sweep (K3 in pipeline)
mkdir -p gpurun_out
for c in llama2-13b-tp2 llama2-70b-tp8; do for m in ce zerocopy; do
  timeout 600 python bench.py --config $c --mode $m --steps 5 --warmup 3 --cpu-sample-gib 2 > gpurun_out/bench_${c}_$m.json 2> gpurun_out/bench_${c}_$m.err
done; done
for w in 256 512 1024; do
  SLLM_SCATTER_WINDOW_MIB=$w timeout 600 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline --no-standalone > gpurun_out/bench_scatter_ce_w$w.json 2> gpurun_out/bench_scatter_ce_w$w.err
done
