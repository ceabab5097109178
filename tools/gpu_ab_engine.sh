# K3 engine A/B with kernel-only timing: TMA ring + vector stores vs + TMA bulk stores
mkdir -p gpurun_out/eng
for e in tma tma_store; do
  SLLM_STANDALONE_ENGINE=$e timeout 600 python bench.py --engine $e --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/eng/bench_scatter_ce_$e.json 2> gpurun_out/eng/bench_scatter_ce_$e.err
  timeout 600 python bench.py --engine $e --mode scatter_zc --steps 5 --warmup 3 --no-cpu-baseline --no-standalone > gpurun_out/eng/bench_scatter_zc_$e.json 2> gpurun_out/eng/bench_scatter_zc_$e.err
done
