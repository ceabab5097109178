# r01u: unit-size A/B (K4 in the CE pipeline, K3 in SCATTER_CE, standalone K3/K4)
mkdir -p gpurun_out
for u in 1024 256 128; do
  SLLM_UNIT_KIB=$u timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ce_u$u.json 2> gpurun_out/bench_ce_u$u.err
  SLLM_UNIT_KIB=$u timeout 600 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline --no-standalone > gpurun_out/bench_scatter_ce_u$u.json 2> gpurun_out/bench_scatter_ce_u$u.err
done
