# r01z: verification-span A/B (K4 in the CE pipeline) on OPT-6.7B and OPT-30B
mkdir -p gpurun_out/span
for v in 2048 4096 8192; do
  SLLM_VERIFY_SPAN_MIB=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-standalone > gpurun_out/span/bench_ce_v$v.json 2> gpurun_out/span/bench_ce_v$v.err
done
