# racecheck + memcheck over loads whose CTAs wrap the stage ring (both TMA engines, every
# contiguous/scatter mode, the P2P fan-out), then the zero-copy bench line
mkdir -p gpurun_out/ring
for t in racecheck memcheck; do
  SANITIZE_ONLY=ring timeout 1500 compute-sanitizer --tool $t --error-exitcode 99 --print-limit 20 python tests/sanitize_gpu.py > gpurun_out/ring/$t.log 2>&1; echo "rc=$?" >> gpurun_out/ring/$t.log
done
timeout 600 python bench.py --mode zerocopy --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ring/bench_zerocopy.json 2> gpurun_out/ring/bench_zerocopy.err
