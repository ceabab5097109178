#!/bin/bash
# One GPU call: tests, smoke, bench.  Outputs -> gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for m in ${BENCH_MODES:-zerocopy ce}; do
  timeout 600 python bench.py --mode $m --steps 5 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_$m.json 2> gpurun_out/bench_$m.err
done
