#!/bin/bash
# One GPU call: tests, smoke, bench, ncu launch list + full capture.  Outputs -> gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
for m in ${BENCH_MODES:-ce zerocopy}; do
  timeout 600 python bench.py --mode $m --steps 5 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_$m.json 2> gpurun_out/bench_$m.err
done
if [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-standalone > gpurun_out/ncu_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:materialise -c 4 -f \
      -o gpurun_out/prof_kernels python tools/ncu_kernels.py > gpurun_out/ncu_kernels.log 2>&1
fi
