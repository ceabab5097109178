mkdir -p gpurun_out/san4
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/san4/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/san4/pytest_gpu.log
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --error-exitcode 99 --print-limit 20 python tests/sanitize_gpu.py > gpurun_out/san4/$t.log 2>&1; echo "rc=$?" >> gpurun_out/san4/$t.log
done
