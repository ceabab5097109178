# compute-sanitizer over every mode / engine / fan-out of the toy load (tests/sanitize_gpu.py)
mkdir -p gpurun_out/sanitizer
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 99 --print-limit 50 python tests/sanitize_gpu.py \
      > gpurun_out/sanitizer/$t.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer/$t.log
done
