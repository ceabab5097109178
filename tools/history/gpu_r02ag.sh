# r02ag: barrier-free unit-end reduction -- correctness (tests, racecheck / memcheck on the
# ring-wrap set), A/B timing against the barrier version (build/ab/base)
O=gpurun_out/r02ag; mkdir -p $O/sanitizer
timeout 1200 python -m pytest tests/test_gpu_load.py tests/test_gpu_edges.py tests/test_gpu_schedule.py tests/test_gpu_fanout_p2p.py tests/test_gpu_concurrency.py -q -x > $O/pytest_subset.log 2>&1; echo "rc=$?" >> $O/pytest_subset.log
SANITIZE_ONLY=ring timeout 900 compute-sanitizer --tool racecheck --error-exitcode 99 --print-limit 50 python tools/sanitize_gpu.py > $O/sanitizer/racecheck_ring.log 2>&1; echo "rc=$?" >> $O/sanitizer/racecheck_ring.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 99 --print-limit 50 python tools/sanitize_gpu.py > $O/sanitizer/racecheck.log 2>&1; echo "rc=$?" >> $O/sanitizer/racecheck.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 50 python tools/sanitize_gpu.py > $O/sanitizer/memcheck.log 2>&1; echo "rc=$?" >> $O/sanitizer/memcheck.log
M=gpu__time_duration.sum
for rep in 1 2; do for v in base new; do
  if [ $v = base ]; then export SLLM_LIB_PATH=build/ab/base/libsllm.so; else unset SLLM_LIB_PATH; fi
  timeout 600 ncu --metrics $M --clock-control none --csv -k regex:materialise -c 4 python tools/ncu_kernels.py 2>/dev/null | grep materialise | sed "s/^/$v,$rep,/" >> $O/ncu.csv
  SLLM_KTIME=1 timeout 300 python tools/k4_sizes.py --max-gib 4 --reps 5 2>&1 | grep "ktime bytes=4294967296" | sed "s/^/$v $rep /" >> $O/k4_live.txt
  timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $O/bench_ce.jsonl 2>> $O/bench.err
  timeout 300 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $O/bench_scatter.jsonl 2>> $O/bench.err
done; done
unset SLLM_LIB_PATH
