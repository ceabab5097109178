# r02o: dynamic unit distribution (tickets) -- correctness first, then A/B against the static
# schedule (SLLM_STATIC_UNITS=1) on in-kernel spans, standalone K4/K3 and the bench lines
O=gpurun_out/r02o; mkdir -p $O/sanitizer
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_load.py tests/test_gpu_edges.py tests/test_gpu_fanout_p2p.py tests/test_gpu_concurrency.py -q -x > $O/pytest_subset.log 2>&1; echo "rc=$?" >> $O/pytest_subset.log
for v in dyn static; do
  if [ $v = static ]; then export SLLM_STATIC_UNITS=1; else unset SLLM_STATIC_UNITS; fi
  SLLM_PROFILE_DUMP=1 SLLM_KTIME=1 timeout 300 python tools/timeline.py --config opt-6.7b --reps 3 --profile 1 > $O/ktime_ce_$v.txt 2>&1
  SLLM_PROFILE_DUMP=1 SLLM_KTIME=1 timeout 300 python tools/timeline.py --config opt-6.7b --mode scatter_ce --reps 3 --profile 1 > $O/ktime_scatter_ce_$v.txt 2>&1
  timeout 300 python tools/k4_sizes.py --max-gib 4 > $O/k4_sizes_$v.jsonl 2>&1
  timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > $O/bench_ce_$v.json 2> $O/bench_ce_$v.err
  timeout 300 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_scatter_ce_$v.json 2> $O/bench_scatter_ce_$v.err
done
unset SLLM_STATIC_UNITS
SANITIZE_ONLY=ring timeout 900 compute-sanitizer --tool racecheck --error-exitcode 99 --print-limit 50 python tools/sanitize_gpu.py \
      > $O/sanitizer/racecheck_ring.log 2>&1; echo "rc=$?" >> $O/sanitizer/racecheck_ring.log
SANITIZE_ONLY=ring timeout 900 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 50 python tools/sanitize_gpu.py \
      > $O/sanitizer/memcheck_ring.log 2>&1; echo "rc=$?" >> $O/sanitizer/memcheck_ring.log
