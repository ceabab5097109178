# r02p: fine tail (last wave in quarter blocks) -- correctness, A/B vs SLLM_FINE_TAIL=0,
# launch overhead micro-benchmark
O=gpurun_out/r02p; mkdir -p $O/sanitizer
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_load.py tests/test_gpu_edges.py tests/test_gpu_fanout_p2p.py tests/test_gpu_concurrency.py tests/test_gpu_fullsize.py -q -x > $O/pytest_subset.log 2>&1; echo "rc=$?" >> $O/pytest_subset.log
for spin in 50 300; do timeout 60 build/launch_gap $spin >> $O/launch_gap.jsonl 2>&1; done
for v in fine nofine; do
  if [ $v = nofine ]; then export SLLM_FINE_TAIL=0; else unset SLLM_FINE_TAIL; fi
  SLLM_PROFILE_DUMP=1 SLLM_KTIME=1 timeout 300 python tools/timeline.py --config opt-6.7b --reps 3 --profile 1 > $O/ktime_ce_$v.txt 2>&1
  SLLM_PROFILE_DUMP=1 SLLM_KTIME=1 timeout 300 python tools/timeline.py --config opt-6.7b --mode scatter_ce --reps 3 --profile 1 > $O/ktime_scatter_ce_$v.txt 2>&1
  SLLM_PROFILE_DUMP=1 SLLM_KTIME=1 timeout 300 python tools/timeline.py --config lora-70b-r32 --reps 3 --profile 1 > $O/ktime_lora_$v.txt 2>&1
  timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > $O/bench_ce_$v.json 2> $O/bench_ce_$v.err
  timeout 300 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_scatter_ce_$v.json 2> $O/bench_scatter_ce_$v.err
  timeout 300 python bench.py --config lora-70b-r32 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_lora_$v.json 2> $O/bench_lora_$v.err
done
unset SLLM_FINE_TAIL
SANITIZE_ONLY=ring timeout 900 compute-sanitizer --tool racecheck --error-exitcode 99 --print-limit 50 python tools/sanitize_gpu.py \
      > $O/sanitizer/racecheck_ring.log 2>&1; echo "rc=$?" >> $O/sanitizer/racecheck_ring.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 50 python tools/sanitize_gpu.py \
      > $O/sanitizer/memcheck.log 2>&1; echo "rc=$?" >> $O/sanitizer/memcheck.log
