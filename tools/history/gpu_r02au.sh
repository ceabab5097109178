# r02au: 2 CTAs/SM default -- full GPU suite, sanitizers (ring wraps 2x as often), benches
O=gpurun_out/r02au; mkdir -p $O/sanitizer
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 99 --print-limit 50 python tools/sanitize_gpu.py > $O/sanitizer/$t.log 2>&1; echo "rc=$?" >> $O/sanitizer/$t.log
done
SANITIZE_ONLY=ring timeout 900 compute-sanitizer --tool racecheck --error-exitcode 99 --print-limit 50 python tools/sanitize_gpu.py > $O/sanitizer/racecheck_ring.log 2>&1; echo "rc=$?" >> $O/sanitizer/racecheck_ring.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_ce.json 2> $O/bench_ce.err
timeout 300 python bench.py --config lora-70b-r32 --steps 20 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_lora.json 2> $O/bench_lora.err
timeout 300 python bench.py --config toy --steps 50 --warmup 5 --no-cpu-baseline --no-standalone > $O/bench_toy.json 2> $O/bench_toy.err
timeout 600 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_scatter_ce.json 2> $O/bench_scatter_ce.err
SLLM_PROFILE_DUMP=1 SLLM_KTIME=1 timeout 300 python tools/timeline.py --config lora-70b-r32 --reps 3 --profile 1 > $O/ktime_lora.txt 2>&1
