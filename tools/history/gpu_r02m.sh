# r02m: clean bench lines after the kMc split, sanitizers on the r02 pipeline (pinned setup block,
# result readback, NUMA binding), short soak
O=gpurun_out/r02m; mkdir -p $O/sanitizer
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_ce.json 2> $O/bench_ce.err
timeout 300 python bench.py --config lora-70b-r32 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_lora.json 2> $O/bench_lora.err
timeout 300 python bench.py --config toy --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_toy.json 2> $O/bench_toy.err
timeout 600 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_scatter_ce.json 2> $O/bench_scatter_ce.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python -m pytest tests/test_gpu_load.py tests/test_gpu_multi.py tests/test_gpu_edges.py tests/test_numa.py -q > $O/pytest_subset.log 2>&1; echo "rc=$?" >> $O/pytest_subset.log
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 99 --print-limit 50 python tools/sanitize_gpu.py \
      > $O/sanitizer/$t.log 2>&1; echo "rc=$?" >> $O/sanitizer/$t.log
done
SANITIZE_ONLY=ring timeout 900 compute-sanitizer --tool racecheck --error-exitcode 99 --print-limit 50 python tools/sanitize_gpu.py \
      > $O/sanitizer/racecheck_ring.log 2>&1; echo "rc=$?" >> $O/sanitizer/racecheck_ring.log
timeout 900 python tools/soak.py --config opt-6.7b --loads 30 > $O/soak.jsonl 2> $O/soak.err
