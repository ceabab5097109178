# r02w: fine tail only for unbalanced launches; profile 3 (in-kernel spans) in the bench line
O=gpurun_out/r02w; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_schedule.py tests/test_gpu_load.py tests/test_gpu_edges.py -q -x > $O/pytest_subset.log 2>&1; echo "rc=$?" >> $O/pytest_subset.log
SLLM_PROFILE_DUMP=1 SLLM_KTIME=1 timeout 300 python tools/timeline.py --config opt-6.7b --reps 3 --profile 1 > $O/ktime_ce.txt 2>&1
SLLM_PROFILE_DUMP=1 SLLM_KTIME=1 timeout 300 python tools/timeline.py --config lora-70b-r32 --reps 3 --profile 1 > $O/ktime_lora.txt 2>&1
SLLM_PROFILE_DUMP=1 SLLM_KTIME=1 timeout 300 python tools/timeline.py --config opt-6.7b --mode scatter_ce --reps 3 --profile 1 > $O/ktime_scatter_ce.txt 2>&1
for rep in 1 2; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | sed "s/^{/{\"rep\": $rep, /" >> $O/bench_ce.jsonl 2>> $O/bench.err
timeout 300 python bench.py --config lora-70b-r32 --steps 20 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"rep\": $rep, /" >> $O/bench_lora.jsonl 2>> $O/bench.err
timeout 300 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"rep\": $rep, /" >> $O/bench_scatter_ce.jsonl 2>> $O/bench.err
done
