# r02av: fine tail from one wave of blocks (2 CTAs/SM) -- tests, LoRA / OPT spans, benches
O=gpurun_out/r02av; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_schedule.py tests/test_gpu_load.py tests/test_gpu_edges.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
SLLM_PROFILE_DUMP=1 SLLM_KTIME=1 timeout 300 python tools/timeline.py --config lora-70b-r32 --reps 3 --profile 1 > $O/ktime_lora.txt 2>&1
SLLM_PROFILE_DUMP=1 SLLM_KTIME=1 timeout 300 python tools/timeline.py --config opt-6.7b --reps 2 --profile 1 > $O/ktime_ce.txt 2>&1
for rep in 1 2; do
timeout 300 python bench.py --config lora-70b-r32 --steps 20 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"rep\": $rep, /" >> $O/bench_lora.jsonl 2>> $O/bench.err
timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline | sed "s/^{/{\"rep\": $rep, /" >> $O/bench_ce.jsonl 2>> $O/bench.err
done
