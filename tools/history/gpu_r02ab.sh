# r02ab: where a toy load's 0.44 ms goes (host phases, device timeline)
O=gpurun_out/r02ab; mkdir -p $O
timeout 300 python tools/host_overhead.py --config toy --reps 50 > $O/host_overhead_toy.jsonl 2>&1
SLLM_PROFILE_DUMP=1 SLLM_KTIME=1 timeout 300 python tools/timeline.py --config toy --reps 5 --profile 2 > $O/timeline_toy.txt 2>&1
SLLM_PROFILE_DUMP=1 SLLM_KTIME=1 timeout 300 python tools/timeline.py --config toy --reps 5 --profile 2 --chunk-mib 2 > $O/timeline_toy_2mib.txt 2>&1
timeout 300 python bench.py --config toy --steps 50 --warmup 5 --no-cpu-baseline --no-standalone > $O/bench_toy.json 2>> $O/bench.err
timeout 300 python bench.py --config toy --mode zerocopy --steps 50 --warmup 5 --no-cpu-baseline --no-standalone > $O/bench_toy_zc.json 2>> $O/bench.err
