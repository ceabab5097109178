# r02n: in-kernel timestamps vs CUDA events per K4 / K3 launch (where the in-pipeline
# per-launch overhead sits)
O=gpurun_out/r02n; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/gpu.txt 2>&1
SLLM_PROFILE_DUMP=1 SLLM_KTIME=1 timeout 300 python tools/timeline.py --config opt-6.7b --reps 3 --profile 1 > $O/ktime_ce.txt 2>&1
SLLM_PROFILE_DUMP=1 SLLM_KTIME=1 timeout 300 python tools/timeline.py --config opt-6.7b --mode scatter_ce --reps 3 --profile 1 > $O/ktime_scatter_ce.txt 2>&1
SLLM_PROFILE_DUMP=1 SLLM_KTIME=1 timeout 300 python tools/timeline.py --config lora-70b-r32 --reps 3 --profile 1 > $O/ktime_lora.txt 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_ce.json 2> $O/bench_ce.err
