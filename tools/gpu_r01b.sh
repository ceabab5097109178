set -x
mkdir -p gpurun_out
bash tools/probe_box.sh
SKIP_TESTS= bash tools/gpu_round.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:materialise_tma -s 2 -c 1 -f -o gpurun_out/prof_pipeline_ce python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-standalone > gpurun_out/ncu_pipeline.log 2>&1
timeout 600 python tools/sweep.py --config lora-70b-r32 --modes ce,zerocopy --chunks 1,4,16,64 --streams 1,2 --reps 7 > gpurun_out/sweep_lora.jsonl 2>&1
timeout 600 python tools/sweep.py --config toy --modes ce,zerocopy,scatter_ce --chunks 1,4,16 --streams 1,2 --reps 7 > gpurun_out/sweep_toy.jsonl 2>&1
