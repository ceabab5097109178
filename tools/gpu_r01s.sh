# r01s: LoRA / OPT-6.7B scatter-mode sweeps after the SCATTER_CE window plan (A/B vs 256 MiB windows)
mkdir -p gpurun_out
timeout 600 python tools/sweep.py --config lora-70b-r32 --modes scatter_ce,scatter_zc,ce --chunks 4,16,64 --streams 2 --reps 5 > gpurun_out/sweep_lora_scatter.jsonl 2> gpurun_out/sweep_lora_scatter.err
SLLM_SCATTER_WINDOW_MIB=256 timeout 600 python tools/sweep.py --config lora-70b-r32 --modes scatter_ce --chunks 4,16,64 --streams 2 --reps 5 > gpurun_out/sweep_lora_scatter_w256.jsonl 2> gpurun_out/sweep_lora_scatter_w256.err
timeout 900 python tools/sweep.py --config opt-6.7b --modes scatter_ce --chunks 1,4,16,64 --streams 2 --reps 3 > gpurun_out/sweep_opt67b_scatter_ce.jsonl 2> gpurun_out/sweep_opt67b_scatter_ce.err
