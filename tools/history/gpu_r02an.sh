# r02an: chunk-size sweeps on the final code (BASELINE configs[1]; LoRA, toy)
O=gpurun_out/r02an; mkdir -p $O
timeout 1200 python tools/sweep.py --config opt-6.7b > $O/sweep_opt67b.jsonl 2> $O/sweep.err
timeout 600 python tools/sweep.py --config lora-70b-r32 --reps 5 > $O/sweep_lora70b_r32.jsonl 2>> $O/sweep.err
timeout 600 python tools/sweep.py --config toy --reps 10 > $O/sweep_toy.jsonl 2>> $O/sweep.err
