O=gpurun_out/r02ao; mkdir -p $O
timeout 1500 python tools/sweep.py --config opt-6.7b --reps 5 > $O/sweep_opt67b.jsonl 2> $O/sweep.err
