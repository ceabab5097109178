O=gpurun_out/r02al; mkdir -p $O
timeout 1200 python tools/soak.py --config opt-6.7b --loads 100 > $O/soak_opt67b.jsonl 2> $O/soak.err; echo "rc=$?" >> $O/soak.err
timeout 900 python tools/soak.py --config lora-70b-r32 --loads 300 > $O/soak_lora.jsonl 2>> $O/soak.err; echo "rc=$?" >> $O/soak.err
