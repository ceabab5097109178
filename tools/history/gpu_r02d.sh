O=gpurun_out/r02d; mkdir -p $O
for g in 1 0; do
  timeout 300 python tools/lora_gap.py --profile 0 --clocks 1 --gc $g --steps 40 >> $O/lora_gap.jsonl 2>> $O/lora_gap.err
done
