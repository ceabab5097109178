# r02ah: H2D peak through plain cudaMemcpyAsync (cuda-python) vs torch copy_
O=gpurun_out/r02ah; mkdir -p $O
for cfg in toy lora-70b-r32 opt-6.7b; do
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"peak\": \"cudart\", /" >> $O/peaks.jsonl 2>> $O/err.txt
  SLLM_BENCH_PEAK_TORCH=1 timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"peak\": \"torch\", /" >> $O/peaks.jsonl 2>> $O/err.txt
done
