O=gpurun_out/r02k; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python tools/k4_sizes.py > $O/k4_sizes.jsonl 2> $O/k4_sizes.err
SLLM_LIB_PATH=build/ab/carve100/libsllm.so timeout 300 python tools/k4_sizes.py > $O/k4_sizes_carve100.jsonl 2>> $O/k4_sizes.err
for span in 2048 4096 8192; do
  SLLM_VERIFY_SPAN_MIB=$span timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-standalone \
     | sed "s/^{/{\"span_mib\": $span, /" >> $O/span_sweep.jsonl 2>> $O/span_sweep.err
done
SLLM_LIB_PATH=build/ab/carve100/libsllm.so timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-standalone \
     | sed "s/^{/{\"variant\": \"carve100\", /" >> $O/span_sweep.jsonl 2>> $O/span_sweep.err
