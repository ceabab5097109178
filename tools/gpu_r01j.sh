mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for e in tma tma_store; do
  SLLM_STANDALONE_ENGINE=$e timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_standalone_$e.json 2>&1
done
timeout 900 python tools/sweep.py --config opt-6.7b --modes zerocopy,scatter_ce,scatter_zc --chunks 64 --streams 2 --engines tma,tma_store --reps 3 > gpurun_out/sweep_engines.jsonl 2>&1
