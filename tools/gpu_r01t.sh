# r01t: granule segment table (K3/K2 scatter) + small-partition window plan
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_scatter_ce.json 2> gpurun_out/bench_scatter_ce.err
timeout 600 python bench.py --mode scatter_zc --steps 5 --warmup 3 --no-cpu-baseline --no-standalone > gpurun_out/bench_scatter_zc.json 2> gpurun_out/bench_scatter_zc.err
timeout 600 python tools/sweep.py --config lora-70b-r32 --modes scatter_ce,scatter_zc --chunks 4,16,64 --streams 2 --reps 5 > gpurun_out/sweep_lora_scatter.jsonl 2> gpurun_out/sweep_lora_scatter.err
