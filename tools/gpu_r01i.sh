mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --config llama2-70b-tp8 --all-partitions --steps 3 --warmup 3 --no-standalone --cpu-sample-gib 2 > gpurun_out/bench_70b_tp8_all.json 2> gpurun_out/bench_70b_tp8_all.err
timeout 600 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_scatter_ce.json 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_ce.json 2>&1
