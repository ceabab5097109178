# bench regression after the --spread change, and --spread itself (degenerate on one GPU:
# every partition of a multi-partition config on cuda:0 from one process)
mkdir -p gpurun_out/spread
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/spread/bench_ce.json 2> gpurun_out/spread/bench_ce.err
timeout 900 python bench.py --config llama2-13b-tp2 --all-partitions --spread --steps 3 --warmup 3 --cpu-sample-gib 1 > gpurun_out/spread/bench_13b_spread.json 2> gpurun_out/spread/bench_13b_spread.err
timeout 600 python bench.py --mode scatter_ce --config llama2-13b-tp2 --all-partitions --spread --steps 3 --warmup 3 --no-cpu-baseline --no-standalone > gpurun_out/spread/bench_13b_spread_scatter.json 2> gpurun_out/spread/bench_13b_spread_scatter.err
