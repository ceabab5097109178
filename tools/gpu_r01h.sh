mkdir -p gpurun_out
timeout 1200 python bench.py --config llama2-70b-tp8 --all-partitions --steps 3 --warmup 3 --no-standalone --cpu-sample-gib 2 > gpurun_out/bench_70b_tp8_all.json 2> gpurun_out/bench_70b_tp8_all.err
