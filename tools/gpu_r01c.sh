# file tier + zero-copy tuning + in-pipeline ZC capture
mkdir -p gpurun_out
timeout 900 python tools/bench_files.py --config opt-6.7b --io-threads 1,2,4,8 --reps 2 > gpurun_out/bench_files.jsonl 2>&1
timeout 900 python tools/sweep.py --config opt-6.7b --modes zerocopy --chunks 16,64 --streams 1,2,3 --ctas 32,64,96,148 --reps 2 > gpurun_out/sweep_zc_ctas.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:materialise_tma -s 6 -c 1 -f \
   -o gpurun_out/prof_pipeline_zc python bench.py --mode zerocopy --steps 1 --warmup 0 --no-cpu-baseline --no-standalone > gpurun_out/ncu_pipeline_zc.log 2>&1
