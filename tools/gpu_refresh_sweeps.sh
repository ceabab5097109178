# refresh the chunk-size / mode sweeps and the full-size parity log on the final kernels
mkdir -p gpurun_out/refresh
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -s > gpurun_out/refresh/pytest_fullsize.log 2>&1; echo "rc=$?" >> gpurun_out/refresh/pytest_fullsize.log
timeout 1800 python tools/sweep.py --config opt-6.7b --modes ce,zerocopy,scatter_ce,scatter_zc --chunks 1,2,4,8,16,32,64 --streams 1,2 --reps 3 > gpurun_out/refresh/sweep_opt67b.jsonl 2> gpurun_out/refresh/sweep_opt67b.err
timeout 900 python tools/sweep.py --config lora-70b-r32 --modes ce,zerocopy,scatter_ce,scatter_zc --chunks 4,16,64 --streams 1,2 --reps 5 > gpurun_out/refresh/sweep_lora70b_r32.jsonl 2> gpurun_out/refresh/sweep_lora70b_r32.err
timeout 600 python tools/sweep.py --config toy --modes ce,zerocopy,scatter_ce,scatter_zc --chunks 1,2,4 --streams 1,2 --reps 10 > gpurun_out/refresh/sweep_toy.jsonl 2> gpurun_out/refresh/sweep_toy.err
