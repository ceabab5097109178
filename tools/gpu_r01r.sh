# r01r: GPU suite after the SCATTER_CE window plan and the NCCL fan-out verification spans
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_scatter_ce.json 2> gpurun_out/bench_scatter_ce.err
for f in bcast allgather; do
  timeout 600 python bench.py --config opt-30b --fanout $f --steps 3 --warmup 3 --no-standalone --cpu-sample-gib 2 > gpurun_out/bench_opt30b_$f.json 2> gpurun_out/bench_opt30b_$f.err
done
timeout 600 python bench.py --config lora-70b-r32 --mode scatter_ce --steps 20 --warmup 5 --no-cpu-baseline --no-standalone > gpurun_out/bench_lora70b_r32_scatter_ce.json 2> gpurun_out/bench_lora70b_r32_scatter_ce.err
