mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fanout_p2p.py -q -x > gpurun_out/pytest_p2p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p2p.log
for i in 1 2 3; do timeout 600 python bench.py --mode ce --steps 5 --warmup 3 --no-cpu-baseline --no-standalone > gpurun_out/bench_ce_$i.json 2>&1; done
