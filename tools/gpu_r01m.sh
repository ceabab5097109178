# r01m: full-size replicated OPT-30B (P2P, 2 replicas on one GPU), OPT-30B bench lines,
# standalone K3 timed around the launch only.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -s -k opt30b > gpurun_out/pytest_opt30b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_opt30b.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_ce.json 2> gpurun_out/bench_ce.err
for f in none p2p bcast; do
  timeout 600 python bench.py --config opt-30b --fanout $f --steps 3 --warmup 3 --no-standalone --cpu-sample-gib 2 > gpurun_out/bench_opt30b_$f.json 2> gpurun_out/bench_opt30b_$f.err
done
