# P2P fan-out check: its GPU tests, then bench.py in the replicated modes at N=1 (opt-6.7b, one partition)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fanout_p2p.py -q -x > gpurun_out/pytest_p2p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p2p.log
for f in p2p bcast; do for m in ce zerocopy; do
  timeout 600 python bench.py --mode $m --fanout $f --steps 5 --warmup 3 --no-cpu-baseline --no-standalone > gpurun_out/bench_${f}_${m}.json 2>&1
done; done
