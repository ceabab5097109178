# r02aa: step-time outliers (per-step list), ZC without the load hint, tests
O=gpurun_out/r02aa; mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1; nvidia-smi topo -m > $O/topo.txt 2>&1; cat /proc/loadavg > $O/loadavg.txt
timeout 600 python -m pytest tests/test_gpu_load.py tests/test_gpu_schedule.py -q -x > $O/pytest_subset.log 2>&1; echo "rc=$?" >> $O/pytest_subset.log
for rep in 1 2 3; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"rep\": $rep, /" >> $O/bench_ce.jsonl 2>> $O/bench.err
cat /proc/loadavg >> $O/loadavg.txt
timeout 300 python bench.py --mode zerocopy --steps 5 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"rep\": $rep, /" >> $O/bench_zc.jsonl 2>> $O/bench.err
done
