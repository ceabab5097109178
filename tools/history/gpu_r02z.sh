# r02z: load hint on the store kernels only (default build) -- tests, ZC / scatter / CE lines
O=gpurun_out/r02z; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_load.py tests/test_gpu_edges.py tests/test_gpu_schedule.py tests/test_gpu_fanout_p2p.py -q -x > $O/pytest_subset.log 2>&1; echo "rc=$?" >> $O/pytest_subset.log
for rep in 1 2; do
timeout 300 python bench.py --mode zerocopy --steps 5 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"rep\": $rep, /" >> $O/bench_zc.jsonl 2>> $O/bench.err
SLLM_LIB_PATH=build/ab/sthint/libsllm.so timeout 300 python bench.py --mode zerocopy --steps 5 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"rep\": $rep, \"variant\": \"no_hint\", /" >> $O/bench_zc.jsonl 2>> $O/bench.err
timeout 300 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"rep\": $rep, /" >> $O/bench_scatter.jsonl 2>> $O/bench.err
timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline | sed "s/^{/{\"rep\": $rep, /" >> $O/bench_ce.jsonl 2>> $O/bench.err
done
