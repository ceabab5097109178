# r02t: per-partition copy windows (64-256 MiB) -- GPU subset, bench lines
O=gpurun_out/r02t; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_load.py tests/test_gpu_edges.py tests/test_gpu_files.py tests/test_gpu_fanout_p2p.py -q -x > $O/pytest_subset.log 2>&1; echo "rc=$?" >> $O/pytest_subset.log
for rep in 1 2; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"rep\": $rep, /" >> $O/bench_ce.jsonl 2>> $O/bench.err
timeout 300 python bench.py --config lora-70b-r32 --steps 20 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"rep\": $rep, /" >> $O/bench_lora.jsonl 2>> $O/bench.err
timeout 300 python bench.py --mode zerocopy --steps 5 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"rep\": $rep, /" >> $O/bench_zc.jsonl 2>> $O/bench.err
done
