O=gpurun_out/r02aq; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python -m pytest tests/test_gpu_load.py tests/test_gpu_edges.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_ce.json 2> $O/bench_ce.err
