# r02ak: final code -- full GPU suite, smoke, soak through the public API
O=gpurun_out/r02ak; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python tools/soak.py --config opt-6.7b --loads 100 > $O/soak.jsonl 2> $O/soak.err; echo "soak rc=$?" >> $O/soak.err
