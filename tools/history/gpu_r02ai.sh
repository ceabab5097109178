O=gpurun_out/r02ai; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_load.py tests/test_c_abi.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
