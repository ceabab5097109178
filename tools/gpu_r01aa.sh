mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py -q > gpurun_out/pytest_edges.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_edges.log
