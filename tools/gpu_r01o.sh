mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -s -k opt30b > gpurun_out/pytest_opt30b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_opt30b.log
