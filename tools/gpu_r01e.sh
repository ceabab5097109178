mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_nvls tools/probe_nvls.cu -lcuda > gpurun_out/probe_nvls.txt 2>&1
timeout 120 /tmp/probe_nvls >> gpurun_out/probe_nvls.txt 2>&1; echo "rc=$?" >> gpurun_out/probe_nvls.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
