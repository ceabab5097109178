mkdir -p gpurun_out
for m in ce zerocopy; do timeout 300 python tools/host_overhead.py --mode $m >> gpurun_out/host_overhead.jsonl 2>&1; done
timeout 300 python tools/host_overhead.py --config toy --mode zerocopy >> gpurun_out/host_overhead.jsonl 2>&1
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -s > gpurun_out/pytest_fullsize.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fullsize.log
free -g >> gpurun_out/pytest_fullsize.log
