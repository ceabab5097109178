mkdir -p gpurun_out
timeout 600 python tools/probe_p2p_group.py > gpurun_out/probe_p2p_group.jsonl 2> gpurun_out/probe_p2p_group.err
timeout 600 python -m pytest tests/test_gpu_load.py -q -x -k "nccl or allgather" > gpurun_out/pytest_allgather.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_allgather.log
