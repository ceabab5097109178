mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_files.py -q -x -k gds > gpurun_out/pytest_gds.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gds.log
ls /dev/nvidia-fs* > gpurun_out/gds_probe.txt 2>&1; lsmod 2>/dev/null | grep -i nvidia_fs >> gpurun_out/gds_probe.txt; cat /tmp/cufile.log 2>/dev/null | tail -20 >> gpurun_out/gds_probe.txt; ls -la cufile.log >> gpurun_out/gds_probe.txt 2>&1; tail -20 cufile.log >> gpurun_out/gds_probe.txt 2>&1
timeout 900 python tools/bench_files.py --config opt-6.7b --io-threads 4 --reps 2 > gpurun_out/bench_files_ce.jsonl 2> gpurun_out/bench_files_ce.err
