mkdir -p gpurun_out/sanitizer
timeout 900 python -m pytest tests/test_gpu_fanout_p2p.py tests/test_gpu_load.py -q -x -k "files or auto or p2p" > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
timeout 900 python tools/sweep_sizes.py > gpurun_out/sweep_sizes.jsonl 2>&1
for m in zerocopy:tma ce:tma scatter_zc:tma; do
  SANITIZE_ONLY=$m timeout 600 compute-sanitizer --tool initcheck --error-exitcode 99 --print-limit 5 python tools/sanitize_gpu.py > gpurun_out/sanitizer/initcheck_${m%%:*}.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer/initcheck_${m%%:*}.log
done
