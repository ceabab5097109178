# r02r: launch overhead with PCIe saturated (and as a CUDA graph); standalone K4 in-kernel spans
O=gpurun_out/r02r; mkdir -p $O
for spin in 50 300; do timeout 120 build/launch_gap $spin >> $O/launch_gap.jsonl 2>&1; done
SLLM_KTIME=1 timeout 300 python tools/k4_sizes.py --max-gib 4 > $O/k4_sizes_ktime.jsonl 2>&1
