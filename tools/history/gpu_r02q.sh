# r02q: launch overhead micro-benchmark; where cuFileDriverOpen blocks
O=gpurun_out/r02q; mkdir -p $O
for spin in 50 300; do timeout 60 build/launch_gap $spin >> $O/launch_gap.jsonl 2>&1; done
timeout 120 bash tools/gds_hang_dump.sh $O
