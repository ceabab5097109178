mkdir -p gpurun_out
df -T /tmp . > gpurun_out/gds_probe.log 2>&1
timeout 120 python tools/probe_gds.py /tmp raw >> gpurun_out/gds_probe.log 2>&1; echo "raw /tmp rc=$?" >> gpurun_out/gds_probe.log
timeout 120 python tools/probe_gds.py $PWD/gpurun_out raw >> gpurun_out/gds_probe.log 2>&1; echo "raw repo rc=$?" >> gpurun_out/gds_probe.log
timeout 120 python tools/probe_gds.py /tmp lib >> gpurun_out/gds_probe.log 2>&1; echo "lib /tmp rc=$?" >> gpurun_out/gds_probe.log
cat cufile.log >> gpurun_out/gds_probe.log 2>&1
rm -f gpurun_out/gds_probe.bin
