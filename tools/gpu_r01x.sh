mkdir -p gpurun_out
export CUFILE_ENV_PATH_JSON=$PWD/tools/gds/cufile_compat.json
timeout 90 python tools/probe_gds.py /tmp raw > gpurun_out/gds_probe2.log 2>&1; echo "raw force_compat rc=$?" >> gpurun_out/gds_probe2.log
ls gpurun_out/ >> gpurun_out/gds_probe2.log
