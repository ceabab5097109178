# r02x: does cuFileDriverOpen return under any cufile.json variant on this box? (20 s each)
O=gpurun_out/gds_variants; mkdir -p $O
for v in nothreads nopoll_nocache compat_only no_udev; do
  CUFILE_ENV_PATH_JSON=$PWD/tools/gds/cufile_$v.json timeout -s KILL 20 python tools/probe_gds.py /tmp raw > $O/probe_$v.txt 2>&1
  echo "$v rc=$?" >> $O/summary.txt
done
CUFILE_FORCE_COMPAT_MODE=true CUFILE_ENV_PATH_JSON=$PWD/tools/gds/cufile_nothreads.json timeout -s KILL 20 python tools/probe_gds.py /tmp raw > $O/probe_envforce.txt 2>&1; echo "envforce rc=$?" >> $O/summary.txt
