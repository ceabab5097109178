O=gpurun_out/r02h; mkdir -p $O
for v in default stage8 stage32 stage64 lanes2 lanes4 stage32_lanes4; do
  if [ $v = default ]; then LP=""; else LP=build/ab/$v/libsllm.so; fi
  SLLM_LIB_PATH=$LP timeout 300 python bench.py --mode zerocopy --steps 5 --warmup 2 --no-cpu-baseline --no-standalone \
     | sed "s/^{/{\"variant\": \"$v\", /" >> $O/zc_ab.jsonl 2>> $O/zc_ab.err
done
M=gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,pcie__throughput.avg.pct_of_peak_sustained_elapsed
timeout 600 ncu --replay-mode range --nvtx --nvtx-include "probe/" --metrics $M --csv --log-file $O/pcie_range.csv \
   python tools/pcie_probe.py > $O/pcie_range.log 2>&1
timeout 600 ncu --replay-mode application --nvtx --nvtx-include "probe/" --metrics $M --csv --log-file $O/pcie_app_range.csv \
   python tools/pcie_probe.py > $O/pcie_app_range.log 2>&1
timeout 600 ncu -k regex:materialise_tma --nvtx --nvtx-include "probe/zerocopy_k2" \
   --metrics $M,syslts__t_requests_aperture_sysmem.sum,syslts__t_sectors_aperture_sysmem.sum,lts__t_sectors_srcunit_tex_aperture_sysmem.sum \
   --csv --log-file $O/pcie_k2_kernel.csv python tools/pcie_probe.py > $O/pcie_k2_kernel.log 2>&1
