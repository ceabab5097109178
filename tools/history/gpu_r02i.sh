O=gpurun_out/r02i; mkdir -p $O
M=gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,pcie__throughput.avg.pct_of_peak_sustained_elapsed
timeout 600 ncu --replay-mode range --nvtx --nvtx-include "probe_ce/" --metrics $M --csv --log-file $O/pcie_ce_range.csv \
   python tools/pcie_probe.py > $O/pcie_ce_range.log 2>&1
timeout 600 ncu -k regex:materialise_tma -s 32 -c 1 \
   --metrics $M,syslts__t_requests_aperture_sysmem.sum,syslts__t_sectors_aperture_sysmem.sum,dram__bytes_write.sum \
   --csv --log-file $O/pcie_k2_kernel.csv python tools/pcie_probe.py > $O/pcie_k2_kernel.log 2>&1
