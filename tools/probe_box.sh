#!/bin/bash
# One-shot box probe: topology, PCIe link, NUMA, host RAM, and a torch H2D bandwidth baseline.
mkdir -p gpurun_out
{
echo "== nproc"; nproc; echo "== affinity"; python -c "import os; print(len(os.sched_getaffinity(0)), os.cpu_count())"
echo "== lscpu"; lscpu | head -30
echo "== free"; free -g
echo "== nvidia-smi"; nvidia-smi
echo "== topo"; nvidia-smi topo -m
echo "== pcie"; nvidia-smi --query-gpu=index,pci.bus_id,pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,pcie.link.width.max,memory.total --format=csv
for d in /sys/bus/pci/devices/*; do if [ -f $d/vendor ] && grep -q 0x10de $d/vendor && grep -q 0x030 $d/class 2>/dev/null; then echo "$d numa=$(cat $d/numa_node) speed=$(cat $d/current_link_speed) width=$(cat $d/current_link_width) mrrs?"; fi; done
echo "== numa"; ls /sys/devices/system/node/ ; cat /sys/devices/system/node/node*/cpulist
echo "== hugepages"; cat /sys/kernel/mm/transparent_hugepage/enabled; grep -i huge /proc/meminfo
echo "== ulimit"; ulimit -l
echo "== iommu"; ls /sys/class/iommu 2>/dev/null | head; cat /proc/cmdline
echo "== df"; df -h / /tmp
} > gpurun_out/probe.txt 2>&1
python - >> gpurun_out/probe.txt 2>&1 <<'PY'
import torch, time
n = 4 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, nb in [("4GiB", n), ("256MiB", 256<<20), ("16MiB", 16<<20)]:
    best = 0
    for _ in range(5):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        d[:nb].copy_(h[:nb], non_blocking=True)
        e.record(); torch.cuda.synchronize()
        best = max(best, nb / (s.elapsed_time(e) * 1e-3) / 1e9)
    print(f"H2D torch {name}: best {best:.2f} GB/s")
best = 0
for _ in range(5):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    h.copy_(d, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    best = max(best, n / (s.elapsed_time(e) * 1e-3) / 1e9)
print(f"D2H torch 4GiB: best {best:.2f} GB/s")
print(torch.cuda.get_device_properties(0))
PY
