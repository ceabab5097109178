"""PCIe view of the two host->device transfer mechanisms: one copy-engine
copy and one zero-copy K2 launch over the same pinned bytes, each inside an NVTX range, for
`ncu --replay-mode range` (PCIe counters of the whole range) and kernel replay (K2 alone).

    ncu --replay-mode range --nvtx --nvtx-include "probe_ce/" --metrics <pcie metrics> python tools/pcie_probe.py
    ncu -k regex:materialise_tma -s 32 -c 1 --metrics <pcie metrics> python tools/pcie_probe.py   (the K2 of
        the probe load: one 1 GiB launch after 2 x 16 warm-up launches; K2 runs on a worker thread, outside
        the main thread's NVTX ranges)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2401_14351_b200 as sllm
    from paper_2401_14351_b200 import workloads
    from synth import models
    n = int(os.environ.get("PROBE_MIB", "1024"))
    inv = [models.TensorSpec(f"w{i}", 0, "f16", (4096, 8192)) for i in range(n // 64)]  # 64 MiB tensors
    idx, bufs = workloads.build_pinned(inv, 9, 4096, 1 << 20)
    L = idx.partitions[0].length
    dst = torch.empty(L, dtype=torch.uint8, device="cuda")
    src = bufs[0].torch()
    for _ in range(2):  # warm
        dst.copy_(src, non_blocking=True)
        sllm.load(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=64 << 20, mode="zerocopy")).free()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("probe_ce")
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    torch.cuda.nvtx.range_push("probe_zc")
    res = sllm.load_start(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 30, mode="zerocopy", verify=False),
                          {0: dst}, None, None)
    res.wait()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    res.free()
    print("probe done", L)


if __name__ == "__main__":
    main()
