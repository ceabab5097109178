"""Standalone launches of the HBM-side kernels for ncu:
K4 (checksum only) over a 4 GiB device buffer and K3 (index-driven scatter + checksum)
over a device-resident OPT-6.7B-shaped partition image (13.3 GB) into per-tensor
buffers.  Inputs are >= 1 GiB so the 126 MB L2 cannot hold them.

    ncu --set full -k regex:materialise -c 4 -o gpurun_out/prof python tools/ncu_kernels.py
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

    n = 4 << 30
    buf = torch.empty(n, dtype=torch.uint8, device="cuda")
    buf.random_(0, 256)
    out = torch.empty(n >> 20, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(2):
        sllm.block_checksums_device(buf.data_ptr(), n, 1 << 20, out.data_ptr(), 0, st)
    torch.cuda.synchronize()
    del buf, out
    inv, _ = models.model_inventory(os.environ.get("NCU_CONFIG", "opt-6.7b"))
    idx = workloads.plan_inventory(inv)
    idx.seal([None] * len(idx.partitions))  # checksums stay 0: the scatter still moves every byte
    L = idx.partitions[0].length
    src = torch.empty(L, dtype=torch.uint8, device="cuda")
    src.random_(0, 256)
    _, per = sllm.allocate(idx, {0: 0}, scatter=True)
    for _ in range(2):
        try:
            sllm.materialise_device(idx, 0, src.data_ptr(), per, 0, st)
        except sllm.SllmError as ex:
            assert ex.status == 9  # random image vs zero table: mismatch expected, bytes moved
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
