"""Probe: does SM-issued zero-copy reading add bandwidth on top of the copy engine?

OPT-6.7B-shaped tensors split into two logical partitions on GPU 0: the first share
loaded by the copy engine (mode ce), the rest concurrently by the zero-copy TMA kernel
(mode zerocopy).  Prints aggregate GB/s per split fraction.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2401_14351_b200 as sllm
    from paper_2401_14351_b200 import workloads
    from synth import models
    inv, seed = models.model_inventory("opt-6.7b")
    total = sum(t.nbytes for t in inv)
    for frac in (0.0, 0.08, 0.15, 0.25):
        acc, out = 0, []
        for t in inv:
            dev = 1 if acc >= total * (1 - frac) else 0
            acc += t.nbytes
            out.append(models.TensorSpec(t.name, dev, t.dtype, t.shape))
        idx, bufs = workloads.build_pinned(out, seed, 4096, 1 << 20, "hyb")
        n = len(idx.partitions)
        bases, _ = sllm.allocate(idx, {p: 0 for p in range(n)})
        modes = ["ce", "zerocopy"]
        best = 0
        for rep in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rs = []
            for p in range(n):
                cfg = sllm.LoadConfig(chunk_bytes=64 << 20, mode=modes[p], n_streams=2)
                rs.append(sllm.load_start(idx, {p: bufs[p]}, {p: 0}, cfg, {p: bases[p]}))
            for r in rs:
                r.wait()
            dt = time.perf_counter() - t0
            if rep:
                best = max(best, total / dt / 1e9)
            del rs
        print(json.dumps({"zc_fraction": frac, "GBps_best": best, "partitions": n}), flush=True)
        del bases, bufs, idx
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
