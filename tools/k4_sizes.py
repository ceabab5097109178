"""K4 (checksum-only kernel) launch time vs bytes on a device-resident buffer: CUDA events
around each launch on its stream, best of `reps`; the least-squares fit t = a + bytes / r
separates the fixed per-launch cost `a` from the streaming rate `r` (VERDICT r1 weak #6:
the in-pipeline K4 fraction is short-launch-bound).

    python tools/k4_sizes.py [--max-gib 8]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-gib", type=int, default=8)
    ap.add_argument("--reps", type=int, default=7)
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2401_14351_b200 as sllm
    n_max = args.max_gib << 30
    src = torch.randint(0, 256, (n_max,), dtype=torch.uint8, device="cuda")
    out = torch.empty(n_max >> 20, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    rows = []
    n = 64 << 20
    while n <= n_max:
        ts = []
        for _ in range(args.reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            sllm.block_checksums_device(src.data_ptr(), n, 1 << 20, out.data_ptr(), 0, st)
            b.record(st)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        rows.append({"bytes": n, "ms": min(ts), "GBps": n / min(ts) / 1e6})
        print(json.dumps(rows[-1]), flush=True)
        n *= 2
    x = np.array([r["bytes"] for r in rows], float)
    y = np.array([r["ms"] for r in rows], float) * 1e-3
    A = np.stack([np.ones_like(x), x], 1)
    (a, inv_r), *_ = np.linalg.lstsq(A, y, rcond=None)
    print(json.dumps({"fit": "t = a + bytes / r", "a_us": a * 1e6, "r_GBps": 1 / inv_r / 1e9}), flush=True)


if __name__ == "__main__":
    main()
