"""Host-side phases of one load (latency-bound workloads: the LoRA adapter, SURVEY §8(f)
rank 3): index parse, sllm_load_start, Python tensor views, wait, free -- host clock, plus
the library's device time, over `reps` loads of the same pinned checkpoint.

    python tools/host_overhead.py [--config lora-70b-r32] [--mode ce] [--reps 20]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="lora-70b-r32")
    ap.add_argument("--mode", default="ce")
    ap.add_argument("--chunk-mib", type=int, default=64)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch
    import paper_2401_14351_b200 as sllm
    from paper_2401_14351_b200 import workloads
    from synth import models
    inv, seed = models.model_inventory(args.config)
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20, args.config, partitions=[0], gpu_of={0: 0})
    blob = idx.serialize()
    cfg = sllm.LoadConfig(chunk_bytes=args.chunk_mib << 20, mode=args.mode)
    bases, per = sllm.allocate(idx, {0: 0}, cfg.scatter)
    st = torch.cuda.current_stream()
    rows = []
    for r in range(args.reps + 3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ix = sllm.Index.from_bytes(blob)
        t1 = time.perf_counter()
        res = sllm.load_start(ix, bufs, {0: 0}, cfg, bases, per, {0: st})
        t2 = time.perf_counter()
        rep = res.wait()
        t3 = time.perf_counter()
        del res, ix
        t4 = time.perf_counter()
        if r >= 3:
            rows.append({"parse": t1 - t0, "start+views": t2 - t1, "wait": t3 - t2, "free": t4 - t3, "total": t4 - t0,
                         "device": rep["t_device_ms_max"] * 1e-3, "issue": rep["t_issue_ns_max"] * 1e-9,
                         "lib_total": rep["t_total_ns"] * 1e-9})
    med = {k: statistics.median(r[k] for r in rows) * 1e3 for k in rows[0]}
    print(json.dumps({"config": args.config, "mode": args.mode, "tensors": len(inv),
                      "bytes": idx.partitions[0].length, "median_ms": med}))


if __name__ == "__main__":
    main()
