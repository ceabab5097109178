"""Where a small load's step time goes: the
bench's step loop on the LoRA adapter with host timestamps around every phase and the
library's device time, so step time - device time = the host gap between loads.

    python tools/lora_gap.py [--config lora-70b-r32] [--steps 30] [--profile 0|1] [--clocks 0|1]
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
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--profile", type=int, default=1)
    ap.add_argument("--clocks", type=int, default=1)
    ap.add_argument("--gc", type=int, default=1, help="0: gc.disable() during the loop; 2: gc.freeze() first")
    ap.add_argument("--overlap-free", type=int, default=0, help="1: drop the previous load's handles during the next")
    ap.add_argument("--verify", type=int, default=1)
    ap.add_argument("--streams", type=int, default=2)
    args = ap.parse_args()
    import torch
    import bench
    import paper_2401_14351_b200 as sllm
    from paper_2401_14351_b200 import workloads
    from synth import models
    inv, seed = models.model_inventory(args.config)
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20, args.config, partitions=[0], gpu_of={0: 0})
    blob = idx.serialize()
    cfg = sllm.LoadConfig(chunk_bytes=args.chunk_mib << 20, mode=args.mode, profile=int(args.profile),
                          verify=bool(args.verify), n_streams=args.streams)
    bases, per = sllm.allocate(idx, {0: 0}, cfg.scatter)
    st = torch.cuda.current_stream()
    rows = []
    import contextlib
    clk = bench.ClockSampler(0) if args.clocks else contextlib.nullcontext()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps + 3)]
    import gc
    prev = None
    if args.gc != 1:
        gc.collect()
        gc.disable() if args.gc == 0 else gc.freeze()
    with clk:
        for r in range(args.steps + 3):
            ev[r][0].record(st)
            t0 = time.perf_counter()
            ix = sllm.Index.from_bytes(blob)
            t1 = time.perf_counter()
            res = sllm.load_start(ix, bufs, {0: 0}, cfg, bases, per, {0: st})
            prev = None
            t2 = time.perf_counter()
            rep = res.wait()
            t3 = time.perf_counter()
            ev[r][1].record(st)
            tv = time.perf_counter()
            if args.overlap_free:   # as bench.py: the previous handles go while the next load runs
                prev = (res, ix)
                tf = tx = time.perf_counter()
            else:
                res.tensors = None
                tf = time.perf_counter()
                res.free()
                tx = time.perf_counter()
                ix.close()
            del res, ix
            t4 = time.perf_counter()
            rows.append({"parse": t1 - t0, "start+views": t2 - t1, "wait": t3 - t2, "free": t4 - t3, "drop_views": tf - tv, "load_free": tx - tf, "index_close": t4 - tx, "host_total": t4 - t0,
                         "device": rep["t_device_ms_max"] * 1e-3, "issue": rep["t_issue_ns_max"] * 1e-9,
                         "lib_total": rep["t_total_ns"] * 1e-9})
    torch.cuda.synchronize()
    for r in range(len(rows)):
        rows[r]["event_step"] = ev[r][0].elapsed_time(ev[r][1]) * 1e-3
        if r + 1 < len(rows):
            rows[r]["event_gap_to_next"] = ev[r][1].elapsed_time(ev[r + 1][0]) * 1e-3
    rows = rows[3:]
    med = {k: statistics.median(r[k] for r in rows if k in r) * 1e3 for k in rows[0]}
    span = ev[3][0].elapsed_time(ev[-1][1]) / (len(ev) - 3)
    L = idx.partitions[0].length
    steps = [round(r["event_step"] * 1e3, 2) for r in rows]
    print(json.dumps({"gc": args.gc, "event_step_ms": steps, "config": args.config, "mode": args.mode, "profile": args.profile, "clocks": args.clocks,
                      "bytes": L, "ms_per_step_events": span, "GBps_events": L / (span * 1e-3) / 1e9,
                      "median_ms": med}))


if __name__ == "__main__":
    main()
