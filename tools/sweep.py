"""Load-configuration sweep on one GPU (BASELINE configs[1]: OPT-6.7B chunk-size sweep).

    python tools/sweep.py [--config opt-6.7b] [--reps 3] [--quick] > gpurun_out/sweep.jsonl

Builds the pinned checkpoint once, measures the H2D copy-engine peak on the same buffer,
then times full loads (verify on) over mode x chunk x streams x CTAs with CUDA events on
the caller stream.  One JSON line per configuration.
"""
import argparse
import itertools
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="opt-6.7b")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--modes", default="ce,zerocopy,scatter_ce,scatter_zc")
    ap.add_argument("--chunks", default="1,2,4,8,16,32,64")
    ap.add_argument("--streams", default="1,2")
    ap.add_argument("--ctas", default="0")
    ap.add_argument("--engines", default="tma")
    args = ap.parse_args()
    import torch
    import paper_2401_14351_b200 as sllm
    from paper_2401_14351_b200 import workloads
    from synth import models, payload
    payload.build_csynth()
    t0 = time.time()
    inv, seed = models.model_inventory(args.config)
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20, args.config, partitions=[0], gpu_of={0: 0})
    L = idx.partitions[0].length
    payload_b = sum(t.nbytes for t in idx.tensors if t.partition == 0)
    print(json.dumps({"setup_s": time.time() - t0, "L": L, "payload": payload_b}), flush=True)
    base = torch.empty(L, dtype=torch.uint8, device="cuda")
    src = bufs[0].torch()
    st = torch.cuda.current_stream()
    for n in sorted({min(1 << 30, L), min(4 << 30, L), L}):  # (sizes clamped to the buffer: bytes counted = bytes copied)
        best = 0
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            base[:n].copy_(src[:n], non_blocking=True)
            b.record()
            b.synchronize()
            best = max(best, n / a.elapsed_time(b) / 1e6)
        print(json.dumps({"h2d_peak_bytes": n, "GBps": best}), flush=True)
    _, per = sllm.allocate(idx, {0: 0}, scatter=True)
    for mode, chunk, S, ctas, eng in itertools.product(args.modes.split(","), [int(c) for c in args.chunks.split(",")],
                                                       [int(s) for s in args.streams.split(",")],
                                                       [int(c) for c in args.ctas.split(",")], args.engines.split(",")):
        cfg = sllm.LoadConfig(chunk_bytes=chunk << 20, n_streams=S, mode=mode, ctas=ctas, engine=eng)
        times, rep = [], None
        try:
            for r in range(args.reps + 1):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                res = sllm.load_start(idx, bufs, {0: 0}, cfg, {0: base}, per, {0: st})
                rep = res.wait()
                b.record(st)
                b.synchronize()
                if r:
                    times.append(a.elapsed_time(b))
                del res
        except Exception as ex:  # noqa: BLE001
            print(json.dumps({"mode": mode, "chunk_mib": chunk, "streams": S, "ctas": ctas, "engine": eng,
                              "error": str(ex)}), flush=True)
            continue
        times.sort()
        print(json.dumps({"mode": mode, "chunk_mib": chunk, "streams": S, "ctas": ctas, "engine": eng,
                          "best_ms": times[0], "median_ms": times[len(times) // 2],
                          "GBps_best": payload_b / times[0] / 1e6, "GBps_median": payload_b / times[len(times) // 2] / 1e6,
                          "lib_device_ms": rep["t_device_ms_max"], "issue_ms": rep["t_issue_ns_max"] / 1e6,
                          "total_ms": rep["t_total_ns"] / 1e6}), flush=True)


if __name__ == "__main__":
    main()
