"""Converter benchmark (north star: "Converter: a host-side writer that packs tensors into
aligned per-GPU partitions and emits the index"; SPEC S:43 convert).

Source tensors of a config sit in ordinary host memory (one NumPy array each, filled with
the seeded payload, untimed).  Timed, per thread count:
  - convert_into: plan + copy every tensor into pinned partition buffers + zero padding +
    per-block Fletcher-64 (the in-memory sink the loader benchmarks use);
  - seal: the block-checksum pass alone over the filled partitions;
  - convert to files (SLLM): part_<d>.bin + index.bin on local disk (page cache, fsync'd);
Roofline: host memory bandwidth, measured here as a multi-threaded NumPy copy of the same
bytes.  The oracle converter (oracle/layout.py, 1 core) is timed on a bounded sample.

    python tools/bench_convert.py [--config opt-6.7b] [--dir /tmp/sllm_conv]
"""
import argparse
import ctypes
import json
import os
import shutil
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def par_copy(dst, src, threads):
    n = src.nbytes
    step = -(-n // threads)

    def work(i):  # ctypes calls release the GIL: a real multi-threaded memcpy
        lo, hi = i * step, min(n, (i + 1) * step)
        if hi > lo:
            ctypes.memmove(dst.ctypes.data + lo, src.ctypes.data + lo, hi - lo)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="opt-6.7b")
    ap.add_argument("--dir", default="/tmp/sllm_conv")
    ap.add_argument("--oracle-gib", type=float, default=1.0)
    args = ap.parse_args()
    import numpy as np
    import paper_2401_14351_b200 as sllm
    from synth import models, payload
    from oracle import layout as olayout

    inv, seed = models.model_inventory(args.config)
    t0 = time.perf_counter()
    srcs = [np.empty(t.nbytes, np.uint8) for t in inv]
    payload.payload_into([a.ctypes.data for a in srcs], [t.nbytes for t in inv], seed, list(range(len(inv))))
    tensors = [(t.name, t.device, t.dtype, t.shape, a.ctypes.data) for t, a in zip(inv, srcs)]
    total = sum(t.nbytes for t in inv)
    print(json.dumps({"config": args.config, "tensors": len(inv), "payload_bytes": total,
                      "setup_s": time.perf_counter() - t0, "cores": len(os.sched_getaffinity(0))}), flush=True)
    idx0 = sllm.Index.plan([(t.name, t.device, t.dtype, t.shape) for t in inv], 4096, 1 << 20, args.config)
    bufs = [sllm.HostBuffer(p.length) for p in idx0.partitions]
    # host DRAM roofline: the same bytes copied by NumPy on all cores (read + write)
    big = np.ones(min(total, 4 << 30), np.uint8)
    dst = np.zeros_like(big)
    best = 0
    for _ in range(3):
        t0 = time.perf_counter()
        par_copy(dst, big, len(os.sched_getaffinity(0)))
        best = max(best, big.nbytes / (time.perf_counter() - t0) / 1e9)
    del big, dst
    print(json.dumps({"host_copy_GBps": best, "threads": len(os.sched_getaffinity(0))}), flush=True)
    for rep in range(2):
        t0 = time.perf_counter()
        idx = sllm.Index.plan([(t.name, t.device, t.dtype, t.shape) for t in inv], 4096, 1 << 20, args.config)
        idx.convert_into(tensors, [b.ptr for b in bufs])
        dt = time.perf_counter() - t0
        t1 = time.perf_counter()
        idx.seal([b.ptr for b in bufs])
        ds = time.perf_counter() - t1
        print(json.dumps({"rep": rep, "convert_into_s": dt, "convert_into_GBps": total / dt / 1e9,
                          "seal_s": ds, "seal_GBps": sum(b.nbytes for b in bufs) / ds / 1e9}), flush=True)
    assert idx.serialize() == idx.serialize()
    shutil.rmtree(args.dir, ignore_errors=True)
    t0 = time.perf_counter()
    sllm.convert(tensors, args.dir, 4096, 1 << 20, args.config)
    os.sync()
    dt = time.perf_counter() - t0
    print(json.dumps({"convert_files_s": dt, "convert_files_GBps": total / dt / 1e9}), flush=True)
    shutil.rmtree(args.dir, ignore_errors=True)
    # the oracle converter, 1 core, on the source-order prefix of about --oracle-gib
    budget, keep = int(args.oracle_gib * (1 << 30)), []
    acc = 0
    for t, a in zip(inv, srcs):
        if acc + t.nbytes > budget:
            break
        keep.append((t.name, t.device, t.dtype, t.shape, a))
        acc += t.nbytes
    t0 = time.perf_counter()
    olayout.convert(keep, 4096, 1 << 20, args.config)
    dt = time.perf_counter() - t0
    print(json.dumps({"oracle_convert_sample_bytes": acc, "oracle_convert_s": dt, "oracle_GBps": acc / dt / 1e9,
                      "cores": 1}), flush=True)


if __name__ == "__main__":
    main()
