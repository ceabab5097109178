"""File-tier benchmark: load a partition from its file through the
whole multi-tier pipeline (O_DIRECT readers -> pinned slot ring -> GPU, verification on),
and compare with the storage roofline measured on the same file (multi-threaded O_DIRECT
read into pinned memory, the analogue of the paper's FIO baseline).

    python tools/bench_files.py [--config opt-6.7b] [--io-threads 4] [--dir /tmp/sllm_ckpt]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def drop_cache(path):
    fd = os.open(path, os.O_RDONLY)
    try:
        os.fsync(fd)
    except OSError:
        pass
    os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
    os.close(fd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="opt-6.7b")
    ap.add_argument("--io-threads", default="1,2,4,8")
    ap.add_argument("--dir", default="/tmp/sllm_bench_ckpt")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--mode", default="ce")
    args = ap.parse_args()
    import torch
    import paper_2401_14351_b200 as sllm
    from paper_2401_14351_b200 import workloads
    from synth import models

    inv, seed = models.model_inventory(args.config)
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20, args.config, partitions=[0], gpu_of={0: 0})
    os.makedirs(args.dir, exist_ok=True)
    part = os.path.join(args.dir, f"part_{idx.partitions[0].device}.bin")
    t0 = time.perf_counter()
    with open(part, "wb") as f:
        f.write(memoryview(bufs[0].numpy()))
    with open(os.path.join(args.dir, "index.bin"), "wb") as f:
        f.write(idx.serialize())
    os.sync()
    print(json.dumps({"write_s": time.perf_counter() - t0, "bytes": idx.partitions[0].length}), flush=True)
    L = idx.partitions[0].length
    payload_b = idx.info()["payload_bytes"]
    import ctypes
    for th in [int(x) for x in args.io_threads.split(",")]:
        # storage roofline: O_DIRECT multi-threaded read of the same file into pinned memory
        best = 0
        for _ in range(args.reps):
            drop_cache(part)
            t0 = time.perf_counter()
            sllm._abi.check(sllm.lib().sllm_host_read_partition(args.dir.encode(), idx.handle, 0,
                                                                ctypes.c_void_p(bufs[0].ptr), th))
            best = max(best, L / (time.perf_counter() - t0) / 1e9)
        # the pipeline: open the index from storage, read + transfer + verify every window
        bases, per = sllm.allocate(idx, {0: 0}, args.mode.startswith("scatter"))
        bestp, rep = 0, None
        for _ in range(args.reps):
            drop_cache(part)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ix = sllm.Index.open(os.path.join(args.dir, "index.bin"))
            res = sllm.load_files(ix, args.dir, {0: 0}, sllm.LoadConfig(chunk_bytes=64 << 20, mode=args.mode),
                                  io_threads=th, bases=bases, per_tensor=per)
            dt = time.perf_counter() - t0
            rep = res.report
            bestp = max(bestp, payload_b / dt / 1e9)
            del res, ix
        print(json.dumps({"config": args.config, "io_threads": th, "mode": args.mode,
                          "storage_odirect_GBps": best, "pipeline_GBps": bestp,
                          "frac_of_storage": bestp / best, "chunks": rep["chunks"]}), flush=True)
        del bases, per
        torch.cuda.empty_cache()
    os.remove(part)


if __name__ == "__main__":
    main()
