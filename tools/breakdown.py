"""The paper's loader breakdown (figure)
replayed on this box: one OPT-6.7B-shaped partition file -> one B200, each stage adding
one technique, caches dropped before every run.

  read_by_tensor : buffered read of every tensor, each copied to the GPU (pageable)
  bulk           : 16 MiB chunks, buffered reads, pageable H2D per chunk
  direct_io      : 1 thread, O_DIRECT (sllm_host_read_partition) into pageable memory, then H2D
  multi_thread   : as direct_io with 4 reader threads
  pinned         : 4 O_DIRECT readers into pinned memory, then one DMA H2D
  pipeline       : sllm load_files -- readers, pinned slot ring and GPU copies overlapped,
                   every block verified on the GPU

    python tools/breakdown.py [--config opt-6.7b] [--dir /tmp/sllm_breakdown]
"""
import argparse
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def drop_cache(path):
    fd = os.open(path, os.O_RDONLY)
    os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
    os.close(fd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="opt-6.7b")
    ap.add_argument("--dir", default="/tmp/sllm_breakdown")
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2401_14351_b200 as sllm
    from paper_2401_14351_b200 import workloads
    from synth import models

    inv, seed = models.model_inventory(args.config)
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20, args.config, partitions=[0], gpu_of={0: 0})
    os.makedirs(args.dir, exist_ok=True)
    part = os.path.join(args.dir, f"part_{idx.partitions[0].device}.bin")
    with open(part, "wb") as f:
        f.write(memoryview(bufs[0].numpy()))
    with open(os.path.join(args.dir, "index.bin"), "wb") as f:
        f.write(idx.serialize())
    os.sync()
    L = idx.partitions[0].length
    payload_b = idx.info()["payload_bytes"]
    dev = torch.empty(L, dtype=torch.uint8, device="cuda")
    raw = np.empty(L + 4096, np.uint8)
    off = (-raw.ctypes.data) % 4096
    pageable = raw[off:off + L]  # 4 KiB-aligned pageable buffer (O_DIRECT-capable)
    out = {"config": args.config, "bytes": L, "cpu": os.cpu_count()}

    def timed(name, fn):
        drop_cache(part)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out[name] = {"s": dt, "GBps": payload_b / dt / 1e9}
        print(json.dumps({name: out[name]}), flush=True)

    def read_by_tensor():
        with open(part, "rb", buffering=0) as f:
            for t in idx.tensors:
                f.seek(t.offset)
                b = f.read(t.nbytes)
                dev[t.offset:t.offset + t.nbytes].copy_(torch.frombuffer(bytearray(b), dtype=torch.uint8))

    def bulk():
        C = 16 << 20
        with open(part, "rb", buffering=0) as f:
            for lo in range(0, L, C):
                n = f.readinto(memoryview(pageable[lo:lo + C]))
                dev[lo:lo + n].copy_(torch.from_numpy(pageable[lo:lo + n]))

    def direct(threads):
        def fn():
            sllm._abi.check(sllm.lib().sllm_host_read_partition(args.dir.encode(), idx.handle, 0,
                                                                ctypes.c_void_p(pageable.ctypes.data), threads))
            dev.copy_(torch.from_numpy(pageable))
        return fn

    def pinned():
        sllm._abi.check(sllm.lib().sllm_host_read_partition(args.dir.encode(), idx.handle, 0,
                                                            ctypes.c_void_p(bufs[0].ptr), 4))
        dev.copy_(bufs[0].torch(), non_blocking=True)

    def pipeline():
        ix = sllm.Index.open(os.path.join(args.dir, "index.bin"))
        sllm.load_files(ix, args.dir, {0: 0}, sllm.LoadConfig(chunk_bytes=64 << 20), io_threads=4,
                        bases={0: dev}, per_tensor={})

    timed("read_by_tensor", read_by_tensor)
    timed("bulk", bulk)
    timed("direct_io", direct(1))
    timed("multi_thread", direct(4))
    timed("pinned", pinned)
    timed("pipeline", pipeline)
    assert torch.equal(dev[:1 << 20].cpu(), bufs[0].torch()[:1 << 20])
    print(json.dumps(out), flush=True)
    os.remove(part)


if __name__ == "__main__":
    main()
