"""Probe: a same-process P2P fan-out group (R replicas on one GPU) over growing
checkpoints and chunk sizes; prints one JSON line per case (ok / error, seconds)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_14351_b200 as sllm  # noqa: E402
from paper_2401_14351_b200 import workloads  # noqa: E402
from synth import models  # noqa: E402

cases = [("toy", None, 1 << 20), ("mid", models.llama2(1024, 12, 4096, 1024, vocab=32000), 1 << 20),
         ("mid", models.llama2(1024, 12, 4096, 1024, vocab=32000), 64 << 20), ("opt-6.7b", None, 64 << 20)]
for name, inv, chunk in cases:
    if inv is None:
        inv, seed = models.model_inventory(name)
    else:
        seed = 9
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    L = idx.partitions[0].length
    for mode in ("ce", "zerocopy"):
        for R in (2,):
            bases = [torch.empty(L, dtype=torch.uint8, device="cuda") for _ in range(R)]
            sigs = [torch.zeros(2 * R, dtype=torch.int32, device="cuda") for _ in range(R)]
            comms = [sllm.Comm.peers(R, r, 0, [b.data_ptr() for b in bases], [s.data_ptr() for s in sigs], 15000)
                     for r in range(R)]
            cfg = sllm.LoadConfig(chunk_bytes=chunk, mode=mode, fanout="p2p")
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = {"model": name, "L": L, "chunk_mib": chunk >> 20, "mode": mode, "R": R}
            try:
                results = [sllm.load_start(idx, bufs, {0: 0}, cfg, {0: bases[r]}, None, None, comms[r]) for r in range(R)]
                errs = []
                for res in results:
                    try:
                        res.wait()
                    except sllm.SllmError as ex:
                        errs.append(str(ex))
                out["s"] = time.perf_counter() - t0
                out["errors"] = errs
                out["ok"] = not errs and all(np.array_equal(r.block_checksums(0), idx.block_checksums(0)) for r in results)
                del results
            except Exception as ex:  # noqa: BLE001
                out["exception"] = repr(ex)
            print(json.dumps(out), flush=True)
            for c in comms:
                c.free()
            del bases, sigs
            torch.cuda.empty_cache()
    for b in bufs.values():
        b.free()
