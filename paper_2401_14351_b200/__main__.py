"""Command line (SPEC S:533-566 `llmctl convert` / `bench-load`, as one tool):

    python -m paper_2401_14351_b200 convert --out DIR [--align 4096] [--block 1048576] FILE.safetensors...
    python -m paper_2401_14351_b200 synth   --config opt-6.7b --out DIR     # seeded synthetic checkpoint
    python -m paper_2401_14351_b200 info    DIR                             # index summary
    python -m paper_2401_14351_b200 load    DIR [--gpu 0] [--mode ce] [--chunk-mib 64] [--io-threads 4]

`load` runs the whole multi-tier path (partition files -> O_DIRECT readers -> pinned slot
ring -> GPU, every block verified) for every partition onto one GPU and prints a JSON
report; it needs a CUDA GPU.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time


def cmd_convert(a):
    from . import formats
    n = formats.convert_safetensors(a.files, a.out, align=a.align, block=a.block, model_id=a.model_id)
    print(json.dumps({"converted_tensors": n, "out": a.out}))


def cmd_synth(a):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from synth import models, payload
    from .api import convert
    inv, seed = models.model_inventory(a.config)
    import numpy as np
    data = [np.empty(t.nbytes, np.uint8) for t in inv]
    payload.payload_into([d.ctypes.data for d in data], [t.nbytes for t in inv], seed, list(range(len(inv))))
    convert([(t.name, t.device, t.dtype, t.shape, d.ctypes.data) for t, d in zip(inv, data)], a.out,
            a.align, a.block, a.config)
    print(json.dumps({"config": a.config, "tensors": len(inv), "bytes": sum(t.nbytes for t in inv), "out": a.out}))


def cmd_info(a):
    from .api import Index
    idx = Index.open(os.path.join(a.dir, "index.bin"))
    info = idx.info()
    parts = [{"device": p.device, "length": p.length, "blocks": p.n_blocks, "tensors": p.n_tensors}
             for p in idx.partitions]
    print(json.dumps({**info, "partitions": parts}, indent=1))


def cmd_load(a):
    import torch
    from .api import Index, LoadConfig, load_files
    idx = Index.open(os.path.join(a.dir, "index.bin"))
    gpus = {p: a.gpu for p in range(len(idx.partitions))}
    cfg = LoadConfig(chunk_bytes=a.chunk_mib << 20, mode=a.mode)
    torch.cuda.synchronize(a.gpu)
    t0 = time.perf_counter()
    res = load_files(idx, a.dir, gpus, cfg, io_threads=a.io_threads)
    torch.cuda.synchronize(a.gpu)
    dt = time.perf_counter() - t0
    rep = res.report
    print(json.dumps({"dir": a.dir, "gpu": a.gpu, "mode": a.mode, "tensors": len(res.tensors),
                      "payload_bytes": rep["payload_bytes"], "seconds": dt, "GBps": rep["payload_bytes"] / dt / 1e9,
                      "verified": rep["bad_partition"] == -1}))


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_2401_14351_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("convert", help="safetensors -> loading-optimized checkpoint")
    c.add_argument("files", nargs="+")
    c.add_argument("--out", required=True)
    c.add_argument("--align", type=int, default=4096)
    c.add_argument("--block", type=int, default=1 << 20)
    c.add_argument("--model-id", default="")
    s = sub.add_parser("synth", help="seeded synthetic checkpoint of a named config")
    s.add_argument("--config", default="toy")
    s.add_argument("--out", required=True)
    s.add_argument("--align", type=int, default=4096)
    s.add_argument("--block", type=int, default=1 << 20)
    i = sub.add_parser("info", help="print the index of a converted checkpoint")
    i.add_argument("dir")
    ld = sub.add_parser("load", help="load a converted checkpoint onto a GPU through the file tier")
    ld.add_argument("dir")
    ld.add_argument("--gpu", type=int, default=0)
    ld.add_argument("--mode", default="ce", choices=["ce", "zerocopy", "scatter_ce", "scatter_zc"])
    ld.add_argument("--chunk-mib", type=int, default=64)
    ld.add_argument("--io-threads", type=int, default=4)
    a = ap.parse_args(argv)
    {"convert": cmd_convert, "synth": cmd_synth, "info": cmd_info, "load": cmd_load}[a.cmd](a)


if __name__ == "__main__":
    main()
