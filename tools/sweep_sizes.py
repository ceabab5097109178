"""Copy engine vs zero-copy kernel by checkpoint size (the SLLM_MODE_AUTO crossover):
single-partition checkpoints of 8 MiB fp16 tensors from 16 MiB to 2 GiB, best-of-N
time-to-loaded (CUDA events on the caller stream, verification on) per mode.

    python tools/sweep_sizes.py [--reps 7] > gpurun_out/sweep_sizes.jsonl
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--sizes-mib", default="16,32,64,128,256,512,1024,2048")
    args = ap.parse_args()
    import torch
    import paper_2401_14351_b200 as sllm
    from paper_2401_14351_b200 import workloads
    from synth import models

    st = torch.cuda.current_stream()
    for mib in [int(x) for x in args.sizes_mib.split(",")]:
        inv = [models.TensorSpec(f"w{i}", 0, "f16", (2048, 2048)) for i in range(mib // 8)]
        idx, bufs = workloads.build_pinned(inv, 11, 4096, 1 << 20)
        L = idx.partitions[0].length
        row = {"size_mib": mib, "bytes": L}
        for mode in ("ce", "zerocopy", "auto"):
            cfg = sllm.LoadConfig(chunk_bytes=min(64 << 20, L), mode=mode)
            bases, per = sllm.allocate(idx, {0: 0})
            best, chosen = 1e9, None
            for r in range(args.reps + 2):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                res = sllm.load_start(idx, bufs, {0: 0}, cfg, bases, per, {0: st})
                rep = res.wait()
                b.record(st)
                b.synchronize()
                if r >= 2:
                    best = min(best, a.elapsed_time(b))
                chosen = rep["mode"]
                del res
            row[mode] = {"ms": best, "GBps": L / best / 1e6, "ran_mode": chosen}
            del bases, per
        print(json.dumps(row), flush=True)
        del idx, bufs


if __name__ == "__main__":
    main()
