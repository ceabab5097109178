"""Per-launch device timeline of one load (SLLM_PROFILE_DUMP): every copy submission and
kernel launch with its start (ms after the load's first event) and duration.

    SLLM_PROFILE_DUMP=1 python tools/timeline.py [--config lora-70b-r32] [--chunk-mib 64] [--streams 2]

With SLLM_KTIME=1 every kernel line also carries the in-kernel span (first CTA start to last
CTA end, %globaltimer) and the CTA start / end spreads, next to the CUDA-event duration.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="lora-70b-r32")
    ap.add_argument("--mode", default="ce")
    ap.add_argument("--chunk-mib", type=int, default=64)
    ap.add_argument("--streams", type=int, default=2)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--profile", type=int, default=2, help="1: kernel launches timed, 2: copies too")
    args = ap.parse_args()
    import torch
    import paper_2401_14351_b200 as sllm
    from paper_2401_14351_b200 import workloads
    from synth import models
    inv, seed = models.model_inventory(args.config)
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20, args.config, partitions=[0], gpu_of={0: 0})
    cfg = sllm.LoadConfig(chunk_bytes=args.chunk_mib << 20, n_streams=args.streams, mode=args.mode, profile=args.profile)
    bases, per = sllm.allocate(idx, {0: 0}, cfg.scatter)
    for r in range(args.reps):
        print(f"--- load {r}", file=sys.stderr, flush=True)
        res = sllm.load_start(idx, bufs, {0: 0}, cfg, bases, per, {0: torch.cuda.current_stream()})
        rep = res.wait()
        print(f"device_ms={rep['t_device_ms_max']:.4f} issue_us={rep['t_issue_ns_max'] / 1e3:.1f}", file=sys.stderr,
              flush=True)
        del res


if __name__ == "__main__":
    main()
