"""Soak test: many back-to-back loads through the public API (allocation + load + verify +
free each time, rotating modes), watching device free memory and host RSS for leaks.

    python tools/soak.py [--config opt-6.7b] [--loads 100]
    python tools/soak.py --config lora-70b-r32 --loads 300 --p2p 2   # in-process P2P group
    python tools/soak.py --config lora-70b-r32 --loads 500 --capture # captured load, replays

Prints one JSON line: loads, failures, seconds, device free memory and RSS before / after
(after the library's idle cache is trimmed), and the GB/s range."""
import argparse
import json
import os
import resource
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rss_gb():
    with open("/proc/self/statm") as f:
        return int(f.read().split()[1]) * os.sysconf("SC_PAGE_SIZE") / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="opt-6.7b")
    ap.add_argument("--loads", type=int, default=100)
    ap.add_argument("--p2p", type=int, default=0, help="R > 1: an in-process P2P group of R replicas on GPU 0 "
                    "(event-ordered), every load verified on every replica")
    ap.add_argument("--capture", action="store_true", help="one captured load, --loads replays (rotating modes "
                    "= one capture per mode)")
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2401_14351_b200 as sllm
    from paper_2401_14351_b200 import workloads
    from synth import models

    inv, seed = models.model_inventory(args.config)
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20, args.config, partitions=[0], gpu_of={0: 0})
    table = idx.block_checksums(0)
    if args.p2p > 1:
        return soak_p2p(args, sllm, torch, np, idx, bufs, table)
    if args.capture:
        return soak_capture(args, sllm, torch, np, idx, bufs, table)
    modes = ["ce", "zerocopy", "scatter_ce", "scatter_zc", "auto"]
    # warm once per mode (pools, module load), then measure the baseline
    for m in modes:
        sllm.load(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=64 << 20, mode=m)).free()
    torch.cuda.synchronize()
    sllm.trim_device_cache(0)
    torch.cuda.empty_cache()
    free0, rss0 = torch.cuda.mem_get_info(0)[0], rss_gb()
    rates, failures, by_mode = [], 0, {m: [] for m in modes}
    t0 = time.perf_counter()
    for i in range(args.loads):
        m = modes[i % len(modes)]
        ts = time.perf_counter()
        res = sllm.load(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=64 << 20, mode=m))
        rates.append(idx.partitions[0].length / (time.perf_counter() - ts) / 1e9)
        by_mode[m].append(rates[-1])
        if not np.array_equal(res.block_checksums(0), table):
            failures += 1
        res.free()
        del res
    dt = time.perf_counter() - t0
    torch.cuda.synchronize()
    sllm.trim_device_cache(0)
    torch.cuda.empty_cache()
    free1, rss1 = torch.cuda.mem_get_info(0)[0], rss_gb()
    print(json.dumps({"config": args.config, "loads": args.loads, "failures": failures, "seconds": dt,
                      "GBps_min": min(rates), "GBps_median": float(np.median(rates)), "GBps_max": max(rates),
                      "device_free_GB_before": free0 / 1e9, "device_free_GB_after": free1 / 1e9,
                      "device_leak_GB": (free0 - free1) / 1e9, "rss_GB_before": rss0, "rss_GB_after": rss1,
                      "maxrss_GB": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6,
                      "per_mode_GBps": {m: {"min": min(v), "median": float(np.median(v)), "slowest_load": int(np.argmin(v))}
                                        for m, v in by_mode.items() if v}}), flush=True)


def soak_capture(args, sllm, torch, np, idx, bufs, table):
    """Captured loads: one capture per mode, then --loads replays rotating over them; every
    replay's block checksums must equal the index table; device / host memory watched."""
    modes = ["ce", "zerocopy", "scatter_ce", "scatter_zc"]
    caps = []
    for m in modes:
        cfg = sllm.LoadConfig(chunk_bytes=64 << 20, mode=m)
        bases, per = sllm.allocate(idx, {0: 0}, cfg.scatter)
        caps.append(sllm.load_capture(idx, bufs, {0: 0}, cfg, bases, per))
        caps[-1].replay().wait()  # warm
    torch.cuda.synchronize()
    free0, rss0 = torch.cuda.mem_get_info(0)[0], rss_gb()
    rates, failures = [], 0
    t0 = time.perf_counter()
    for i in range(args.loads):
        c = caps[i % len(caps)]
        ts = time.perf_counter()
        c.replay().wait()
        rates.append(idx.partitions[0].length / (time.perf_counter() - ts) / 1e9)
        failures += not np.array_equal(c.block_checksums(0), table)
    dt = time.perf_counter() - t0
    torch.cuda.synchronize()
    free1, rss1 = torch.cuda.mem_get_info(0)[0], rss_gb()
    for c in caps:
        c.free()
    print(json.dumps({"config": args.config, "captured_modes": modes, "replays": args.loads, "failures": failures,
                      "seconds": dt, "GBps_min": min(rates), "GBps_median": float(np.median(rates)),
                      "device_free_GB_before": free0 / 1e9, "device_free_GB_after": free1 / 1e9,
                      "device_leak_GB": (free0 - free1) / 1e9, "rss_GB_before": rss0, "rss_GB_after": rss1}),
          flush=True)


def soak_p2p(args, sllm, torch, np, idx, bufs, table):
    """Back-to-back loads of one in-process P2P group (R replicas on GPU 0, CUDA-event
    ordering, one epoch per load), rotating CE / zero-copy; every replica's block checksums
    must equal the index table after every load."""
    R, L = args.p2p, idx.partitions[0].length
    bases = [torch.empty(L, dtype=torch.uint8, device="cuda") for _ in range(R)]
    sigs = [torch.zeros(2 * R, dtype=torch.int32, device="cuda") for _ in range(R)]
    comms = [sllm.Comm.peers(R, r, 0, [b.data_ptr() for b in bases], [s.data_ptr() for s in sigs], 60000)
             for r in range(R)]
    modes = ["ce", "zerocopy"]
    for m in modes:  # warm once per mode (worker threads, pools), then measure the baseline
        cfg = sllm.LoadConfig(chunk_bytes=64 << 20, mode=m, fanout="p2p")
        for r in [sllm.load_start(idx, bufs, {0: 0}, cfg, {0: bases[r]}, None, None, comms[r]) for r in range(R)]:
            r.wait()
    torch.cuda.synchronize()
    sllm.trim_device_cache(0)
    torch.cuda.empty_cache()
    free0, rss0 = torch.cuda.mem_get_info(0)[0], rss_gb()
    rates, failures = [], 0
    t0 = time.perf_counter()
    for i in range(args.loads):
        cfg = sllm.LoadConfig(chunk_bytes=64 << 20, mode=modes[i % 2], fanout="p2p")
        ts = time.perf_counter()
        rs = [sllm.load_start(idx, bufs, {0: 0}, cfg, {0: bases[r]}, None, None, comms[r]) for r in range(R)]
        for r in rs:
            r.wait()
        rates.append(R * L / (time.perf_counter() - ts) / 1e9)
        failures += sum(not np.array_equal(r.block_checksums(0), table) for r in rs)
        del rs
    dt = time.perf_counter() - t0
    torch.cuda.synchronize()
    sllm.trim_device_cache(0)
    torch.cuda.empty_cache()
    free1, rss1 = torch.cuda.mem_get_info(0)[0], rss_gb()
    equal = all(torch.equal(bases[0], b) for b in bases[1:])  # (its temporaries come after the reading)
    for c in comms:
        c.free()
    print(json.dumps({"config": args.config, "p2p_ranks": R, "loads": args.loads, "failures": failures,
                      "replicas_equal": equal, "seconds": dt, "GBps_replicas_min": min(rates),
                      "GBps_replicas_median": float(np.median(rates)), "device_free_GB_before": free0 / 1e9,
                      "device_free_GB_after": free1 / 1e9, "device_leak_GB": (free0 - free1) / 1e9,
                      "rss_GB_before": rss0, "rss_GB_after": rss1}), flush=True)


if __name__ == "__main__":
    main()
