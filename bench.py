"""Checkpoint-load benchmark (BASELINE.json metric: "checkpoint load GB/s &
time-to-loaded-model at 1/2/4/8 B200 vs PCIe peak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config opt-6.7b] [--mode zerocopy|ce|scatter_ce|scatter_zc]
                    [--chunk-mib 16] [--streams 2] [--ctas 0] [--no-cpu-baseline]

A "step" is one pass of the whole hot path over the synthetic
checkpoint already sitting in pinned host DRAM: open the index from its bytes (a1), plan
chunks (a3), move every partition byte host->HBM (a4), materialise the tensors (a5),
verify every 1 MiB block's Fletcher-64 on the GPU (a6), complete (a8).  Destinations
are preallocated (a2; T_alloc is reported separately, Q19).  N=1 runs
BASELINE configs[1] (OPT-6.7B-shaped, 13.3 GB fp16, 1 partition).  Under torchrun every
rank loads its own copy of that partition from its own pinned buffer over its own PCIe
link (weak scaling, no collective: SURVEY §8(e)).

value = payload bytes loaded by all ranks / max-over-ranks device time (GB/s, 10^9).
The partition (13.3 GB) is ~100x the 126 MB L2, so no flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "checkpoint load GB/s & time-to-loaded-model at 1/2/4/8 B200 vs PCIe peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="opt-6.7b")
    ap.add_argument("--mode", default="ce", choices=["ce", "zerocopy", "scatter_ce", "scatter_zc"])
    ap.add_argument("--chunk-mib", type=int, default=64)
    ap.add_argument("--streams", type=int, default=2)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--engine", default="tma", choices=["tma", "tma_store", "ldg"],
                    help="kernel engine: TMA ring + vector stores (default), + TMA bulk stores, LDG/STG tiles")
    ap.add_argument("--all-partitions", action="store_true",
                    help="load every partition of a multi-partition config onto this rank's GPU (e.g. the whole "
                         "LLaMA-2-70B TP8 checkpoint on one B200)")
    ap.add_argument("--spread", action="store_true",
                    help="with --all-partitions: partition p on GPU p %% (visible GPUs), all from this one process -- "
                         "the paper's model manager loading every GPU of a server (P:721-727)")
    ap.add_argument("--fanout", default="none", choices=["none", "bcast", "allgather", "p2p"],
                    help="replicated checkpoint: every rank ends with a full replica; rank r reads slice r over "
                         "PCIe and the rest arrives over NVLink (bcast: NCCL broadcasts, allgather: in-place NCCL "
                         "all-gather per round of round-robin chunks, p2p: fused peer stores)")
    ap.add_argument("--cpu-sample-gib", type=float, default=4.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-standalone", action="store_true")
    ap.add_argument("--no-profile", action="store_true", help="no per-launch CUDA events in the timed region")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# SLLM_BENCH_SAME_GPU=1: every rank on cuda:0 with a gloo group -- a plumbing check of the
# multi-rank paths (barriers, max-over-ranks timing, IPC peer groups) on a 1-GPU box; its
# numbers share one PCIe link and are not scaling results.
SAME_GPU = os.environ.get("SLLM_BENCH_SAME_GPU") == "1"


def gpu_of(local):
    return 0 if SAME_GPU else local


def max_over_ranks(x: float, world: int) -> float:
    """Max of a per-rank float over the job (device tensor on NCCL, host tensor on gloo)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    nccl = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=torch.cuda.current_device() if nccl else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,clocks.mem,clocks.max.mem")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for k, n in enumerate(names):
                if len(r) > 4 + k and r[4 + k].lower() == "active":
                    reasons.add(n)
        num = lambda k: [float(r[k]) for r in self.rows if len(r) > k and r[k].replace(".", "").isdigit()]
        mem, mem_max = num(8), num(9)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "mem_mhz": statistics.median(mem) if mem else None, "mem_max_mhz": max(mem_max) if mem_max else None}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic(mode, bytes_per_launch, key="traffic_over_algorithmic"):
    """`traffic` for the roofline: DRAM bytes per launch from the committed `ncu --set full`
    capture of an in-pipeline launch (profiles/<round>/ncu_traffic_<mode>.json, written by
    tools/ncu_traffic.py), scaled from the captured launch's algorithmic bytes to this
    run's average launch.  None when no capture is committed for the mode."""
    import glob
    hits = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", f"ncu_traffic_{mode}.json")))
    if not hits:
        return None, None
    cap = json.load(open(hits[-1]))
    if key not in cap:
        return None, None
    return cap[key] * bytes_per_launch, os.path.relpath(hits[-1], ROOT)


def arm_config(args, world, parts, payload_bytes, raw_bytes, replicated, extra=None):
    """The JSON line's `config` -- identical for our arm and the reference arm."""
    return {"workload": args.config, "mode": args.mode, "fanout": args.fanout, "chunk_mib": args.chunk_mib,
            "engine": args.engine, "streams": args.streams, "ctas": args.ctas, "partitions_per_gpu": parts,
            "payload_bytes_per_gpu": payload_bytes, "raw_bytes_per_gpu": raw_bytes,
            "verify": "fletcher64 per 1 MiB block, every block",
            "l2": f"inputs {raw_bytes / 1e9:.1f} GB per GPU >> 126 MB L2, no flush needed",
            "parallelism": f"replicated x{world} ({args.fanout})" if replicated else f"sharded x{world}",
            **(extra or {})}


def run_reference(args, rank, world):
    """Reference arm = the CPU oracle as it stands (oracle/loader.py) on this box's host
    cores, each step a bounded sample of the same workload."""
    if rank != 0:
        return
    import numpy as np
    from oracle import index as oindex, layout as olayout, loader as oloader
    from synth import models, payload

    inv, seed = models.model_inventory(args.config)
    # per-step sample: --cpu-sample-gib, shrunk so that warmup + steps stay within ~60 GB of
    # oracle work (~2 minutes on one core) whatever K and W the driver passes
    budget = int(min(args.cpu_sample_gib * (1 << 30), max(256 << 20, 60e9 / max(1, args.warmup + args.steps))))
    # oracle converter over the sample's tensors (prefix of partition 0 in source order)
    lay = olayout.plan([(t.name, t.device, t.dtype, t.shape, t.nbytes) for t in inv], 4096, 1 << 20)
    d0 = lay.devices()[0]
    first = min((e for e in lay.entries if e.device == d0), key=lambda e: e.offset)
    budget = max(budget, -(-(first.offset + first.size) // (1 << 20)) << 20)  # at least one whole tensor
    keep = [i for i, e in enumerate(lay.entries) if e.device == d0 and e.offset + e.size <= budget]
    sub = [inv[i] for i in keep]
    tensors = [(t.name, t.device, t.dtype, t.shape, payload.payload_bytes(seed, keep[k], t.nbytes))
               for k, t in enumerate(sub)]
    slay, sparts = olayout.convert(tensors, 4096, 1 << 20, args.config)
    blob = oindex.write(slay)
    times, got = [], 0
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        got = oloader.load_sample(blob, sparts, budget)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    T = sum(times)
    v = got * args.steps / T / 1e9
    n_parts = len(lay.devices())
    sel = list(range(n_parts)) if args.all_partitions else [0]
    devs = [lay.devices()[p] for p in sel]
    ref_config = arm_config(args, world, len(sel), sum(e.size for e in lay.entries if e.device in devs),
                            sum(lay.partitions[d] for d in devs), args.fanout != "none")
    line = {"metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": T / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "impl": "reference",
            "config": ref_config,
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": f"parse index + copy + verify {got} B of {args.config} partition 0"},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(args, bufs, idx, inv, seed):
    """The oracle as it stands, single process (1 core), on a bounded sample of the same
    pinned partition: parse index, copy tensors, recompute and compare checksums."""
    from oracle import loader as oloader
    budget = int(args.cpu_sample_gib * (1 << 30))
    p0 = sorted(bufs)[0]
    first = min((t for t in idx.tensors if t.partition == p0), key=lambda t: t.offset)
    budget = max(budget, -(-(first.offset + first.nbytes) // (1 << 20)) << 20)  # at least one whole tensor
    blob = idx.serialize()
    src = {idx.partitions[p].device: bufs[p].numpy() for p in bufs}
    t0 = time.perf_counter()
    got = oloader.load_sample(blob, src, budget)
    dt = time.perf_counter() - t0
    return {"value": got / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"{got} payload bytes ({args.cpu_sample_gib} GiB budget) of partition 0: parse index, "
                      f"copy every tensor, recompute+compare 1 MiB Fletcher-64 blocks; {dt:.1f} s"}


def h2d_peak(bufs, bases, torch, gib=4, reps=3, world=1, gpus=None):
    """B_h2d(N): the copy engine's best host->device rate from the same pinned buffer into
    the same destination over >= 4 GiB: max of one 4 GiB
    cudaMemcpyAsync and back-to-back 64 MiB cudaMemcpyAsync calls on one stream, best of
    `reps` each.  Under torchrun every rep starts on a barrier so all N links (and the host
    DRAM / PCIe switches they share) are loaded at once; the aggregate is N * bytes / the
    slowest rank's time.  With partitions on several GPUs of this process (--spread) one
    partition per GPU copies at once, aggregate = their bytes / the slowest GPU's time.
    Returns (aggregate GB/s, {method: aggregate GB/s})."""
    firsts = {}
    for p in sorted(bufs):
        firsts.setdefault(gpus[p] if gpus else torch.cuda.current_device(), p)
    sizes = {g: min(gib << 30, bufs[p].nbytes) for g, p in firsts.items()}
    out = {}
    for name, piece in (("single_4GiB", None), ("chunked_64MiB", 64 << 20)):
        best = 0.0
        for _ in range(reps):
            for g in firsts:
                torch.cuda.synchronize(g)
            if world > 1:
                import torch.distributed as dist
                dist.barrier()
            evs = []
            for g, p in firsts.items():
                n = sizes[g]
                src, dst = bufs[p].torch()[:n], bases[p][:n]
                with torch.cuda.device(g):
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    for o in range(0, n, piece or n):
                        dst[o:o + (piece or n)].copy_(src[o:o + (piece or n)], non_blocking=True)
                    e.record()
                evs.append((s, e))
            for s, e in evs:
                e.synchronize()
            ms = max_over_ranks(max(s.elapsed_time(e) for s, e in evs), world)
            best = max(best, world * sum(sizes.values()) / (ms * 1e-3) / 1e9)
        out[name] = best
    return max(out.values()), out


def standalone_hbm(idx, bufs, torch, sllm, reps=5):
    """K4 (checksum) and K3 (scatter + checksum) on the device-resident partition image
    (the real partition bytes, copied to HBM once; >= 1 GiB), HBM roofline.
    K4: CUDA events around the call on the launching stream (the call is asynchronous).
    K3: CUDA events the library records around the launch itself (the call also uploads
    the segment and checksum tables and reads the result word, which are not the kernel).
    Best of `reps`."""
    p = sorted(bufs)[0]
    L = idx.partitions[p].length
    n = min(L, 4 << 30) // (1 << 20) * (1 << 20)
    if 2 * L + (1 << 30) > torch.cuda.mem_get_info()[0]:  # image + per-tensor buffers must fit
        return None
    src = torch.empty(L, dtype=torch.uint8, device="cuda")
    src.copy_(bufs[p].torch())
    out = torch.empty(-(-n // (1 << 20)), dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    res = {}
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sllm.block_checksums_device(src.data_ptr(), n, 1 << 20, out.data_ptr(), 0, st)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    t = min(ts) * 1e-3
    table = idx.block_checksums(p)[:out.numel()]
    res["k4"] = {"bytes": n, "ms": t * 1e3, "GBps": n / t / 1e9,
                 "checksums_equal_index": bool((out.cpu().numpy().view("uint64") == table).all())}
    # K3: scatter the whole partition image into per-tensor buffers (read L + write payload)
    _, per = sllm.allocate(idx, {p: 0}, scatter=True, partitions=[p])
    ts = [sllm.materialise_device(idx, p, src.data_ptr(), per, 0, st, timed=True) for _ in range(reps)]
    t = min(ts) * 1e-3
    payload = sum(x.nbytes for x in idx.tensors if x.partition == p)
    res["k3"] = {"bytes": L + payload, "ms": t * 1e3, "GBps": (L + payload) / t / 1e9, "status_ok": True,
                 "timing": "library CUDA events around the K3 launch"}
    del per, src, out
    torch.cuda.empty_cache()
    return res


def main():
    args = parse()
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        import torch
        torch.cuda.set_device(gpu_of(local))
        if SAME_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return

    import torch
    import paper_2401_14351_b200 as sllm
    from paper_2401_14351_b200 import workloads
    from synth import models, payload

    payload.build_csynth()
    gpu = gpu_of(local)
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)

    # ---- setup (untimed): synthetic checkpoint packed into pinned DRAM by the converter
    t0 = time.perf_counter()
    inv, seed = models.model_inventory(args.config)
    replicated = args.fanout != "none"
    if replicated and len(set(t.device for t in inv)) != 1:
        raise SystemExit("--fanout needs a single-partition (replicated) checkpoint config")
    n_parts = len(set(t.device for t in inv))
    if args.all_partitions:
        sel = list(range(n_parts))
    else:
        sel = [0] if world == 1 or n_parts == 1 else [rank]
    if args.spread and (not args.all_partitions or world > 1 or replicated):
        raise SystemExit("--spread goes with --all-partitions in a single process (no fan-out)")
    ndev = torch.cuda.device_count() if args.spread else 1
    gpu_map = {p: (p % ndev if args.spread else gpu) for p in sel}
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20, args.config, partitions=sel, gpu_of=gpu_map)
    t_setup = time.perf_counter() - t0
    blob = idx.serialize()
    parts = sorted(bufs)
    gpus = {p: gpu_map[p] for p in parts}
    used = sorted(set(gpus.values()))

    def sync_all():
        for g in used:
            torch.cuda.synchronize(g)
    cfg = sllm.LoadConfig(chunk_bytes=args.chunk_mib << 20, n_streams=args.streams, mode=args.mode,
                          ctas=args.ctas, profile=True, fanout=args.fanout, engine=args.engine)
    # a2: destination allocation (reported separately, Q19)
    torch.cuda.synchronize()
    ta = time.perf_counter()
    bases, per_tensor = sllm.allocate(idx, gpus, cfg.scatter, partitions=parts)
    torch.cuda.synchronize()
    t_alloc = time.perf_counter() - ta
    payload_bytes = sum(t.nbytes for t in idx.tensors if t.partition in bufs)
    raw_bytes = sum(idx.partitions[p].length for p in parts)

    b_h2d, b_h2d_methods = h2d_peak(bufs, bases if not cfg.scatter else {p: torch.empty(min(4 << 30, idx.partitions[p].length),
                                                                          dtype=torch.uint8, device=f"cuda:{gpus[p]}") for p in parts},
                     torch, world=world, gpus=gpus)
    stream = torch.cuda.current_stream(gpu)
    streams = {p: torch.cuda.current_stream(gpus[p]) for p in parts}
    comm = None
    if args.fanout == "p2p":      # peer group bound to every rank's replica (CUDA IPC over the process group)
        if world > 1:
            comm = sllm.Comm.peers_from_process_group(bases[0])
        else:
            sig = torch.zeros(2, dtype=torch.int32, device=dev)
            comm = sllm.Comm.peers(1, 0, gpu, [bases[0].data_ptr()], [sig.data_ptr()], keep=[sig])
    elif args.fanout in ("bcast", "allgather"):  # NCCL communicator over the process group
        comm = sllm.Comm.from_process_group(gpu) if world > 1 else sllm.Comm.init_rank(sllm.Comm.unique_id(), 1, 0, gpu)

    def step(prof: bool):
        c = sllm.LoadConfig(**{**cfg.__dict__, "profile": prof})
        ix = sllm.Index.from_bytes(blob)                  # a1: open + validate the index
        res = sllm.load_start(ix, bufs, gpus, c, bases, per_tensor, streams, comm)
        return res, ix

    for _ in range(args.warmup):
        res, ix = step(False)
        res.wait()
        del res, ix
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    sync_all()
    reports = []
    with ClockSampler(gpu) as clk:
        # one start/end pair per GPU this process loads (its caller stream is gated on the
        # load); the step time is the slowest GPU's
        marks = {g: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for g in used}
        for g in used:
            marks[g][0].record(torch.cuda.current_stream(g))
        for _ in range(args.steps):
            res, ix = step(not args.no_profile)
            reports.append(res.wait())
            del res, ix
        for g in used:
            marks[g][1].record(torch.cuda.current_stream(g))
        sync_all()
    if world > 1:
        dist.barrier()
    ms_total = max_over_ranks(max(a.elapsed_time(b) for a, b in marks.values()), world)
    ms_step = ms_total / args.steps
    # every rank ends the step with its own loaded model (sharded: its partition; replicated:
    # a full replica, of which it moved 1/N over PCIe)
    value = payload_bytes * world / (ms_step * 1e-3) / 1e9
    pcie_bytes = raw_bytes if not replicated else sum(r["transferred_bytes"] for r in reports) / len(reports)

    # ---- end-to-end through the public API (a2 allocation + index open + load + wait +
    #      D2H of the verification word), host wall clock, pinned sources
    if comm is None:  # e2e allocates its own destinations: give the timed loop's back first
        bases = per_tensor = None
        torch.cuda.empty_cache()
    e2e_t = []
    for _ in range(2):
        sync_all()
        t0 = time.perf_counter()
        ix = sllm.Index.from_bytes(blob)
        if comm is None:
            res = sllm.load(ix, bufs, gpus, sllm.LoadConfig(**{**cfg.__dict__, "profile": False}))
        else:  # a replicated group is bound to its replicas: no per-step allocation
            res = sllm.load_start(ix, bufs, gpus, sllm.LoadConfig(**{**cfg.__dict__, "profile": False}), bases,
                                  per_tensor, {p: stream for p in parts}, comm)
            res.wait()
        sync_all()
        e2e_t.append(time.perf_counter() - t0)
        del res, ix
    t_e2e = max_over_ranks(min(e2e_t), world)  # the job's end-to-end time is its slowest rank's
    e2e = {"value": payload_bytes * world / t_e2e / 1e9, "unit": "GB/s",
           "h2d_bytes_per_step": int(pcie_bytes) + sum(idx.partitions[p].n_blocks * 8 for p in parts),
           "d2h_bytes_per_step": 8 * len(parts),
           "includes": ("index open + load + verify + wait (replicas preallocated: the peer group is bound to them)"
                        if comm is not None else "torch allocation + index open + load + verify + wait"),
           "time_to_loaded_model_s": t_e2e}

    # ---- roofline of the dominant kernel, from the library's per-launch CUDA events
    rep = reports[-1]
    kern_ms = sum(r["t_kernel_ms_sum"] for r in reports) / len(reports)
    kern_launches = rep["kernel_launches"]
    kern_bytes = rep["kernel_bytes"]
    roof = None
    pcie_rate = pcie_bytes * world / (ms_step * 1e-3) / 1e9
    h2d = {"bound": "pcie", "achieved": pcie_rate, "peak": b_h2d, "unit": "GB/s",
           "frac": pcie_rate / b_h2d, "peak_methods": b_h2d_methods, "n_links": world,
           "what": "host->device bytes of the whole step (a1-a8) over its device time vs the copy engine's "
                   "measured host->device peak on the same buffers (all links at once under torchrun)"}
    if args.mode in ("ce", "scatter_ce") and kern_launches and kern_ms > 0:
        # the step's kernel: K4 (CE) / K3 (SCATTER_CE) on each landed chunk, per-launch
        # CUDA events recorded by the library on its kernel stream over the timed region
        per_launch_bytes = kern_bytes / kern_launches * (2 if args.mode == "scatter_ce" else 1)
        avg_ms = kern_ms / kern_launches
        achieved = per_launch_bytes / (avg_ms * 1e-3) / 1e9
        hbm = peaks().get("hbm_gbs", 6551.4)
        traffic, traffic_src = ncu_traffic(args.mode, per_launch_bytes)
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "traffic_source": traffic_src,
                "kernel": "materialise_tma_kernel<%s> (in pipeline)" %
                ("checksum only" if args.mode == "ce" else "scatter+checksum"),
                "launches_per_step": kern_launches, "avg_launch_ms": avg_ms,
                "bytes_per_launch": per_launch_bytes,
                "note": "one CTA per SM; each launch verifies a span of landed windows (up to 2 GiB, halving towards the end) "
                        "(1 MiB blocks split into equal units for wave balance) beside the PCIe copies"}
    if args.mode in ("zerocopy", "scatter_zc") and kern_launches and kern_ms > 0:
        # zero-copy kernel: every byte it reads crosses PCIe -> bound by the host link.
        # Launches on the S streams overlap, so the kernel's rate is its bytes per step
        # over the step's device time (the kernel is the only work in the step).
        achieved = kern_bytes / (ms_step * 1e-3) / 1e9
        traffic, traffic_src = ncu_traffic(args.mode, kern_bytes / kern_launches, key="sysmem_over_algorithmic")
        roof = {"bound": "pcie", "achieved": achieved, "peak": b_h2d / world, "unit": "GB/s",
                "frac": achieved / (b_h2d / world), "traffic": traffic, "traffic_source": traffic_src,
                "traffic_note": "bytes the launch pulled from host memory over PCIe (ncu syslts sysmem sectors x 32) "
                                "-- the bounding link; its HBM writes mostly stay in the 126 MB L2 past the launch",
                "kernel": "materialise_tma_kernel<store,check> (zero-copy host source)",
                "launches_per_step": kern_launches, "avg_launch_ms": kern_ms / max(kern_launches, 1),
                "peak_source": "cudaMemcpyAsync H2D from the same pinned buffer, 4 GiB, best of 5, this run"}
    standalone = None
    if not args.no_standalone and rank == 0:
        bases = per_tensor = None
        torch.cuda.empty_cache()
        standalone = standalone_hbm(idx, bufs, torch, sllm)
    if standalone is not None:
        hbm = peaks().get("hbm_gbs", 6551.4)
        k4 = standalone["k4"]
        standalone["k4"]["frac_hbm"] = k4["GBps"] / hbm
        standalone["k3"]["frac_hbm"] = standalone["k3"]["GBps"] / hbm
        if roof is None:
            roof = {"bound": "hbm", "achieved": k4["GBps"], "peak": hbm, "unit": "GB/s", "frac": k4["GBps"] / hbm,
                    "traffic": None, "kernel": "materialise_kernel<checksum only> (K4, standalone 4 GiB)"}
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, bufs, idx, inv, seed)
    clocks = clk.summary()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u8", "data": "synthetic",
                "config": arm_config(args, world, len(parts), payload_bytes, raw_bytes, replicated, {
                    **({"spread": f"{len(parts)} partitions over GPUs {used} from one process"} if args.spread else {}),
                    **({"same_gpu_plumbing_check": "all ranks on cuda:0 (gloo); not a scaling number"}
                       if SAME_GPU and world > 1 else {})}),
                "time_to_loaded_model_s": ms_step * 1e-3, "t_alloc_s": t_alloc, "t_setup_s": t_setup,
                "b_h2d_measured_GBps": b_h2d, "frac_h2d": pcie_rate / b_h2d,
                "gpu_launches": int(rep["kernel_launches"]) * args.steps,
                "copy_calls_per_step": int(rep["copy_calls"]),
                "clocks": clocks, "e2e": e2e, "roofline": roof, "roofline_h2d": h2d, "standalone_hbm": standalone,
                "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.free()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
