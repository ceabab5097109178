"""Checkpoint-load benchmark (BASELINE.json metric: "checkpoint load GB/s &
time-to-loaded-model at 1/2/4/8 B200 vs PCIe peak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config auto|opt-6.7b|llama2-70b-tp8|...] [--mode ce|zerocopy|scatter_ce|scatter_zc]
                    [--fanout none|bcast|allgather|p2p] [--chunk-mib 64] [--streams 2] [--ctas 0]

A "step" is one pass of the whole hot path over the synthetic
checkpoint already sitting in pinned host DRAM: open the index from its bytes (a1), plan
chunks (a3), move every partition byte host->HBM (a4), materialise the tensors (a5),
verify every 1 MiB block's Fletcher-64 on the GPU (a6), fan out (a7, replicated configs),
complete (a8).  Destinations are preallocated (a2; T_alloc is reported separately,
DESIGN.md Q19; `e2e` includes it).

Launch.  One process per GPU.  `--gpus N` with N > 1 outside torchrun re-launches this
script under `torch.distributed.run` with N ranks (and fails loudly when fewer than N GPUs
are visible); under torchrun WORLD_SIZE must equal N.

Workload (`--config auto`, the default) -- BASELINE.json configs by GPU count:
  N = 1: configs[1] OPT-6.7B (13.3 GB, 1 partition);  N = 2: configs[2] LLaMA-2-13B TP2;
  N = 4: LLaMA-2-70B TP4;  N = 8: configs[3] LLaMA-2-70B TP8 (the north star);
  with a fan-out: configs[4] OPT-30B replicated.
Sharded configs: rank r loads partition r (mod #partitions) over its own PCIe link from a
NUMA-local pinned source, no collective (weak scaling).  Replicated: every
rank ends with a full replica, each byte crossing PCIe once (a7).

value = payload bytes loaded by all ranks / max-over-ranks device time (GB/s, 10^9).
Per-GPU inputs (>= 13 GB) are ~100x the 126 MB L2: no flush between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "checkpoint load GB/s & time-to-loaded-model at 1/2/4/8 B200 vs PCIe peak"
# BASELINE.json configs by GPU count (sharded); replicated runs use configs[4]
CONFIG_FOR_N = {1: "opt-6.7b", 2: "llama2-13b-tp2", 4: "llama2-70b-tp4", 8: "llama2-70b-tp8"}
REPLICATED_CONFIG = "opt-30b"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="auto",
                    help="workload; auto = BASELINE config for the GPU count (see module docstring)")
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
    ap.add_argument("--fanout", default="none", choices=["none", "bcast", "allgather", "p2p", "nvls"],
                    help="replicated checkpoint: every rank ends with a full replica; rank r reads slice r over "
                         "PCIe and the rest arrives over NVLink (bcast: NCCL broadcasts, allgather: in-place NCCL "
                         "all-gathers, p2p: fused peer stores, nvls: multicast stores from ONE process over "
                         "--nvls-gpus GPUs)")
    ap.add_argument("--nvls-gpus", type=int, default=0, help="--fanout nvls: group size (0 = every visible GPU)")
    ap.add_argument("--cpu-sample-gib", type=float, default=2.0,
                    help="oracle sample per partition (cpu_baseline and --impl reference)")
    ap.add_argument("--cpu-reps", type=int, default=3, help="timed oracle reps for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-standalone", action="store_true")
    ap.add_argument("--no-baselines", action="store_true", help="replicated runs: skip the naive / root-broadcast lines")
    ap.add_argument("--no-profile", action="store_true", help="no per-launch CUDA events in the timed region")
    ap.add_argument("--capture", action="store_true",
                    help="captured load (sllm_load_capture): the load recorded once as CUDA graphs outside the "
                         "timed region (a1-a3 once), each step one replay (a4-a8) + wait -- repeated loads of one "
                         "checkpoint from the same pinned source into the same destinations; no fan-out")
    ap.add_argument("--plumbing", action="store_true",
                    help="CPU-only dry run of the launch / rank / max-over-ranks plumbing (gloo, host memcpy in place "
                         "of the load; not a measurement)")
    return ap.parse_args(argv)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# SLLM_BENCH_SAME_GPU=1: every rank on cuda:0 with a gloo group -- a plumbing check of the
# multi-rank paths (barriers, max-over-ranks timing, IPC peer groups) on a 1-GPU box; its
# numbers share one PCIe link and are not scaling results.
SAME_GPU = os.environ.get("SLLM_BENCH_SAME_GPU") == "1"


def gpu_of(local):
    return 0 if SAME_GPU else local


def resolve_config(args, world: int) -> str:
    if args.config != "auto":
        return args.config
    if args.fanout != "none":
        return REPLICATED_CONFIG
    return CONFIG_FOR_N.get(world, CONFIG_FOR_N[1])


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def fail_loudly(msg: str, code: int = 2):
    print(json.dumps({"metric": METRIC, "error": msg}), file=sys.stderr, flush=True)
    raise SystemExit(code)


def visible_gpus() -> int:
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def maybe_self_launch(args, argv) -> None:
    """`--gpus N` (N > 1) outside torchrun: re-launch under torch.distributed.run with N ranks
    (one process per GPU), rendezvous on 127.0.0.1; exit with the launcher's status."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    if not args.plumbing and not SAME_GPU and args.impl == "ours":
        n = visible_gpus()
        if n < args.gpus:
            fail_loudly(f"--gpus {args.gpus} needs {args.gpus} visible GPUs, found {n}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__), *argv]
    raise SystemExit(subprocess.run(cmd).returncode)


def max_over_ranks(x, world: int):
    """Max of a per-rank float (or list of floats) over the job."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    nccl = dist.get_backend() == "nccl"
    vec = x if isinstance(x, (list, tuple)) else [x]
    t = torch.tensor(vec, dtype=torch.float64, device=torch.cuda.current_device() if nccl else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out = [float(v) for v in t.tolist()]
    return out if isinstance(x, (list, tuple)) else out[0]


def step_stats(ms):
    return {"median": statistics.median(ms), "min": min(ms), "max": max(ms), "n": len(ms),
            "all": [round(float(x), 3) for x in ms]}


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
        num = lambda k: [float(r[k]) for r in self.rows if len(r) > k and r[k].replace(".", "").isdigit()]  # noqa: E731
        mem, mem_max = num(8), num(9)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "mem_mhz": statistics.median(mem) if mem else None, "mem_max_mhz": max(mem_max) if mem_max else None}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def bitexact_sample(res, inv, seed: int, torch, n_random: int = 10) -> dict:
    """Sampled tensors of a finished load compared byte for byte with the seeded payload
    generator (synth/payload.py, the inputs' own source -- no oracle arithmetic): the first
    and last three tensors in source order, the largest, the smallest and `n_random` seeded
    picks.  Every block of every timed load was also checked on the GPU against the index's
    Fletcher-64 table (a mismatch fails the load with SLLM_E_CHECKSUM)."""
    import random
    import numpy as np
    from synth import payload
    cand = [e for e, t in enumerate(inv) if t.name in res.tensors]
    if not cand:
        return None
    pick = set(cand[:3] + cand[-3:])
    pick.add(max(cand, key=lambda e: inv[e].nbytes))
    pick.add(min(cand, key=lambda e: inv[e].nbytes))
    pick.update(random.Random(seed).sample(cand, min(n_random, len(cand))))
    pick = sorted(pick)
    want = [np.empty(inv[e].nbytes, np.uint8) for e in pick]
    payload.payload_into([a.ctypes.data for a in want], [a.size for a in want], seed, pick)
    equal = True
    for e, w in zip(pick, want):
        got = res.tensors[inv[e].name].reshape(-1).view(torch.uint8).cpu().numpy()
        equal &= bool(np.array_equal(got, w))
    return {"equal": equal, "tensors_checked": len(pick), "tensors_loaded": len(cand),
            "bytes_checked": int(sum(inv[e].nbytes for e in pick)),
            "against": "seeded payload generator (synth/payload.py), last timed load, untimed",
            "every_block_checked_on_gpu": "each timed load compared every 1 MiB block's Fletcher-64 with the "
                                          "index table (mismatch = SLLM_E_CHECKSUM)"}


def host_description() -> dict:
    """the host cores the oracle runs on."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "affinity_cores": len(os.sched_getaffinity(0))}


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


def arm_config(args, config, world, parts, payload_bytes, raw_bytes, replicated, extra=None):
    """The JSON line's `config` -- identical for our arm and the reference arm."""
    return {"workload": config, "mode": args.mode, "fanout": args.fanout, "chunk_mib": args.chunk_mib,
            "engine": args.engine, "streams": args.streams, "ctas": args.ctas, "partitions_per_gpu": parts,
            "payload_bytes_per_gpu": payload_bytes, "raw_bytes_per_gpu": raw_bytes,
            "verify": "fletcher64 per 1 MiB block, every block",
            "l2": f"inputs {raw_bytes / 1e9:.1f} GB per GPU >> 126 MB L2, no flush needed",
            "parallelism": f"replicated x{world} ({args.fanout})" if replicated else f"sharded x{world}",
            **(extra or {})}


# ---------------------------------------------------------------------------------------
# The oracle leg (cpu_baseline of our arm, and the whole reference arm).  ONE protocol for
# both: the first `budget` bytes of each sampled partition (whole tensors), converted by the
# oracle's converter into fresh NumPy memory, then oracle.loader.load_sample (parse the
# index, copy every tensor, recompute + compare every 1 MiB Fletcher-64 block) timed per
# rep.  Mode (i): one process = 1 core.  Mode (ii): P = min(#partitions,
# usable cores) processes, one partition sample each, started together per rep; aggregate =
# all payload / (last end - first start).
# ---------------------------------------------------------------------------------------
def _oracle_sample_inputs(config: str, part: int, budget: int):
    import numpy as np
    from oracle import index as oindex, layout as olayout
    from synth import models, payload
    inv, seed = models.model_inventory(config)
    lay = olayout.plan([(t.name, t.device, t.dtype, t.shape, t.nbytes) for t in inv], 4096, 1 << 20)
    d = lay.devices()[part]
    ents = [(i, e) for i, e in enumerate(lay.entries) if e.device == d]
    first_end = min(e.offset + e.size for _, e in ents)
    budget = max(budget, -(-first_end // (1 << 20)) << 20)       # at least one whole tensor
    keep = [i for i, e in ents if e.offset + e.size <= budget]
    arrs = [np.empty(inv[i].nbytes, np.uint8) for i in keep]      # the seeded payloads (O10)
    payload.payload_into([a.ctypes.data for a in arrs], [a.size for a in arrs], seed, keep)
    tensors = [(inv[i].name, d, inv[i].dtype, inv[i].shape, a) for i, a in zip(keep, arrs)]
    slay, sparts = olayout.convert(tensors, 4096, 1 << 20, config)
    return oindex.write(slay), sparts, budget


def _oracle_worker(config, parts, budget, reps, barrier, q):
    try:
        from oracle import loader as oloader
        inputs = [_oracle_sample_inputs(config, p, budget) for p in parts]
        spans = []
        got = 0
        for _ in range(reps):
            if barrier is not None:
                barrier.wait()
            t0 = time.perf_counter()  # CLOCK_MONOTONIC: comparable across processes
            got = sum(oloader.load_sample(blob, sp, b) for blob, sp, b in inputs)
            spans.append((t0, time.perf_counter()))
        q.put(("ok", got, spans))
    except Exception as ex:  # noqa: BLE001
        import traceback
        q.put(("error", repr(ex), traceback.format_exc()))


def oracle_run(config: str, parts, budget: int, reps: int) -> dict:
    """Time the oracle on samples of `parts` (mode (i) for one partition, mode (ii) for
    several).  Returns per-rep aggregate seconds and the payload per rep."""
    import multiprocessing as mp
    parts = list(parts)
    cores = len(os.sched_getaffinity(0))
    P = max(1, min(len(parts), cores))
    if P == 1:
        import queue
        q = queue.Queue()
        _oracle_worker(config, parts, budget, reps, None, q)
        res = [q.get()]
    else:
        ctx = mp.get_context("spawn")
        q, barrier = ctx.Queue(), ctx.Barrier(P)
        groups = [parts[i::P] for i in range(P)]
        procs = [ctx.Process(target=_oracle_worker, args=(config, g, budget, reps, barrier, q)) for g in groups]
        for p in procs:
            p.start()
        res = [q.get(timeout=3600) for _ in procs]
        for p in procs:
            p.join(timeout=60)
    for r in res:
        if r[0] != "ok":
            raise RuntimeError(f"oracle worker failed: {r[1]}\n{r[2]}")
    got = sum(r[1] for r in res)
    secs = [max(r[2][k][1] for r in res) - min(r[2][k][0] for r in res) for k in range(reps)]
    return {"payload": got, "secs": secs, "cores": P, "partitions": len(parts)}


def oracle_line_fields(run: dict, budget: int, config: str, timed_reps) -> dict:
    secs = run["secs"][-timed_reps:] if timed_reps else run["secs"]
    med = statistics.median(secs)
    return {"value": run["payload"] / med / 1e9, "unit": "GB/s", "cores": run["cores"], "kind": "oracle",
            "mode": "(i) 1 process" if run["cores"] == 1 else f"(ii) {run['cores']} processes, one partition each",
            "median_s": med, "min_s": min(secs), "best_GBps": run["payload"] / min(secs) / 1e9, "reps": len(secs),
            "sample": f"first {budget / 2**30:.2f} GiB (whole tensors) of each of {run['partitions']} partition(s) of "
                      f"{config}: {run['payload']} payload bytes per rep -- parse index, copy every tensor, "
                      f"recompute + compare every 1 MiB Fletcher-64 block (oracle/loader.py load_sample); inputs "
                      f"built by the oracle converter in fresh NumPy memory, untimed",
            "host": host_description()}


def oracle_budget(args) -> int:
    """Per-partition sample: --cpu-sample-gib, shrunk for the reference arm so that warm-up +
    timed steps stay within ~60 GB of oracle work per process (a few minutes)."""
    b = int(args.cpu_sample_gib * (1 << 30))
    if args.impl == "reference":
        b = min(b, max(256 << 20, int(60e9 / max(1, args.warmup + args.steps))))
    return b


def run_reference(args, rank, world):
    """Reference arm = the CPU oracle as it stands (oracle/loader.py) on this box's host
    cores, each step one bounded sample of the same workload (rank 0 only under torchrun)."""
    if rank != 0:
        return
    from oracle import layout as olayout
    from synth import models
    config = resolve_config(args, world)
    inv, _ = models.model_inventory(config)
    lay = olayout.plan([(t.name, t.device, t.dtype, t.shape, t.nbytes) for t in inv], 4096, 1 << 20)
    n_parts = len(lay.devices())
    replicated = args.fanout != "none"
    # the partitions our arm loads per node: all of a sharded config across its ranks (each
    # rank one), partition 0 of a replicated or single-GPU run
    if args.all_partitions:
        sel = list(range(n_parts))
    elif replicated or n_parts == 1:
        sel = [0]
    else:
        sel = sorted({r % n_parts for r in range(world)})
    budget = oracle_budget(args)
    run = oracle_run(config, sel, budget, args.warmup + args.steps)
    cpu = oracle_line_fields(run, budget, config, args.steps)
    T = sum(run["secs"][args.warmup:])
    v = run["payload"] * args.steps / T / 1e9
    cpu["value"] = v
    devs = [lay.devices()[p] for p in sel]
    per_gpu = sel[:1] if not args.all_partitions else sel
    pdevs = [lay.devices()[p] for p in per_gpu]
    line = {"metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": T / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic", "impl": "reference",
            "config": arm_config(args, config, world, len(per_gpu), sum(e.size for e in lay.entries if e.device in pdevs),
                                 sum(lay.partitions[d] for d in pdevs), replicated),
            "step_s": step_stats(run["secs"][args.warmup:]),
            "cpu_baseline": cpu,
            "sampled_partitions": [int(d) for d in devs],
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
# Plumbing dry run (CPU, gloo): the launcher, rank -> partition selection, barriers and
# max-over-ranks timing, with a host memcpy of each rank's partition standing in for the
# load.  Not a measurement; tests/test_bench_launch.py drives it.
# ---------------------------------------------------------------------------------------
def run_plumbing(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist
    from synth import models
    config = resolve_config(args, world)
    inv, _ = models.model_inventory(config)
    devs = sorted({t.device for t in inv})
    sel = choose_partitions(args, rank, world, len(devs), args.fanout != "none")
    nbytes = min(sum(t.nbytes for t in inv if t.device == devs[sel[0]]), 64 << 20)
    src = np.random.default_rng(rank).integers(0, 256, nbytes, dtype=np.uint8)
    dst = np.empty_like(src)
    if world > 1:
        dist.barrier()
    secs = []
    for _ in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        dst[:] = src
        secs.append(time.perf_counter() - t0)
    secs = max_over_ranks(secs[args.warmup:], world)
    ranks = [None] * world
    mine = {"rank": rank, "local_rank": local, "pid": os.getpid(), "partitions": sel,
            "world_size_env": int(os.environ.get("WORLD_SIZE", 1))}
    if world > 1:
        dist.all_gather_object(ranks, mine)
    else:
        ranks = [mine]
    if rank == 0:
        T = sum(secs)
        print(json.dumps({"metric": METRIC, "value": nbytes * world * args.steps / T / 1e9, "unit": "GB/s",
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": T / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
                          "plumbing": True, "config": {"workload": config}, "ranks": ranks}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def choose_partitions(args, rank, world, n_parts, replicated):
    if args.all_partitions:
        return list(range(n_parts))
    if replicated or n_parts == 1:
        return [0]
    return [rank % n_parts]


# ---------------------------------------------------------------------------------------
# Rooflines measured in the same run
# ---------------------------------------------------------------------------------------
def _rt_ok(rt, ret):
    """Unwrap a cuda-python runtime call's (error, value...) tuple; raise on any error."""
    ret = ret if isinstance(ret, tuple) else (ret,)
    if ret[0] != rt.cudaError_t.cudaSuccess:
        raise RuntimeError(f"CUDA runtime call failed: {ret[0]}")
    return ret[1] if len(ret) > 1 else None


def h2d_peak(bufs, bases, torch, gib=4, reps=5, world=1, gpus=None):
    """B_h2d(N): the copy engine's best host->device rate from the same pinned buffer into
    the same destination over >= 4 GiB: max of one 4 GiB
    cudaMemcpyAsync and back-to-back 64 MiB cudaMemcpyAsync calls on one stream, best of
    `reps` each (plain cudaMemcpyAsync through the cuda-python runtime bindings when present,
    queued behind a ~1 ms stream hold).  Under torchrun every rep starts on a barrier so all N links (and the host
    DRAM / PCIe switches they share) are loaded at once; the aggregate is N * bytes / the
    slowest rank's time.  With partitions on several GPUs of this process (--spread) one
    partition per GPU copies at once, aggregate = their bytes / the slowest GPU's time.
    Returns (aggregate GB/s, {method: aggregate GB/s})."""
    try:  # the CUDA runtime bindings (cuda-python): copies issued without torch's copy_ path
        from cuda.bindings import runtime as rt
    except ImportError:
        rt = None
    if os.environ.get("SLLM_BENCH_PEAK_TORCH") == "1":  # A/B: torch copy_ instead
        rt = None
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
                step = piece or n
                with torch.cuda.device(g):
                    # hold the stream ~1 ms so every copy is enqueued before the start event
                    # runs: the events then time the copy engine, not the host's copy issue
                    torch.cuda._sleep(2_000_000)
                    if rt is not None:  # plain cudaMemcpyAsync calls, no framework in the way
                        st = torch.cuda.current_stream(g).cuda_stream
                        _rt_ok(rt, rt.cudaSetDevice(g))
                        s, e = _rt_ok(rt, rt.cudaEventCreate()), _rt_ok(rt, rt.cudaEventCreate())
                        _rt_ok(rt, rt.cudaEventRecord(s, st))
                        for o in range(0, n, step):
                            _rt_ok(rt, rt.cudaMemcpyAsync(bases[p].data_ptr() + o, bufs[p].ptr + o, min(step, n - o),
                                                          rt.cudaMemcpyKind.cudaMemcpyHostToDevice, st))
                        _rt_ok(rt, rt.cudaEventRecord(e, st))
                    else:
                        src, dst = bufs[p].torch()[:n], bases[p][:n]
                        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        s.record()
                        for o in range(0, n, step):
                            dst[o:o + step].copy_(src[o:o + step], non_blocking=True)
                        e.record()
                evs.append((s, e))
            if rt is not None:
                for s, e in evs:
                    _rt_ok(rt, rt.cudaEventSynchronize(e))
                times = [_rt_ok(rt, rt.cudaEventElapsedTime(s, e)) for s, e in evs]
                for s, e in evs:
                    rt.cudaEventDestroy(s)
                    rt.cudaEventDestroy(e)
            else:
                for s, e in evs:
                    e.synchronize()
                times = [s.elapsed_time(e) for s, e in evs]
            ms = max_over_ranks(max(times), world)
            best = max(best, world * sum(sizes.values()) / (ms * 1e-3) / 1e9)
        out[name] = best
    return max(out.values()), out


def nvlink_peaks(torch, world, gpu, mib=1024, reps=3):
    """NVLink fan-out roofline, measured over the job's NCCL process group
    in the same run, best of `reps`, barrier-started, max-over-ranks time:
      bcast_GBps     : ncclBroadcast of `mib` MiB, root rotating (bus bandwidth = algorithm
                       bandwidth for a broadcast);
      allgather_busbw: ncclAllGather of mib/N MiB per rank, busbw = (N-1)/N * total / t;
      p2p_ingress    : every rank sends `mib` MiB to rank+1 and receives from rank-1 at once
                       (ncclSend/Recv), per-rank ingress rate.
    A replicated load's NVLink bound is S(N-1)/N per GPU of ingress over these rates."""
    import torch.distributed as dist
    dev = torch.device("cuda", gpu) if dist.get_backend() == "nccl" else torch.device("cpu")
    if dev.type == "cpu":  # gloo plumbing runs (SLLM_BENCH_SAME_GPU): a token size
        mib = min(mib, 64)
    n = (mib << 20)
    buf = torch.empty(n, dtype=torch.uint8, device=dev)
    rbuf = torch.empty(n, dtype=torch.uint8, device=dev)
    per = n // world
    ag_in = buf[:per]
    ag_out = [rbuf[q * per:(q + 1) * per] for q in range(world)]
    rank = dist.get_rank()

    def timed(fn):
        best = None
        for _ in range(reps):
            dist.barrier()
            if dev.type == "cuda":
                torch.cuda.synchronize(gpu)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                fn()
                e.record()
                e.synchronize()
                ms = s.elapsed_time(e)
            else:
                t0 = time.perf_counter()
                fn()
                ms = (time.perf_counter() - t0) * 1e3
            ms = max_over_ranks(ms, world)
            best = ms if best is None else min(best, ms)
        return best

    k = [0]

    def bcast():
        dist.broadcast(buf, src=k[0] % world)
        k[0] += 1

    def p2p():
        ops = [dist.P2POp(dist.isend, buf, (rank + 1) % world), dist.P2POp(dist.irecv, rbuf, (rank - 1) % world)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()

    t_b = timed(bcast)
    t_ag = timed(lambda: dist.all_gather(ag_out, ag_in))
    t_p = timed(p2p)
    return {"bcast_GBps": n / (t_b * 1e-3) / 1e9,
            "allgather_busbw_GBps": (world - 1) / world * per * world / (t_ag * 1e-3) / 1e9,
            "p2p_ingress_GBps": n / (t_p * 1e-3) / 1e9, "bytes": n, "backend": dist.get_backend()}


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
    _, per = sllm.allocate(idx, {p: torch.cuda.current_device()}, scatter=True, partitions=[p])  # beside `src`
    ts = [sllm.materialise_device(idx, p, src.data_ptr(), per, 0, st, timed=True) for _ in range(reps)]
    t = min(ts) * 1e-3
    payload = sum(x.nbytes for x in idx.tensors if x.partition == p)
    res["k3"] = {"bytes": L + payload, "ms": t * 1e3, "GBps": (L + payload) / t / 1e9, "status_ok": True,
                 "timing": "library CUDA events around the K3 launch"}
    del per, src, out
    torch.cuda.empty_cache()
    return res


def replicated_baselines(sllm, torch, idx, bufs, gpus, cfg, bases, world, rank, reps=2):
    """the replicated load without the fan-out, at the same N, same buffers.
      naive      : every rank loads the whole partition over its own PCIe link (N*S PCIe bytes);
      root_bcast : rank 0 loads S, then one NCCL broadcast of S to every rank (S over one link).
    Aggregate GB/s = N full replicas / max-over-ranks device time, best of `reps`."""
    import torch.distributed as dist
    from dataclasses import replace
    p = 0
    S = idx.partitions[p].length
    payload = sum(t.nbytes for t in idx.tensors if t.partition == p)
    nc = replace(cfg, fanout="none", profile=False)
    st = torch.cuda.current_stream(gpus[p])
    out = {}
    for name in ("naive", "root_bcast"):
        best = None
        for _ in range(reps):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st)
            if name == "naive" or rank == 0:
                res = sllm.load_start(idx, {p: bufs[p]}, {p: gpus[p]}, nc, bases, None, {p: st}, None)
                res.wait()
                del res
            if name == "root_bcast" and world > 1:
                dist.broadcast(bases[p], src=0)
            e.record(st)
            e.synchronize()
            ms = max_over_ranks(s.elapsed_time(e), world)
            best = ms if best is None else min(best, ms)
        out[name] = {"value": payload * world / (best * 1e-3) / 1e9, "unit": "GB/s", "ms": best,
                     "pcie_bytes_total": S * (world if name == "naive" else 1)}
    return out


def run_nvls(args):
    """Replicated checkpoint over an NVLS multicast group driven by this one process (SURVEY
    §8(f) rank 4; the paper's model manager loading every GPU of a server): R GPUs,
    rank r reads slice r over its own PCIe link, its loading kernel stores every vector once
    through the multicast address and the NVSwitch writes all R replicas.  Fails loudly
    (exit 2) where the platform cannot create multicast objects."""
    import torch
    import paper_2401_14351_b200 as sllm
    from paper_2401_14351_b200 import workloads
    from synth import models, payload
    payload.build_csynth()
    R = args.nvls_gpus or visible_gpus()
    if R < 1 or visible_gpus() < R:
        fail_loudly(f"--fanout nvls over {R} GPUs needs {R} visible GPUs, found {visible_gpus()}")
    config = args.config if args.config != "auto" else REPLICATED_CONFIG
    inv, seed = models.model_inventory(config)
    if len(set(t.device for t in inv)) != 1:
        fail_loudly("--fanout nvls needs a single-partition (replicated) checkpoint config")
    t0 = time.perf_counter()
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20, config, partitions=[0], gpu_of={0: 0})
    t_setup = time.perf_counter() - t0
    blob = idx.serialize()
    L = idx.partitions[0].length
    payload_bytes = sum(t.nbytes for t in idx.tensors)
    try:
        comms = sllm.Comm.nvls(list(range(R)), L)
    except sllm.SllmError as ex:
        fail_loudly(f"NVLS unavailable on this platform: {ex}")
    bases = [c.replica()[:L] for c in comms]
    cfg = sllm.LoadConfig(chunk_bytes=args.chunk_mib << 20, n_streams=args.streams, mode=args.mode,
                          ctas=args.ctas, fanout="nvls", engine=args.engine)
    streams = [torch.cuda.current_stream(r) for r in range(R)]
    # B_h2d(R): every GPU copies 4 GiB of the partition at once (the R links together)
    n = min(4 << 30, L)
    best = 0.0
    for _ in range(3):
        for r in range(R):
            torch.cuda.synchronize(r)
        evs = []
        for r in range(R):
            with torch.cuda.device(r):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                bases[r][:n].copy_(bufs[0].torch()[:n], non_blocking=True)
                b.record()
                evs.append((a, b))
        for a, b in evs:
            b.synchronize()
        best = max(best, R * n / (max(a.elapsed_time(b) for a, b in evs) * 1e-3) / 1e9)

    def step():
        ix = sllm.Index.from_bytes(blob)
        results = [sllm.load_start(ix, bufs, {0: r}, cfg, {0: bases[r]}, None, {0: streams[r]}, comms[r])
                   for r in range(R)]
        return [res.wait() for res in results]
    for _ in range(args.warmup):
        step()
    for r in range(R):
        torch.cuda.synchronize(r)
    marks = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(R)]
             for _ in range(args.steps)]
    reports = []
    with ClockSampler(0) as clk:
        for k in range(args.steps):
            for r in range(R):
                marks[k][r][0].record(streams[r])
            reports = step()
            for r in range(R):
                marks[k][r][1].record(streams[r])
        for r in range(R):
            torch.cuda.synchronize(r)
    ms_steps = [max(m[r][0].elapsed_time(m[r][1]) for r in range(R)) for m in marks]
    ms_step = max(marks[0][r][0].elapsed_time(marks[-1][r][1]) for r in range(R)) / args.steps
    ok = all(c.replica()[:L].cpu().numpy().tobytes() == bufs[0].numpy()[:L].tobytes() for c in comms[:1])
    pcie = sum(rep["transferred_bytes"] for rep in reports)
    value = payload_bytes * R / (ms_step * 1e-3) / 1e9
    line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": R, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": arm_config(args, config, R, 1, payload_bytes, L, True,
                                 {"nvls": f"one process, multicast group over GPUs 0..{R - 1}"}),
            "time_to_loaded_model_s": ms_step * 1e-3, "step_ms": step_stats(ms_steps), "t_setup_s": t_setup,
            "b_h2d_measured_GBps": best, "frac_h2d": pcie / (ms_step * 1e-3) / 1e9 / best,
            "roofline_h2d": {"bound": "pcie", "achieved": pcie / (ms_step * 1e-3) / 1e9, "peak": best, "unit": "GB/s",
                             "frac": pcie / (ms_step * 1e-3) / 1e9 / best, "n_links": R},
            "replica0_equals_source": ok, "gpu_launches": sum(int(rep["kernel_launches"]) for rep in reports) * args.steps,
            "clocks": clk.summary(), "e2e": None, "roofline": None, "cpu_baseline": None}
    print(json.dumps(line), flush=True)
    for c in comms:
        c.free()


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    maybe_self_launch(args, argv)
    rank, world, local = dist_env()
    if world > 1 and args.gpus not in (1, world):
        fail_loudly(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)  # rank 0 alone (no process group: the others exit at once)
        return
    if args.plumbing:
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
        run_plumbing(args, rank, world, local)
        return
    if args.fanout == "nvls":
        if world > 1:
            fail_loudly("--fanout nvls drives every GPU of the group from one process: run without torchrun")
        run_nvls(args)
        return
    import torch
    if world > 1:
        import torch.distributed as dist
        if not SAME_GPU and visible_gpus() < world:
            fail_loudly(f"{world} ranks need {world} visible GPUs, found {visible_gpus()}")
        if SAME_GPU and args.fanout == "p2p":
            # ranks sharing a GPU must not run kernels that spin on each other's flags: the
            # load workers wait for the peers' flags on the host instead
            os.environ["SLLM_PEER_WAIT"] = "host"
        torch.cuda.set_device(gpu_of(local))
        if SAME_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif not torch.cuda.is_available():
        fail_loudly("no CUDA GPU visible (bench.py measures the GPU path; --plumbing for a CPU dry run)")

    import paper_2401_14351_b200 as sllm
    from paper_2401_14351_b200 import workloads
    from synth import models, payload

    payload.build_csynth()
    gpu = gpu_of(local)
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    config = resolve_config(args, world)

    # ---- setup (untimed): synthetic checkpoint packed into pinned DRAM by the converter
    t0 = time.perf_counter()
    inv, seed = models.model_inventory(config)
    replicated = args.fanout != "none"
    if replicated and len(set(t.device for t in inv)) != 1:
        raise SystemExit("--fanout needs a single-partition (replicated) checkpoint config")
    n_parts = len(set(t.device for t in inv))
    sel = choose_partitions(args, rank, world, n_parts, replicated)
    if args.spread and (not args.all_partitions or world > 1 or replicated):
        raise SystemExit("--spread goes with --all-partitions in a single process (no fan-out)")
    ndev = torch.cuda.device_count() if args.spread else 1
    gpu_map = {p: (p % ndev if args.spread else gpu) for p in sel}
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20, config, partitions=sel, gpu_of=gpu_map)
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

    peak_dst = bases if not cfg.scatter else {
        p: torch.empty(min(4 << 30, idx.partitions[p].length), dtype=torch.uint8, device=f"cuda:{gpus[p]}") for p in parts}
    b_h2d, b_h2d_methods = h2d_peak(bufs, peak_dst, torch, world=world, gpus=gpus)
    del peak_dst
    nvl = None
    if replicated and world > 1:
        nvl = nvlink_peaks(torch, world, gpu)
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

    captured = None
    if args.capture:
        if comm is not None:
            fail_loudly("--capture has no fan-out")
        captured = sllm.load_capture(sllm.Index.from_bytes(blob), bufs, gpus,
                                     sllm.LoadConfig(**{**cfg.__dict__, "profile": 0}), bases, per_tensor)

    def step(prof: bool):
        if captured is not None:  # one replay of the recorded graphs on the caller streams
            return captured.replay(streams), captured.index
        # profile 3: per-launch CUDA events + in-kernel spans (two %globaltimer atomics per CTA)
        c = sllm.LoadConfig(**{**cfg.__dict__, "profile": 3 if prof else 0})
        ix = sllm.Index.from_bytes(blob)                  # a1: open + validate the index
        res = sllm.load_start(ix, bufs, gpus, c, bases, per_tensor, streams, comm)
        return res, ix

    for _ in range(args.warmup):
        res, ix = step(not args.no_profile)  # the timed steps' exact work (profile level included)
        res.wait()
        del res, ix
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    sync_all()
    # serving-style Python hygiene: setup objects move to the permanent GC generation, so a
    # collection inside the timed loop scans only what the loads create
    import gc
    gc.collect()
    gc.freeze()
    reports = []
    prev = None
    with ClockSampler(gpu) as clk:
        # per-step start/end events on every GPU this process loads (its caller stream is
        # gated on the load); a step's time is its slowest GPU's, the run's the sum
        marks = [{g: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for g in used}
                 for _ in range(args.steps)]
        for k in range(args.steps):
            for g in used:
                marks[k][g][0].record(torch.cuda.current_stream(g))
            res, ix = step(not args.no_profile)
            # the previous step's model handles (its torch views, index) are released while this
            # load's transfer runs -- unloading a model never gates loading the next one
            prev = None
            reports.append(res.wait())
            for g in used:
                marks[k][g][1].record(torch.cuda.current_stream(g))
            prev = (res, ix)
            del res, ix
        sync_all()
    # the last timed load's tensors vs the seeded payloads, byte for byte (untimed)
    bitexact = bitexact_sample(prev[0], inv, seed, torch) if prev is not None else None
    prev = None
    if captured is not None:  # (its graphs and reserved destinations go before the e2e leg)
        captured.free()
        captured = None
    gc.unfreeze()
    if world > 1:
        dist.barrier()
    first_last = max(marks[0][g][0].elapsed_time(marks[-1][g][1]) for g in used)
    ms_total = max_over_ranks(first_last, world)
    ms_steps = max_over_ranks([max(m[g][0].elapsed_time(m[g][1]) for g in used) for m in marks], world)
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
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        ix = sllm.Index.from_bytes(blob)
        if comm is None:
            res = sllm.load(ix, bufs, gpus, sllm.LoadConfig(**{**cfg.__dict__, "profile": False}))
        else:  # a replicated group is bound to its replicas: no per-step allocation
            res = sllm.load_start(ix, bufs, gpus, sllm.LoadConfig(**{**cfg.__dict__, "profile": False}), bases,
                                  per_tensor, streams, comm)
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

    baselines = None
    if replicated and not args.no_baselines:
        baselines = replicated_baselines(sllm, torch, idx, bufs, gpus, cfg, bases, world, rank)

    # ---- roofline of the dominant kernel, from the library's per-launch CUDA events
    rep = reports[-1]
    kern_ms = sum(r["t_kernel_ms_sum"] for r in reports) / len(reports)
    kern_launches = rep["kernel_launches"]
    kern_bytes = rep["kernel_bytes"]
    roof = None
    pcie_rate = pcie_bytes * world / (ms_step * 1e-3) / 1e9
    h2d = {"bound": "pcie", "achieved": pcie_rate, "peak": b_h2d, "unit": "GB/s",
           "frac": pcie_rate / b_h2d, "peak_methods": b_h2d_methods, "n_links": world * len(used),
           "what": "host->device bytes of the whole step (a1-a8) over its device time vs the copy engine's "
                   "measured host->device peak on the same buffers (all links at once, barrier-started)"}
    if args.mode in ("ce", "scatter_ce") and kern_launches and kern_ms > 0:
        # the step's kernel: K4 (CE) / K3 (SCATTER_CE) on each landed chunk, per-launch
        # CUDA events recorded by the library on its kernel stream over the timed region
        per_launch_bytes = kern_bytes / kern_launches * (2 if args.mode == "scatter_ce" else 1)
        avg_ms = kern_ms / kern_launches
        achieved = per_launch_bytes / (avg_ms * 1e-3) / 1e9
        hbm = peaks().get("hbm_gbs", 6551.4)
        traffic, traffic_src = ncu_traffic(args.mode, per_launch_bytes)
        dram_pct, _ = ncu_traffic(args.mode, 1.0, key="dram_pct_of_peak")
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "traffic_source": traffic_src,
                "ncu_dram_pct_of_peak": dram_pct,  # the captured launch against ncu's own DRAM peak (cold)
                "kernel": "materialise_tma_kernel<%s> (in pipeline)" %
                ("checksum only" if args.mode == "ce" else "scatter+checksum"),
                "launches_per_step": kern_launches, "avg_launch_ms": avg_ms,
                "bytes_per_launch": per_launch_bytes,
                "peak_what": "MEASURED_PEAKS.json hbm_gbs: a device copy's read+write bytes per second; K4 only "
                             "reads, and a read-only stream has no read/write turnaround on the HBM bus, so it can "
                             "exceed the copy figure (ncu: K4 at ~90 % of the DRAM peak, profiles/r02)",
                "note": "two CTAs per SM, units handed out by ticket; each launch verifies a span of landed windows "
                        "(up to 4 GiB, shrinking towards the end) beside the PCIe copies"}
        span_ms = sum(r.get("t_kernel_span_ms_sum", 0.0) for r in reports) / len(reports)
        if span_ms > 0:  # the same launches timed from inside (first CTA start .. last CTA end)
            ach_in = per_launch_bytes / (span_ms / kern_launches * 1e-3) / 1e9
            roof["in_kernel"] = {"achieved": ach_in, "frac": ach_in / hbm, "avg_span_ms": span_ms / kern_launches,
                                 "what": "%globaltimer span of each launch; the CUDA-event time also holds the launch "
                                         "and completion, which cost ~30 us each while the copy engine saturates "
                                         "PCIe (profiles/r02/launch_gap.jsonl)"}
        if replicated and world > 1:
            roof["note"] = ("replicated load: the fan-out launches also store every byte they read into the "
                            f"{world - 1} peer replica(s) (NVLink; here counted as reads only) and the received "
                            "ranges are verified by K4 launches -- see roofline_nvlink for the fan-out's rate")
    if args.mode in ("zerocopy", "scatter_zc") and kern_launches and kern_ms > 0:
        # zero-copy kernel: every byte it reads crosses PCIe -> bound by the host link.
        # Launches on the S streams overlap, so the kernel's rate is its bytes per step
        # over the step's device time (the kernel is the only work in the step).
        achieved = kern_bytes / (ms_step * 1e-3) / 1e9
        traffic, traffic_src = ncu_traffic(args.mode, kern_bytes / kern_launches, key="sysmem_over_algorithmic")
        per_link = b_h2d / (world * len(used))
        roof = {"bound": "pcie", "achieved": achieved, "peak": per_link, "unit": "GB/s",
                "frac": achieved / per_link, "traffic": traffic, "traffic_source": traffic_src,
                "traffic_note": "bytes the launch pulled from host memory over PCIe (ncu syslts sysmem sectors x 32) "
                                "-- the bounding link; its HBM writes mostly stay in the 126 MB L2 past the launch",
                "kernel": "materialise_tma_kernel<store,check> (zero-copy host source)",
                "launches_per_step": kern_launches, "avg_launch_ms": kern_ms / max(kern_launches, 1),
                "peak_source": "cudaMemcpyAsync H2D from the same pinned buffer, 4 GiB, best of 3, this run"}
    nvlink = None
    if nvl is not None:
        # each GPU receives S(N-1)/N over NVLink per load; its rate against the measured
        # collective rates of the same group
        ingress = (idx.partitions[0].length - pcie_bytes) / (ms_step * 1e-3) / 1e9
        ref = {"bcast": nvl["bcast_GBps"], "allgather": nvl["allgather_busbw_GBps"],
               "p2p": nvl["p2p_ingress_GBps"]}[args.fanout]
        nvlink = {"bound": "nvlink", "achieved": ingress, "peak": ref, "unit": "GB/s", "frac": ingress / ref,
                  "what": "per-GPU NVLink ingress of the fan-out (S(N-1)/N per load) over its device time vs the "
                          "measured rate of the matching collective on the same group", "measured": nvl}
    standalone = None
    if not args.no_standalone and rank == 0 and not replicated:
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
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        budget = oracle_budget(args)
        run = oracle_run(config, parts, budget, args.cpu_reps)
        cpu = oracle_line_fields(run, budget, config, None)
    clocks = clk.summary()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u8", "data": "synthetic",
                "config": arm_config(args, config, world, len(parts), payload_bytes, raw_bytes, replicated, {
                    **({"spread": f"{len(parts)} partitions over GPUs {used} from one process"} if args.spread else {}),
                    **({"same_gpu_plumbing_check": "all ranks on cuda:0 (gloo); not a scaling number"}
                       if SAME_GPU and world > 1 else {}),
                    **({"peer_wait": "host (load workers poll the peers' flags; no kernel waits on another rank)"}
                       if os.environ.get("SLLM_PEER_WAIT") == "host" and args.fanout == "p2p" else {}),
                    **({"capture": "load recorded once as CUDA graphs outside the timed region (index parse and plan "
                                   "once); step = one replay (transfer, verify, materialise) + wait"}
                       if args.capture else {})}),
                "time_to_loaded_model_s": ms_step * 1e-3, "step_ms": step_stats(ms_steps), "bitexact": bitexact,
                "t_alloc_s": t_alloc, "t_setup_s": t_setup,
                "b_h2d_measured_GBps": b_h2d, "frac_h2d": pcie_rate / b_h2d,
                "gpu_launches": int(rep["kernel_launches"]) * args.steps,
                "copy_calls_per_step": int(rep["copy_calls"]),
                "clocks": clocks, "e2e": e2e, "roofline": roof, "roofline_h2d": h2d, "roofline_nvlink": nvlink,
                "replicated_baselines": baselines, "standalone_hbm": standalone,
                "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.free()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
