"""Multi-GPU parity and the round-1 hardening checks.

The N >= 2 cases need >= 2 physical GPUs and skip below that (this build's GPU box has
one); on an NVSwitch node they run every multi-GPU path for real:
  * sharded: one load call puts partition p on GPU p (the paper's model manager loading a
    server) -- every tensor and block checksum equals the oracle's;
  * replicated over NCCL with nranks >= 2, as separate processes (one per GPU) and as one
    process driving both GPUs (sllm_comm_init_all), bcast and allgather, CE and ZC;
  * the fused P2P fan-out across devices: in one process (plain pointers, peer access) and
    across processes (CUDA IPC mappings over NVLink);
  * the caller's current CUDA device is unchanged by loads onto other GPUs.
Every replica must equal the oracle's P_0 byte for byte (O9(c)); every block checksum the
oracle's (O9(d)).  Expected values come only from oracle/ and the synth payload definition.
"""
import os
import socket
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2401_14351_b200 as sllm  # noqa: E402
from paper_2401_14351_b200 import workloads  # noqa: E402
from oracle import layout as olayout  # noqa: E402
from synth import models, payload  # noqa: E402

NGPU = torch.cuda.device_count()
multi = pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")


def oracle_of(inv, seed, A=4096, B=1 << 20):
    payloads = [payload.payload_bytes(seed, e, t.nbytes) for e, t in enumerate(inv)]
    lay, parts = olayout.convert([(t.name, t.device, t.dtype, t.shape, p) for t, p in zip(inv, payloads)], A, B)
    return lay, parts, payloads


def replicated_inventory(seed=41, n=24):
    """~70 MB single partition (two 64 MiB fan-out units: one full round and a ragged one)."""
    rng = np.random.default_rng(seed)
    return [models.TensorSpec(f"r{i}", 0, "f16", (int(rng.integers(600, 1800)), 1031)) for i in range(n)], seed


# ---- single GPU: the round-1 hardening ------------------------------------------------
def test_zerocopy_rejects_misaligned_source_auto_keeps_ce():
    """ZEROCOPY / SCATTER_ZC read the source with 16-byte vectors and TMA: a source whose
    device alias is not 16-byte aligned is refused (SLLM_E_INVALID) before anything runs;
    AUTO keeps the copy engine for it and the result is still bit-exact."""
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, payloads = oracle_of(inv, seed)
    L = idx.partitions[0].length
    host = sllm.HostBuffer(L + 4096)
    host.numpy()[8:8 + L] = oparts[0]
    src = host.ptr + 8
    for mode in ("zerocopy", "scatter_zc"):
        with pytest.raises(sllm.SllmError) as ex:
            sllm.load(idx, {0: src}, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20, mode=mode))
        assert ex.value.status == 1 and "16-byte aligned" in str(ex.value)
    res = sllm.load(idx, {0: src}, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20, mode="auto"))
    assert res.report["mode"] == 0                     # SLLM_MODE_CE
    assert np.array_equal(res._keep[3][0].cpu().numpy(), oparts[0])
    assert res.block_checksums(0).tolist() == lay.checksums[0]
    del res
    host.free()


def test_current_device_unchanged_single_gpu():
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    torch.cuda.set_device(0)
    res = sllm.load(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20))
    res.free()
    assert torch.cuda.current_device() == 0


# ---- >= 2 GPUs ----------------------------------------------------------------------------
@multi
def test_current_device_restored_after_load_on_other_gpu():
    """a load onto GPU 1 issued from a thread whose current device is 0 leaves it
    on 0 -- after start, wait, block-checksum readback and free."""
    inv = models.llama2(256, 2, 512, 64, vocab=1024, tp=2)
    idx, bufs = workloads.build_pinned(inv, 5, 4096, 1 << 20, gpu_of={0: 0, 1: 1})
    torch.cuda.set_device(0)
    bases, _ = sllm.allocate(idx, {1: 1}, partitions=[1])
    res = sllm.load_start(idx, {1: bufs[1]}, {1: 1}, sllm.LoadConfig(chunk_bytes=1 << 20), bases)
    assert torch.cuda.current_device() == 0
    res.wait()
    assert torch.cuda.current_device() == 0
    res.block_checksums(1)
    assert torch.cuda.current_device() == 0
    res.free()
    assert torch.cuda.current_device() == 0


@multi
@pytest.mark.parametrize("mode", ["ce", "zerocopy", "scatter_ce", "scatter_zc"])
def test_sharded_one_call_partition_per_gpu(mode):
    """LLaMA-2-shaped TP checkpoint, partition p -> GPU p from one call (one worker per
    partition, one PCIe link each, no collective): bit-exact against the oracle."""
    n = min(NGPU, 4)
    inv = models.llama2(512, 2, 1024, 128, vocab=2048, tp=n)
    gpus = {p: p for p in range(n)}
    idx, bufs = workloads.build_pinned(inv, 6, 4096, 1 << 20, gpu_of=gpus)
    lay, oparts, payloads = oracle_of(inv, 6)
    res = sllm.load(idx, bufs, gpus, sllm.LoadConfig(chunk_bytes=1 << 20, mode=mode))
    for e, t in enumerate(inv):
        got = res.tensors[t.name]
        assert got.device.index == lay.devices().index(t.device)
        assert np.array_equal(got.contiguous().view(torch.uint8).reshape(-1).cpu().numpy(), payloads[e]), t.name
    for p, d in enumerate(lay.devices()):
        assert res.block_checksums(p).tolist() == lay.checksums[d]


@multi
@pytest.mark.parametrize("fanout", ["bcast", "allgather"])
@pytest.mark.parametrize("mode", ["ce", "zerocopy"])
def test_nccl_fanout_single_process_init_all(fanout, mode):
    """sllm_comm_init_all over GPUs 0..R-1, one host thread per rank issuing its part of the
    collective load: every GPU ends with P_0, each byte crossed PCIe once in total."""
    R = min(NGPU, 4)
    inv, seed = replicated_inventory()
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, _ = oracle_of(inv, seed)
    L = idx.partitions[0].length
    comms = sllm.Comm.init_all(list(range(R)))
    bases = [torch.full((L,), 0xA5, dtype=torch.uint8, device=f"cuda:{r}") for r in range(R)]
    for r in range(R):
        torch.cuda.synchronize(r)
    cfg = sllm.LoadConfig(chunk_bytes=2 << 20, mode=mode, fanout=fanout)
    reps, errs = [None] * R, []

    def rank(r):
        try:
            res = sllm.load_start(idx, bufs, {0: r}, cfg, {0: bases[r]}, None, None, comms[r])
            reps[r] = (res.wait(), res.block_checksums(0).tolist())
        except Exception as ex:  # noqa: BLE001
            errs.append((r, ex))
    th = [threading.Thread(target=rank, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    for r in range(R):
        assert np.array_equal(bases[r].cpu().numpy(), oparts[0]), r
        assert reps[r][1] == lay.checksums[0]
        assert reps[r][0]["fanout_bytes"] == L - reps[r][0]["transferred_bytes"]
    assert sum(rep[0]["transferred_bytes"] for rep in reps) == L
    for c in comms:
        c.free()


@multi
@pytest.mark.parametrize("mode", ["ce", "zerocopy"])
def test_p2p_fanout_across_gpus_one_process(mode):
    """The fused P2P fan-out with replicas on different GPUs (NVLink peer stores; plain
    pointers in one process, peer access enabled by the library)."""
    R = min(NGPU, 4)
    inv, seed = replicated_inventory(43)
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, _ = oracle_of(inv, seed)
    L = idx.partitions[0].length
    bases = [torch.empty(L, dtype=torch.uint8, device=f"cuda:{r}") for r in range(R)]
    sigs = [torch.zeros(2 * R, dtype=torch.int32, device=f"cuda:{r}") for r in range(R)]
    comms = [sllm.Comm.peers(R, r, r, [b.data_ptr() for b in bases], [s.data_ptr() for s in sigs], 30000)
             for r in range(R)]
    cfg = sllm.LoadConfig(chunk_bytes=1 << 20, mode=mode, fanout="p2p")
    for epoch in range(2):
        for r, b in enumerate(bases):
            b.fill_(0x3C + epoch)
            torch.cuda.synchronize(r)
        results = [sllm.load_start(idx, bufs, {0: r}, cfg, {0: bases[r]}, None, None, comms[r]) for r in range(R)]
        reports = [res.wait() for res in results]
        for r in range(R):
            assert np.array_equal(bases[r].cpu().numpy(), oparts[0]), (epoch, r)
            assert results[r].block_checksums(0).tolist() == lay.checksums[0]
        assert sum(rep["transferred_bytes"] for rep in reports) == L
        del results
    for c in comms:
        c.free()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _proc_worker(rank, world, port, kind, mode, q):
    """One process per GPU: NCCL communicator from the process group (bcast / allgather) or a
    peer group over CUDA IPC (p2p)."""
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(rank)
        inv, seed = replicated_inventory(47)
        idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20, gpu_of={0: rank})
        lay, oparts, _ = oracle_of(inv, seed)
        L = idx.partitions[0].length
        base = torch.full((L,), 0x5A, dtype=torch.uint8, device=f"cuda:{rank}")
        torch.cuda.synchronize()
        comm = sllm.Comm.peers_from_process_group(base, timeout_ms=30000) if kind == "p2p" \
            else sllm.Comm.from_process_group(rank)
        dist.barrier()
        ok, moved = True, 0
        for _ in range(2):
            res = sllm.load_start(idx, bufs, {0: rank}, sllm.LoadConfig(chunk_bytes=2 << 20, mode=mode, fanout=kind),
                                  {0: base}, None, None, comm)
            rep = res.wait()
            ok &= bool(np.array_equal(base.cpu().numpy(), oparts[0]))
            ok &= res.block_checksums(0).tolist() == lay.checksums[0]
            moved = rep["transferred_bytes"]
            del res
        t = torch.tensor([moved], dtype=torch.int64)
        dist.all_reduce(t)
        ok &= int(t.item()) == L
        comm.free()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, ""))
    except Exception as ex:  # noqa: BLE001
        import traceback
        q.put((rank, False, traceback.format_exc()))


@multi
@pytest.mark.parametrize("kind", ["bcast", "allgather", "p2p"])
@pytest.mark.parametrize("mode", ["ce", "zerocopy"])
def test_fanout_one_process_per_gpu(kind, mode):
    import torch.multiprocessing as mp
    R = min(NGPU, 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_proc_worker, args=(r, R, port, kind, mode, q)) for r in range(R)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in out), out


# ---- NVLS multicast fan-out ---------------------------------------
def _nvls_or_skip(gpus, nbytes):
    """The group, or a skip naming why the platform cannot create multicast objects (the
    library's clean SLLM_E_INVALID; this build's 1-GPU VMs, profiles/r01/probe_nvls.txt)."""
    try:
        return sllm.Comm.nvls(gpus, nbytes, timeout_ms=30000)
    except sllm.SllmError as ex:
        assert ex.status == 1, ex          # capability failure is SLLM_E_INVALID, nothing else
        pytest.skip(f"NVLS multicast not available on this platform: {ex}")


def test_nvls_capability_probe_is_clean():
    """Creating an NVLS group either works or fails with SLLM_E_INVALID naming the driver
    call -- never a crash or a sticky CUDA error: a plain load still runs afterwards."""
    try:
        comms = sllm.Comm.nvls([0], 1 << 20)
        for c in comms:
            c.free()
    except sllm.SllmError as ex:
        assert ex.status == 1 and "NVLS" in str(ex)
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, _ = oracle_of(inv, seed)
    res = sllm.load(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20))
    assert np.array_equal(res._keep[3][0].cpu().numpy(), oparts[0])


def test_nvls_fanout_needs_an_nvls_group():
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    L = idx.partitions[0].length
    base = torch.empty(L, dtype=torch.uint8, device="cuda")
    sig = torch.zeros(2, dtype=torch.int32, device="cuda")
    peers = sllm.Comm.peers(1, 0, 0, [base.data_ptr()], [sig.data_ptr()])
    with pytest.raises(sllm.SllmError) as ex:    # a P2P peer group has no multicast address
        sllm.load_start(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20, fanout="nvls"), {0: base}, None, None,
                        peers)
    assert ex.value.status == 1 and "NVLS" in str(ex.value)
    peers.free()


@pytest.mark.parametrize("mode", ["ce", "zerocopy"])
def test_nvls_fanout_every_replica_bit_exact(mode):
    """All visible GPUs (up to 8) in one NVLS group driven by this process: rank r moves its
    slice over PCIe and its loading kernel stores every vector once through the multicast
    address; every replica ends equal to P_0, every block checksum to the oracle's, and the
    group moved each byte over PCIe once."""
    R = min(NGPU, 8)
    inv, seed = replicated_inventory(53)
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, _ = oracle_of(inv, seed)
    L = idx.partitions[0].length
    comms = _nvls_or_skip(list(range(R)), L)
    reps = [c.replica() for c in comms]
    assert all(r.numel() >= L for r in reps)
    cfg = sllm.LoadConfig(chunk_bytes=1 << 20, mode=mode, fanout="nvls")
    for epoch in range(2):
        for r in range(R):
            reps[r].fill_(0x6B + epoch)
            torch.cuda.synchronize(r)
        results = [sllm.load_start(idx, bufs, {0: r}, cfg, {0: reps[r]}, None, None, comms[r]) for r in range(R)]
        reports = [res.wait() for res in results]
        for r in range(R):
            assert np.array_equal(reps[r][:L].cpu().numpy(), oparts[0]), (epoch, r)
            assert results[r].block_checksums(0).tolist() == lay.checksums[0]
            assert reports[r]["fanout_bytes"] == L - reports[r]["transferred_bytes"]
        assert sum(rep["transferred_bytes"] for rep in reports) == L
        del results
    for c in comms:
        c.free()


def test_bench_nvls_fails_loudly_or_runs():
    """`bench.py --fanout nvls` either measures the multicast group or exits 2 naming why the
    platform has no NVLS -- never a silent fallback to another fan-out."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--fanout", "nvls", "--config", "toy",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=root)
    if out.returncode == 0:
        line = json.loads(out.stdout.strip().splitlines()[-1])
        assert line["replica0_equals_source"] and line["config"]["fanout"] == "nvls"
    else:
        assert out.returncode == 2 and "NVLS unavailable" in out.stderr, out.stderr[-2000:]
