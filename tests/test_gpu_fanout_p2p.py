"""GPU parity of the fused P2P fan-out (SLLM_FANOUT_P2P).

A replicated checkpoint (one partition) is loaded by a group of R ranks: rank r moves
only its slice over PCIe and its loading kernel stores every vector into all R replicas;
device-side release/acquire signals order the peers' stores before each rank verifies
what it received.  Only one GPU is available here, so the "peers" are R replicas on the
same GPU in one process (plain pointers; the in-process ranks order each other with CUDA
events, so no kernel waits for another rank's kernel).  The one-process-per-rank wiring
(CUDA IPC handles exchanged over a gloo group, flags written by the peers' kernels) runs on
one GPU with the flags waited for on the host (SLLM_PEER_WAIT=host); its device-side wait
kernels need one GPU per rank -- kernels that spin on another rank's flag must not share a
GPU.  Every replica must equal the oracle's partition P_0
byte for byte (O9(c)) and every block checksum must equal the oracle's (O9(d)).
"""
import os
import socket

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


def oracle_of(inv, seed, A=4096, B=1 << 20):
    payloads = [payload.payload_bytes(seed, e, t.nbytes) for e, t in enumerate(inv)]
    lay, parts = olayout.convert([(t.name, t.device, t.dtype, t.shape, p) for t, p in zip(inv, payloads)], A, B)
    return lay, parts, payloads


def group(R, L, timeout_ms=20000):
    bases = [torch.empty(L, dtype=torch.uint8, device="cuda") for _ in range(R)]
    sigs = [torch.zeros(2 * R, dtype=torch.int32, device="cuda") for _ in range(R)]
    comms = [sllm.Comm.peers(R, r, 0, [b.data_ptr() for b in bases], [s.data_ptr() for s in sigs], timeout_ms)
             for r in range(R)]
    return bases, sigs, comms


def start_all(idx, bufs, cfg, bases, comms):
    return [sllm.load_start(idx, bufs, {0: 0}, cfg, {0: bases[r]}, None, None, comms[r]) for r in range(len(comms))]


@pytest.mark.parametrize("R", [1, 2, 3, 4])
@pytest.mark.parametrize("mode", ["ce", "zerocopy"])
@pytest.mark.parametrize("chunk", [1 << 20, 2 << 20])
def test_p2p_fanout_same_gpu(R, mode, chunk):
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, payloads = oracle_of(inv, seed)
    L = idx.partitions[0].length
    slices = sllm.replica_slices(L, chunk, R)
    bases, sigs, comms = group(R, L)
    cfg = sllm.LoadConfig(chunk_bytes=chunk, mode=mode, fanout="p2p")
    for epoch in range(3):  # the signal epochs advance per collective load
        for b in bases:
            b.fill_(0xA5)
        torch.cuda.synchronize()
        results = start_all(idx, bufs, cfg, bases, comms)
        reports = [res.wait() for res in results]
        for r, (res, rep) in enumerate(zip(results, reports)):
            assert np.array_equal(bases[r].cpu().numpy(), oparts[0]), (r, epoch)
            assert res.block_checksums(0).tolist() == lay.checksums[0]
            lo, hi = slices[r]
            assert rep["transferred_bytes"] == hi - lo          # each byte crosses "PCIe" once
            assert rep["fanout_bytes"] == L - (hi - lo)
            # in-process ranks are ordered by CUDA events: the slice's one loading launch
            # (a toy slice is one copy window) + K4 on each received range, no signal / wait kernels
            assert rep["kernel_launches"] == (1 if hi > lo else 0) + (lo > 0) + (hi < L), rep["kernel_launches"]
            for e in (0, len(inv) - 2, len(inv) - 1):           # views of this replica
                t = inv[e]
                got = res.tensors[t.name].reshape(-1).view(torch.uint8).cpu().numpy()
                assert np.array_equal(got, payloads[e])
        assert sum(rep["transferred_bytes"] for rep in reports) == L
        del results
    for c in comms:
        c.free()


@pytest.mark.parametrize("mode", ["ce", "zerocopy"])
def test_p2p_fault_reported_by_every_rank(mode):
    """A flipped source byte in rank 1's slice: rank 1 catches it reading the host, every
    other rank catches it in what arrived over the peer stores -- same (partition, block)."""
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    L = idx.partitions[0].length
    R, chunk = 3, 1 << 20
    lo, hi = sllm.replica_slices(L, chunk, R)[1]
    pos = lo + (hi - lo) // 2 + 12345
    src = bufs[0].numpy()
    src[pos] ^= 0x40
    try:
        bases, sigs, comms = group(R, L)
        cfg = sllm.LoadConfig(chunk_bytes=chunk, mode=mode, fanout="p2p")
        results = start_all(idx, bufs, cfg, bases, comms)
        for res in results:
            with pytest.raises(sllm.SllmError) as ex:
                res.wait()
            assert ex.value.status == 9
            assert res.report["bad_partition"] == 0 and res.report["bad_block"] == pos >> 20
        del results
        for c in comms:
            c.free()
    finally:
        src[pos] ^= 0x40


def test_p2p_missing_peer_times_out():
    """A peer that never loads: the waiting rank fails with SLLM_E_PEER after the group's
    timeout instead of hanging the GPU."""
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    L = idx.partitions[0].length
    bases, sigs, comms = group(2, L, timeout_ms=1500)
    res = sllm.load_start(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20, mode="zerocopy", fanout="p2p"),
                          {0: bases[0]}, None, None, comms[0])
    with pytest.raises(sllm.SllmError) as ex:
        res.wait()
    assert ex.value.status == 12
    del res
    for c in comms:
        c.free()


def test_p2p_rejects_bad_setup():
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    L = idx.partitions[0].length
    bases, sigs, comms = group(2, L)
    other = torch.empty(L, dtype=torch.uint8, device="cuda")
    cfg = sllm.LoadConfig(chunk_bytes=1 << 20, mode="ce", fanout="p2p")
    with pytest.raises(sllm.SllmError) as ex:   # dst must be the rank's own replica
        sllm.load_start(idx, bufs, {0: 0}, cfg, {0: other}, None, None, comms[0])
    assert ex.value.status == 1
    _, per_tensor = sllm.allocate(idx, {0: 0}, scatter=True)
    with pytest.raises(sllm.SllmError):         # scatter modes have no replica base
        sllm.load_start(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20, mode="scatter_ce", fanout="p2p"),
                        {0: bases[0]}, per_tensor, None, comms[0])
    nccl = sllm.Comm.init_rank(sllm.Comm.unique_id(), 1, 0, 0)
    with pytest.raises(sllm.SllmError):         # a peer group is not an NCCL communicator and vice versa
        sllm.load_start(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20, fanout="bcast"),
                        {0: bases[0]}, None, None, comms[0])
    with pytest.raises(sllm.SllmError):
        sllm.load_start(idx, bufs, {0: 0}, cfg, {0: bases[0]}, None, None, nccl)
    nccl.free()
    for c in comms:
        c.free()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ipc_worker(rank, world, port, mode, wait, q):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SLLM_PEER_WAIT=wait)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(rank if wait == "device" else 0)
        inv, seed = models.model_inventory("toy")
        idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
        lay, oparts, _ = oracle_of(inv, seed)
        L = idx.partitions[0].length
        base = torch.empty(L, dtype=torch.uint8, device="cuda")
        comm = sllm.Comm.peers_from_process_group(base, timeout_ms=30000)
        ok = True
        for it in range(3):  # back to back: the done/ready signals order the epochs, no barrier
            if it == 0:
                base.fill_(0x5A)
                torch.cuda.synchronize()
                dist.barrier()
            res = sllm.load_start(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20, mode=mode, fanout="p2p"),
                                  {0: base}, None, None, comm)
            rep = res.wait()
            ok &= bool(np.array_equal(base.cpu().numpy(), oparts[0]))
            ok &= res.block_checksums(0).tolist() == lay.checksums[0]
            ok &= rep["fanout_bytes"] == L - rep["transferred_bytes"]
            del res
        comm.free()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, ""))
    except Exception as ex:  # noqa: BLE001
        q.put((rank, False, repr(ex)))


def _ipc_absent_peer_worker(rank, world, port, q):
    """Rank 1 joins the group but never loads: rank 0's host-polled wait must fail with
    SLLM_E_PEER after the group timeout (and not hang)."""
    try:
        import time
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SLLM_PEER_WAIT="host")
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        inv, seed = models.model_inventory("toy")
        idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
        base = torch.empty(idx.partitions[0].length, dtype=torch.uint8, device="cuda")
        comm = sllm.Comm.peers_from_process_group(base, timeout_ms=1500)
        ok, msg = True, ""
        if rank == 0:
            t0 = time.perf_counter()
            res = sllm.load_start(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20, mode="ce", fanout="p2p"),
                                  {0: base}, None, None, comm)
            try:
                res.wait()
                ok, msg = False, "load succeeded without its peer"
            except sllm.SllmError as ex:
                dt = time.perf_counter() - t0
                ok = ex.status == 12 and 1.0 < dt < 30.0
                msg = f"status {ex.status} after {dt:.2f} s: {ex}"
            del res
        dist.barrier()  # rank 1 keeps its replica mapped until rank 0 is done
        comm.free()
        dist.destroy_process_group()
        q.put((rank, ok, msg))
    except Exception as ex:  # noqa: BLE001
        q.put((rank, False, repr(ex)))


def test_p2p_two_processes_absent_peer_host_wait_times_out():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_absent_peer_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in out), out


@pytest.mark.parametrize("wait", ["host", "device"])
@pytest.mark.parametrize("mode", ["ce", "zerocopy"])
def test_p2p_fanout_two_processes_ipc(mode, wait):
    """Two processes, one replica each, peers mapped with CUDA IPC (the real multi-process
    wiring of bench.py --fanout p2p).  wait=host: both ranks on GPU 0, flags polled by the
    load workers; wait=device: the device-side wait kernels, one GPU per rank."""
    if wait == "device" and torch.cuda.device_count() < 2:
        pytest.skip("device-side flag waits of one process per rank need one GPU per rank")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, mode, wait, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in out), out


@pytest.mark.parametrize("R,mode,chunk", [(2, "ce", 1 << 20), (3, "zerocopy", 1 << 20), (3, "ce", 2 << 20)])
def test_p2p_from_files_reads_each_byte_once(tmp_path, R, mode, chunk):
    """Replicated checkpoint straight from its partition file (file tier + fused fan-out):
    rank r reads only its slice from storage -- the group reads every byte once -- and every
    replica still ends equal to P_0."""
    inv, seed = models.model_inventory("toy")
    payloads = [payload.payload_bytes(seed, e, t.nbytes) for e, t in enumerate(inv)]
    sllm.convert([(t.name, t.device, t.dtype, t.shape, p.ctypes.data) for t, p in zip(inv, payloads)],
                 str(tmp_path), 4096, 1 << 20, "toy")
    lay, oparts, _ = oracle_of(inv, seed)
    idx = sllm.Index.open(str(tmp_path / "index.bin"))
    L = idx.partitions[0].length
    slices = sllm.replica_slices(L, chunk, R)
    bases, sigs, comms = group(R, L)
    cfg = sllm.LoadConfig(chunk_bytes=chunk, mode=mode, fanout="p2p")
    for _ in range(2):
        for b in bases:
            b.fill_(0x3C)
        torch.cuda.synchronize()
        # (all ranks share this thread's stream: ordering them on it would serialise the group,
        # so the caller-stream gate is off -- each process of a real group has its own stream)
        results = [sllm.load_files(idx, str(tmp_path), {0: 0}, cfg, io_threads=2, wait=False, stream_of_caller=False,
                                   bases={0: bases[r]}, per_tensor={}, comm=comms[r]) for r in range(R)]
        reports = [res.wait() for res in results]
        for r, rep in enumerate(reports):
            lo, hi = slices[r]
            assert rep["storage_bytes"] == hi - lo
            assert np.array_equal(bases[r].cpu().numpy(), oparts[0]), r
            assert results[r].block_checksums(0).tolist() == lay.checksums[0]
        assert sum(rep["storage_bytes"] for rep in reports) == L
        del results
    for c in comms:
        c.free()


def test_bcast_from_files_single_rank(tmp_path):
    inv, seed = models.model_inventory("toy")
    payloads = [payload.payload_bytes(seed, e, t.nbytes) for e, t in enumerate(inv)]
    sllm.convert([(t.name, t.device, t.dtype, t.shape, p.ctypes.data) for t, p in zip(inv, payloads)],
                 str(tmp_path), 4096, 1 << 20, "toy")
    lay, oparts, _ = oracle_of(inv, seed)
    idx = sllm.Index.open(str(tmp_path / "index.bin"))
    comm = sllm.Comm.init_rank(sllm.Comm.unique_id(), 1, 0, 0)
    res = sllm.load_files(idx, str(tmp_path), {0: 0}, sllm.LoadConfig(chunk_bytes=2 << 20, fanout="bcast"),
                          comm=comm)
    assert res.report["storage_bytes"] == idx.partitions[0].length
    assert np.array_equal(res._keep[3][0].cpu().numpy(), oparts[0])
    del res
    comm.free()
