"""Multi-process (world_size 2-3, gloo, CPU) coverage of the N>1 host logic.

* The NCCL unique id of the replicated path is created by the library on rank 0 and
  distributed through torch.distributed (Comm.from_process_group's exchange).
* The replicated fan-out schedule the library executes (sllm_replica_round): every rank
  moves only its own slice "over PCIe" (a host copy here), then the rounds are replayed
  with gloo broadcasts in place of ncclBroadcast.  Every rank must end with P_0 exactly
  (O9(c)) and every partition byte must have crossed "PCIe" exactly once in total.
* The sharded path: rank r picks partition r of a shared index and loads it with the
  oracle; the union over ranks covers every tensor exactly once.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker_fanout(rank, world, port, chunk, q):
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        _init(rank, world, port)
        import paper_2401_14351_b200 as sllm
        from oracle import layout as olayout
        from synth import models, payload
        # NCCL unique id from the library on rank 0, exchanged over the process group
        obj = [sllm.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        assert len(obj[0]) == 128 and all(i == ids[0] for i in ids)
        # one replicated partition (the oracle's bytes are the expected result)
        rng = np.random.default_rng(7)
        inv = [models.TensorSpec(t.name, 0, t.dtype, t.shape)
               for t in models.random_inventory(rng, 300, 1, 6 << 20)]
        tensors = [(t.name, 0, t.dtype, t.shape, payload.payload_bytes(3, e, t.nbytes)) for e, t in enumerate(inv)]
        lay, parts = olayout.convert(tensors, 4096, 1 << 16)
        P0 = parts[0]
        L = P0.size
        buf = torch.zeros(L, dtype=torch.uint8)
        lo, hi = sllm.replica_slices(L, chunk, world)[rank]
        buf[lo:hi] = torch.from_numpy(P0[lo:hi])          # this rank's PCIe slice
        pcie = torch.tensor([hi - lo], dtype=torch.int64)
        for rnd in sllm.replica_schedule(L, chunk, world):
            for src, (a, b) in enumerate(rnd):
                if b > a:
                    view = buf[a:b]
                    dist.broadcast(view, src=src)         # stands in for ncclBroadcast
        assert np.array_equal(buf.numpy(), P0)
        dist.all_reduce(pcie)
        assert int(pcie.item()) == L                      # each byte crossed PCIe once in total
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as ex:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))


def _worker_allgather(rank, world, port, chunk, q):
    """fanout="allgather": rank r moves chunks r, r+N, ... "over PCIe"; every full round is
    one in-place all-gather (gloo all_gather into views of the replica stands in for
    ncclAllGather), the ragged last round per-owner broadcasts."""
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        _init(rank, world, port)
        import paper_2401_14351_b200 as sllm
        from oracle import layout as olayout
        from synth import models, payload
        rng = np.random.default_rng(11)
        inv = [models.TensorSpec(t.name, 0, t.dtype, t.shape)
               for t in models.random_inventory(rng, 300, 1, 6 << 20)]
        tensors = [(t.name, 0, t.dtype, t.shape, payload.payload_bytes(5, e, t.nbytes)) for e, t in enumerate(inv)]
        lay, parts = olayout.convert(tensors, 4096, 1 << 16)
        P0 = parts[0]
        L = P0.size
        buf = torch.zeros(L, dtype=torch.uint8)
        pcie = 0
        for full, rnd in sllm.allgather_schedule(L, chunk, world):
            a, b = rnd[rank]
            if b > a:                                     # this rank's own chunk of the round
                buf[a:b] = torch.from_numpy(P0[a:b])
                pcie += b - a
            if full:
                lo = rnd[0][0]
                views = [buf[lo + q * chunk:lo + (q + 1) * chunk] for q in range(world)]
                dist.all_gather(views, buf[a:b].clone())  # stands in for the in-place ncclAllGather
            else:
                for src, (x, y) in enumerate(rnd):
                    if y > x:
                        dist.broadcast(buf[x:y], src=src)
        assert np.array_equal(buf.numpy(), P0)
        t = torch.tensor([pcie], dtype=torch.int64)
        dist.all_reduce(t)
        assert int(t.item()) == L                         # each byte crossed PCIe once in total
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))


def _worker_sharded(rank, world, port, q):
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        _init(rank, world, port)
        import paper_2401_14351_b200 as sllm
        from oracle import loader as oloader
        from paper_2401_14351_b200 import workloads
        from synth import models, payload
        inv = models.llama2(192, 2, 384, 48, vocab=516, tp=world)
        idx = workloads.plan_inventory(inv)
        blob = [idx.serialize() if rank == 0 else None]   # the index travels, partitions do not
        dist.broadcast_object_list(blob, src=0)
        mine = sllm.Index.from_bytes(blob[0])
        p = rank
        part = np.zeros(mine.partitions[p].length, np.uint8)
        names = []
        for e, t in enumerate(mine.tensors):
            if t.partition == p:
                part[t.offset:t.offset + t.nbytes] = payload.payload_bytes(0, e, t.nbytes)
                names.append(t.name)
        ptrs = [part.ctypes.data if i == p else None for i in range(world)]
        mine.seal(ptrs)                                    # this rank's block table only
        res = oloader.load(mine.serialize(), {mine.partitions[i].device: (part if i == p else
                                              np.zeros(mine.partitions[i].length, np.uint8)) for i in range(world)},
                           verify=False)
        for n in names:
            e = mine.find(n)
            assert res.tensors[n].tobytes() == payload.payload_bytes(0, e, mine.tensors[e].nbytes).tobytes()
        allnames = [None] * world
        dist.all_gather_object(allnames, names)
        flat = [n for ns in allnames for n in ns]
        assert sorted(flat) == sorted(t.name for t in inv) and len(flat) == len(set(flat))
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))


def _run(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert out[r] == "ok", out[r]


@pytest.mark.parametrize("world,chunk", [(2, 1 << 16), (3, 1 << 16), (2, 3 << 16)])
def test_replicated_fanout_schedule_gloo(world, chunk):
    _run(_worker_fanout, world, chunk)


@pytest.mark.parametrize("world,chunk", [(2, 1 << 16), (3, 1 << 16), (3, 3 << 16)])
def test_allgather_fanout_schedule_gloo(world, chunk):
    _run(_worker_allgather, world, chunk)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_partition_per_rank_gloo(world):
    _run(_worker_sharded, world)


def test_schedule_properties():
    import paper_2401_14351_b200 as sllm
    for L, C, N in [(13_594_624, 1 << 20, 8), (100 << 16, 1 << 16, 3), (1 << 16, 1 << 16, 4), (59_949_920_256, 64 << 20, 8)]:
        rounds = sllm.replica_schedule(L, C, N)
        covered = sorted((a, b) for rnd in rounds for (a, b) in rnd if b > a)
        pos = 0
        for a, b in covered:
            assert a == pos and b - a <= C
            pos = b
        assert pos == L
        assert len(rounds) == max(-(-(b - a) // C) for a, b in sllm.replica_slices(L, C, N))


def test_allgather_schedule_properties():
    """Round-robin ownership: chunk k -> rank k % N; a round is N adjacent chunks, full iff
    all N are whole; the rounds cover [0, L) exactly once."""
    import paper_2401_14351_b200 as sllm
    for L, C, N in [(13_594_624, 1 << 20, 8), (100 << 16, 1 << 16, 3), (1 << 16, 1 << 16, 4), (99 << 16, 1 << 16, 3),
                    (59_949_920_256, 64 << 20, 8), (5 << 16, 1 << 16, 1)]:
        rounds = sllm.allgather_schedule(L, C, N)
        nch = -(-L // C)
        assert len(rounds) == -(-nch // N)
        pos = 0
        for r, (full, rnd) in enumerate(rounds):
            for q, (a, b) in enumerate(rnd):
                k = r * N + q
                if k < nch:
                    assert (a, b) == (k * C, min((k + 1) * C, L)) and a == pos
                    pos = b
                else:
                    assert a == b
            assert full == all(b - a == C for a, b in rnd)
            if r + 1 < len(rounds):
                assert full
        assert pos == L


def test_allgather_round_errors():
    import ctypes as C
    import paper_2401_14351_b200 as sllm
    from paper_2401_14351_b200 import _abi
    arr = (C.c_uint64 * 6)()
    n, full = C.c_uint64(), C.c_int32()
    assert sllm.lib().sllm_allgather_round(10 << 16, 1 << 16, 3, 0, arr, C.byref(n), C.byref(full)) == _abi.OK
    assert n.value == 4 and full.value == 1
    assert sllm.lib().sllm_allgather_round(10 << 16, 1 << 16, 3, 3, arr, None, C.byref(full)) == _abi.OK
    assert full.value == 0 and [arr[i] for i in range(6)] == [9 << 16, 10 << 16, 0, 0, 0, 0]
    assert sllm.lib().sllm_allgather_round(10 << 16, 1 << 16, 3, 4, arr, None, None) == _abi.E_LOOKUP
    assert sllm.lib().sllm_allgather_round(10 << 16, 0, 3, 0, arr, None, None) == _abi.E_INVALID
    assert sllm.lib().sllm_allgather_round(10 << 16, 1 << 16, 0, 0, arr, None, None) == _abi.E_INVALID


def test_fanout_unit():
    """The NCCL fan-outs slice and run rounds in whole >= 64 MiB windows of chunks (one
    copy + one grouped collective per round); P2P / none keep the chunk.  The
    schedule functions replayed above are the ones the loader calls with this unit."""
    import paper_2401_14351_b200 as sllm
    M = 1 << 20
    for C, U in [(1 * M, 64 * M), (16 * M, 64 * M), (64 * M, 64 * M), (3 * M, 63 * M), (128 * M, 128 * M),
                 (1 << 16, 64 * M)]:
        assert sllm.fanout_unit(C, "bcast") == U and sllm.fanout_unit(C, "allgather") == U
        assert sllm.fanout_unit(C, "p2p") == C and sllm.fanout_unit(C, "none") == C
    # OPT-30B over 8 ranks at 16 MiB chunks: 894 units, 112 rounds instead of 447 per-chunk rounds
    L = 59_949_969_408
    U = sllm.fanout_unit(16 * M, "bcast")
    assert len(sllm.replica_schedule(L, U, 8)) == 112 and len(sllm.replica_schedule(L, 16 * M, 8)) == 447
