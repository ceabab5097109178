"""Small loads in every mode / engine / fan-out for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck), each checked byte-exact against the CPU oracle:

    compute-sanitizer --tool memcheck --error-exitcode 99 python tests/sanitize_gpu.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import paper_2401_14351_b200 as sllm
    from paper_2401_14351_b200 import workloads
    from oracle import layout as olayout
    from synth import models, payload

    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    pl = [payload.payload_bytes(seed, e, t.nbytes) for e, t in enumerate(inv)]
    lay, parts = olayout.convert([(t.name, t.device, t.dtype, t.shape, p) for t, p in zip(inv, pl)], 4096, 1 << 20)
    n = 0
    only = os.environ.get("SANITIZE_ONLY")  # e.g. "zerocopy:tma" -- one load, nothing else
    if only == "ring":  # the ~0.5 GB scatter loads only: every CTA wraps its stage ring many times
        mid = models.llama2(1024, 12, 4096, 1024, vocab=32000)
        midx, mbufs = workloads.build_pinned(mid, 9, 4096, 1 << 20)
        for engine in ("tma", "tma_store"):
            for mode in ("scatter_ce", "scatter_zc", "ce", "zerocopy"):
                res = sllm.load(midx, mbufs, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20, mode=mode, engine=engine))
                assert np.array_equal(res.block_checksums(0), midx.block_checksums(0)), (engine, mode)
                del res
        # P2P fan-out group of 2 on this GPU: every vector also stored into the peer replica
        L = midx.partitions[0].length
        bases = [torch.empty(L, dtype=torch.uint8, device="cuda") for _ in range(2)]
        sigs = [torch.zeros(4, dtype=torch.int32, device="cuda") for _ in range(2)]
        comms = [sllm.Comm.peers(2, r, 0, [b.data_ptr() for b in bases], [s.data_ptr() for s in sigs], 60000)
                 for r in range(2)]
        for mode in ("ce", "zerocopy"):
            cfg = sllm.LoadConfig(chunk_bytes=1 << 20, mode=mode, fanout="p2p")
            rs = [sllm.load_start(midx, mbufs, {0: 0}, cfg, {0: bases[r]}, None, None, comms[r]) for r in range(2)]
            for r in rs:
                r.wait()
            assert torch.equal(bases[0], bases[1])
            del rs
        for c in comms:
            c.free()
        print("sanitize_gpu ok: ring-wrap loads (2 engines x 4 modes, P2P ce/zerocopy)")
        return
    for engine in ("tma", "ldg", "tma_store"):
        for mode in ("ce", "zerocopy", "scatter_ce", "scatter_zc"):
            if only and only != f"{mode}:{engine}":
                continue
            res = sllm.load(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=2 << 20, mode=mode, engine=engine))
            for e, t in enumerate(inv):
                got = res.tensors[t.name].reshape(-1).view(torch.uint8).cpu().numpy()
                assert np.array_equal(got, pl[e]), (engine, mode, t.name)
            assert res.block_checksums(0).tolist() == lay.checksums[0]
            n += 1
            del res
    if only:
        print(f"sanitize_gpu ok: {n} load ({only})")
        return
    # P2P fan-out, 2 ranks on this GPU
    L = idx.partitions[0].length
    bases = [torch.empty(L, dtype=torch.uint8, device="cuda") for _ in range(2)]
    sigs = [torch.zeros(4, dtype=torch.int32, device="cuda") for _ in range(2)]
    comms = [sllm.Comm.peers(2, r, 0, [b.data_ptr() for b in bases], [s.data_ptr() for s in sigs], 60000)
             for r in range(2)]
    for mode in ("ce", "zerocopy"):
        cfg = sllm.LoadConfig(chunk_bytes=1 << 20, mode=mode, fanout="p2p")
        rs = [sllm.load_start(idx, bufs, {0: 0}, cfg, {0: bases[r]}, None, None, comms[r]) for r in range(2)]
        for r in rs:
            r.wait()
        for b in bases:
            assert np.array_equal(b.cpu().numpy(), parts[0])
        n += 2
        del rs
    for c in comms:
        c.free()
    # NCCL fan-outs with a 1-rank communicator (grouped broadcasts / in-place all-gathers)
    comm = sllm.Comm.init_rank(sllm.Comm.unique_id(), 1, 0, 0)
    for fanout in ("bcast", "allgather"):
        for mode in ("ce", "zerocopy"):
            res = sllm.load(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=2 << 20, mode=mode, fanout=fanout), comm=comm)
            assert np.array_equal(res._keep[3][0].cpu().numpy(), parts[0]), (fanout, mode)
            n += 1
            del res
    comm.free()
    # a ~0.5 GB checkpoint with 1 MiB chunks: several SCATTER_CE staging windows (the window
    # plan) and the granule-bounded segment search over hundreds of segments
    mid = models.llama2(1024, 12, 4096, 1024, vocab=32000)
    midx, mbufs = workloads.build_pinned(mid, 9, 4096, 1 << 20)
    for mode in ("scatter_ce", "scatter_zc"):
        res = sllm.load(midx, mbufs, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20, mode=mode))
        assert np.array_equal(res.block_checksums(0), midx.block_checksums(0)), mode
        for e in (0, len(mid) // 2, len(mid) - 1):
            t = mid[e]
            got = res.tensors[t.name].reshape(-1).view(torch.uint8).cpu().numpy()
            assert np.array_equal(got, payload.payload_bytes(9, e, t.nbytes)), (mode, t.name)
        n += 1
        del res
    for b in mbufs.values():
        b.free()
    # standalone K3 (device-resident image -> per-tensor buffers)
    img = torch.from_numpy(parts[0].copy()).cuda()
    _, per = sllm.allocate(idx, {0: 0}, scatter=True)
    sllm.materialise_device(idx, 0, img.data_ptr(), per)
    for e, t in enumerate(inv):
        assert np.array_equal(per[t.name].reshape(-1).view(torch.uint8).cpu().numpy(), pl[e]), t.name
    del img, per
    # standalone kernels
    src = torch.from_numpy(parts[0].copy()).cuda()
    out = torch.zeros(idx.partitions[0].n_blocks, dtype=torch.int64, device="cuda")
    sllm.block_checksums_device(src.data_ptr(), L, 1 << 20, out.data_ptr())
    torch.cuda.synchronize()
    assert [int(v) & (2**64 - 1) for v in out.cpu().tolist()] == lay.checksums[0]
    print(f"sanitize_gpu ok: {n} loads + standalone K3 + standalone K4")


if __name__ == "__main__":
    main()
