"""GPU parity: the CUDA load path (through the C ABI) against the CPU oracle.

Every comparison is exact (bytes / integers): loaded partition bytes, per-tensor bytes,
device-computed block checksums and fault reports, for every mode (copy engine +
checksum kernel, zero-copy kernel, staging + scatter kernel, zero-copy scatter), chunk
sizes spanning several tiles with a ragged tail, 1-4 streams, alignment 16 and 4096.
Expected values come only from oracle/ (and the synth payload definition)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2401_14351_b200 as sllm  # noqa: E402
from paper_2401_14351_b200 import workloads  # noqa: E402
from oracle import fletcher, index as oindex, layout as olayout, loader as oloader  # noqa: E402
from synth import models, payload  # noqa: E402

MODES = ["ce", "zerocopy", "scatter_ce", "scatter_zc"]


def oracle_of(inv, seed, A, B):
    payloads = [payload.payload_bytes(seed, e, t.nbytes) for e, t in enumerate(inv)]
    lay, parts = olayout.convert([(t.name, t.device, t.dtype, t.shape, p) for t, p in zip(inv, payloads)], A, B)
    return lay, parts, payloads


def check_against_oracle(res, idx, inv, lay, oparts, payloads, parts_loaded, cfg):
    # tensors: every byte (Q13: byte equality, never float ==)
    for e, t in enumerate(inv):
        pidx = lay.devices().index(t.device)
        if pidx not in parts_loaded:
            continue
        got = res.tensors[t.name]
        got_b = got.contiguous().view(torch.uint8).reshape(-1).cpu().numpy() if got.dim() else \
            got.reshape(1).view(torch.uint8).cpu().numpy()
        assert np.array_equal(got_b, payloads[e]), t.name
    if not cfg.scatter:   # whole partitions, padding included (O9(a))
        for p in parts_loaded:
            d = lay.devices()[p]
            base = res._keep[3][p]
            assert np.array_equal(base.cpu().numpy(), oparts[d]), f"partition {p}"
    if cfg.verify:        # device checksums == oracle (O9(d))
        for p in parts_loaded:
            d = lay.devices()[p]
            assert res.block_checksums(p).tolist() == lay.checksums[d]


@pytest.mark.parametrize("engine", ["tma", "ldg", "tma_store"])
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("chunk,streams", [(1 << 20, 1), (2 << 20, 2), (4 << 20, 3), (16 << 20, 2)])
def test_toy_all_modes(mode, chunk, streams, engine):
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, payloads = oracle_of(inv, seed, 4096, 1 << 20)
    cfg = sllm.LoadConfig(chunk_bytes=chunk, n_streams=streams, mode=mode, engine=engine)
    res = sllm.load(idx, bufs, {0: 0}, cfg)
    rep = res.report
    assert rep["bad_partition"] == -1 and rep["payload_bytes"] == 13_569_860
    assert rep["transferred_bytes"] == 13_594_624
    assert rep["chunks"] == -(-13_594_624 // chunk)
    check_against_oracle(res, idx, inv, lay, oparts, payloads, [0], cfg)


@pytest.mark.parametrize("engine", ["tma", "ldg", "tma_store"])
@pytest.mark.parametrize("mode", MODES)
def test_toy_align16_and_small_blocks(mode, engine):
    inv, seed = models.model_inventory("toy")
    for A, B, C in [(16, 1 << 20, 1 << 20), (16, 4096, 1 << 20), (256, 1 << 16, 3 << 16)]:
        idx, bufs = workloads.build_pinned(inv, seed, A, B)
        lay, oparts, payloads = oracle_of(inv, seed, A, B)
        cfg = sllm.LoadConfig(chunk_bytes=C, n_streams=2, mode=mode, ctas=7, engine=engine)
        res = sllm.load(idx, bufs, {0: 0}, cfg)
        check_against_oracle(res, idx, inv, lay, oparts, payloads, [0], cfg)


@pytest.mark.parametrize("seed", range(24))
def test_random_checkpoints(seed):
    """S:570 acceptance 1 on the GPU: random checkpoints (1-4 logical partitions, all on
    GPU 0), random mode/chunk/streams/CTAs, byte-exact against the oracle."""
    rng = np.random.default_rng(5000 + seed)
    inv = models.random_inventory(rng, int(rng.integers(1, 2000)), int(rng.integers(1, 5)), 24 << 20)
    A = int(rng.choice([16, 256, 4096]))
    B = int(rng.choice([4096, 1 << 16, 1 << 20]))
    idx, bufs = workloads.build_pinned(inv, seed, A, B)
    lay, oparts, payloads = oracle_of(inv, seed, A, B)
    mode = MODES[seed % 4]
    chunk = B * int(rng.integers(1, 5)) if B >= 1 << 16 else 1 << 16
    cfg = sllm.LoadConfig(chunk_bytes=chunk, n_streams=int(rng.integers(1, 5)), mode=mode,
                          ctas=int(rng.choice([0, 1, 5, 64])), engine=["tma", "ldg", "tma_store"][(seed // 4) % 3])
    n = len(idx.partitions)
    res = sllm.load(idx, bufs, {p: 0 for p in range(n)}, cfg)
    check_against_oracle(res, idx, inv, lay, oparts, payloads, list(range(n)), cfg)


@pytest.mark.parametrize("engine", ["tma", "ldg", "tma_store"])
@pytest.mark.parametrize("mode", MODES)
def test_fault_injection_names_block(mode, engine):
    """A flipped source byte in block j yields SLLM_E_CHECKSUM(0, j) -- the same
    (partition, block) the oracle loader reports (O9(d))."""
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    host = bufs[0].numpy()
    clean = host.copy()
    rng = np.random.default_rng(MODES.index(mode))
    for _ in range(3):
        pos = int(rng.integers(0, host.size))
        host[pos] ^= np.uint8(1 << int(rng.integers(0, 8)))
        with pytest.raises(Exception) as oex:
            oloader.load(idx.serialize(), {0: host})
        assert (oex.value.partition, oex.value.block) == (0, pos // (1 << 20))
        cfg = sllm.LoadConfig(chunk_bytes=2 << 20, mode=mode, engine=engine)
        bases, per_tensor = sllm.allocate(idx, {0: 0}, cfg.scatter)
        res = sllm.load_start(idx, bufs, {0: 0}, cfg, bases, per_tensor)
        with pytest.raises(sllm.SllmError) as ex:
            res.wait()
        assert ex.value.status == 9
        assert (res.report["bad_partition"], res.report["bad_block"]) == (0, pos // (1 << 20))
        host[:] = clean


def test_profile_levels():
    """profile 1 times every kernel launch with CUDA events; 3 adds the launches' in-kernel
    spans (first CTA start .. last CTA end), which lie inside the event times; 4 is rejected.
    Profiling never changes the loaded bytes."""
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, payloads = oracle_of(inv, seed, 4096, 1 << 20)
    for mode in MODES:
        for prof in (0, 1, 3):
            cfg = sllm.LoadConfig(chunk_bytes=1 << 20, mode=mode, profile=prof)
            res = sllm.load(idx, bufs, {0: 0}, cfg)
            rep = res.report
            check_against_oracle(res, idx, inv, lay, oparts, payloads, [0], cfg)
            if prof == 0:
                assert rep["t_kernel_ms_sum"] == 0 and rep["t_kernel_span_ms_sum"] == 0
            else:
                assert rep["t_kernel_ms_sum"] > 0 and rep["kernel_bytes"] > 0, (mode, prof)
            if prof == 3:
                assert 0 < rep["t_kernel_span_ms_sum"] <= rep["t_kernel_ms_sum"], (mode, rep)
            elif prof == 1:
                assert rep["t_kernel_span_ms_sum"] == 0
    with pytest.raises(sllm.SllmError) as ex:
        sllm.load(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20, profile=4))
    assert ex.value.status == 1


def test_verify_off_still_exact():
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, payloads = oracle_of(inv, seed, 4096, 1 << 20)
    for mode in MODES:
        cfg = sllm.LoadConfig(chunk_bytes=1 << 20, mode=mode, verify=False)
        res = sllm.load(idx, bufs, {0: 0}, cfg)
        # one kernel per 64 MiB window of chunks (none at all for CE without verification)
        assert res.report["kernel_launches"] == (0 if mode == "ce" else -(-res.report["chunks"] // 64))
        check_against_oracle(res, idx, inv, lay, oparts, payloads, [0], cfg)


@pytest.mark.parametrize("engine", ["tma", "ldg", "tma_store"])
@pytest.mark.parametrize("mode", ["scatter_ce", "scatter_zc"])
def test_scatter_canaries(mode, engine):
    """O9(b): guard bytes around every per-tensor destination stay untouched."""
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, payloads = oracle_of(inv, seed, 4096, 1 << 20)
    G = 256
    total = sum(G + ((t.nbytes + 15) // 16) * 16 + G for t in idx.tensors)
    arena = torch.full((total,), 0xCD, dtype=torch.uint8, device="cuda:0")
    per_tensor, spans, off = {}, [], 0
    dts = {"f16": torch.float16}
    for t in idx.tensors:
        lo = off + G
        per_tensor[t.name] = arena[lo:lo + t.nbytes].view(dts[t.dtype]).view(t.shape)
        spans.append((lo, lo + t.nbytes))
        off = lo + ((t.nbytes + 15) // 16) * 16 + G
    res = sllm.load_start(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20, mode=mode, engine=engine), None,
                          per_tensor)
    res.wait()
    a = arena.cpu().numpy()
    mask = np.ones(a.size, bool)
    for (lo, hi), e in zip(spans, range(len(inv))):
        assert np.array_equal(a[lo:hi], payloads[e])
        mask[lo:hi] = False
    assert (a[mask] == 0xCD).all()


def test_caller_stream_ordering():
    """views exist before the data; work queued on the caller's stream after
    start sees the loaded bytes without an explicit wait (the stream waits on the load)."""
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, payloads = oracle_of(inv, seed, 4096, 1 << 20)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        bases, _ = sllm.allocate(idx, {0: 0})
        res = sllm.load_start(idx, bufs, {0: 0}, sllm.LoadConfig(mode="zerocopy"), bases, None, {0: s})
        t = res.tensors["lm_head.weight"]
        copy = t.view(torch.uint8).clone()   # queued on s after start
    s.synchronize()
    e = [i for i, x in enumerate(inv) if x.name == "lm_head.weight"][0]
    assert np.array_equal(copy.reshape(-1).cpu().numpy(), payloads[e])
    res.wait()


def test_busy_rejected():
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    bases, _ = sllm.allocate(idx, {0: 0})
    r1 = sllm.load_start(idx, bufs, {0: 0}, sllm.LoadConfig(), bases)
    with pytest.raises(sllm.SllmError) as ex:
        sllm.load_start(idx, bufs, {0: 0}, sllm.LoadConfig(), bases)
    assert ex.value.status == 10
    r1.wait()
    r2 = sllm.load_start(idx, bufs, {0: 0}, sllm.LoadConfig(), bases)   # free again after wait
    r2.wait()


def test_handles_before_wait():
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    bases, _ = sllm.allocate(idx, {0: 0})
    res = sllm.load_start(idx, bufs, {0: 0}, sllm.LoadConfig(), bases)
    h = res.handle_of("layers.1.mlp.fc2.weight")
    t = idx.tensors[idx.find("layers.1.mlp.fc2.weight")]
    assert h["ptr"] == bases[0].data_ptr() + t.offset and h["shape"] == (384, 1536) and h["gpu"] == 0
    res.wait()
    with pytest.raises(sllm.SllmError):
        res.handle_of("nope")


def test_device_checksum_kernel_matches_oracle():
    rng = np.random.default_rng(3)
    for n, B in [(16, 16), (4096 * 3 + 48, 4096), ((1 << 20) * 5 + 4096, 1 << 20), ((64 << 20) + 16 * 7, 1 << 20)]:
        x = rng.integers(0, 256, size=n, dtype=np.uint8)
        d = torch.from_numpy(x).cuda()
        nb = -(-n // B)
        out = torch.zeros(nb, dtype=torch.int64, device="cuda")
        sllm.block_checksums_device(d.data_ptr(), n, B, out.data_ptr())
        torch.cuda.synchronize()
        got = [int(v) & (2**64 - 1) for v in out.cpu().tolist()]
        assert got == fletcher.block_checksums(x, B)


def test_device_checksum_extreme_words():
    # all words M-1 / M / 0 patterns exercise every fold of the closed form
    for word in (0xFFFFFFFE, 0xFFFFFFFF, 0x80000001, 0):
        x = np.full((1 << 20) // 4 * 3, word, dtype="<u4").view(np.uint8)
        d = torch.from_numpy(x.copy()).cuda()
        out = torch.zeros(3, dtype=torch.int64, device="cuda")
        sllm.block_checksums_device(d.data_ptr(), x.size, 1 << 20, out.data_ptr())
        torch.cuda.synchronize()
        assert [int(v) & (2**64 - 1) for v in out.cpu().tolist()] == fletcher.block_checksums(x, 1 << 20)


@pytest.mark.parametrize("engine", ["", "ldg", "tma", "tma_store"])
def test_materialise_device_matches_oracle(engine, monkeypatch):
    monkeypatch.setenv("SLLM_STANDALONE_ENGINE", engine)
    inv = models.llama2(512, 3, 1024, 128, vocab=2048, tp=2)
    idx, bufs = workloads.build_pinned(inv, 11, 4096, 1 << 16)
    lay, oparts, payloads = oracle_of(inv, 11, 4096, 1 << 16)
    for p in range(2):
        d = lay.devices()[p]
        src = torch.from_numpy(oparts[d].copy()).cuda()
        _, per_tensor = sllm.allocate(idx, {0: 0, 1: 0}, scatter=True)
        sllm.materialise_device(idx, p, src.data_ptr(), per_tensor)
        for e, t in enumerate(inv):
            if t.device == d:
                assert np.array_equal(per_tensor[t.name].view(torch.uint8).reshape(-1).cpu().numpy(), payloads[e])
        src[100] ^= 1
        with pytest.raises(sllm.SllmError) as ex:
            sllm.materialise_device(idx, p, src.data_ptr(), per_tensor)
        assert ex.value.status == 9


@pytest.mark.parametrize("workload", ["toy", "300mb"])
def test_fanout_single_rank_nccl(workload):
    """The replicated path with one rank exercises NCCL init + grouped broadcasts / in-place
    all-gathers; the result must equal P_0 exactly (O9(c)).  Rounds run in whole 64 MiB
    units of chunks (sllm_fanout_unit): the toy is one ragged round, the ~300 MB replica
    four full rounds (in-place all-gathers) and a ragged last one."""
    if workload == "toy":
        inv, seed = models.model_inventory("toy")
    else:
        rng = np.random.default_rng(31)   # 60 tensors of 2.5-7.5 MB with odd shapes (~300 MB)
        inv, seed = [models.TensorSpec(f"w{i}", 0, "f16", (int(rng.integers(1200, 3700)), 1029))
                     for i in range(60)], 31
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, payloads = oracle_of(inv, seed, 4096, 1 << 20)
    L = idx.partitions[0].length
    comm = sllm.Comm.init_rank(sllm.Comm.unique_id(), 1, 0, 0)
    for fanout in ("bcast", "allgather"):
        U = sllm.fanout_unit(2 << 20, fanout)
        if workload != "toy" and fanout == "allgather":
            rounds = sllm.allgather_schedule(L, U, 1)
            assert sum(f for f, _ in rounds) >= 4 and not rounds[-1][0]
        for mode in ("ce", "zerocopy"):
            cfg = sllm.LoadConfig(chunk_bytes=2 << 20, mode=mode, fanout=fanout)
            res = sllm.load(idx, bufs, {0: 0}, cfg, comm=comm)
            check_against_oracle(res, idx, inv, lay, oparts, payloads, [0], cfg)
            assert res.report["transferred_bytes"] == L
            assert res.report["copy_calls"] <= -(-L // U) + 1 if mode == "ce" else True
    comm.free()


def test_fanout_comm_init_all_single_process():
    """The single-process communicator (sllm_comm_init_all, one handle per GPU of the
    process) drives the NCCL fan-outs exactly like a per-rank communicator."""
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, payloads = oracle_of(inv, seed, 4096, 1 << 20)
    (comm,) = sllm.Comm.init_all([0])
    for fanout in ("bcast", "allgather"):
        cfg = sllm.LoadConfig(chunk_bytes=1 << 20, mode="ce", fanout=fanout)
        res = sllm.load(idx, bufs, {0: 0}, cfg, comm=comm)
        check_against_oracle(res, idx, inv, lay, oparts, payloads, [0], cfg)
    comm.free()


def test_allgather_rejects_files_and_peer_groups(tmp_path):
    inv, seed = models.model_inventory("toy")
    payloads = [payload.payload_bytes(seed, e, t.nbytes) for e, t in enumerate(inv)]
    sllm.convert([(t.name, t.device, t.dtype, t.shape, p.ctypes.data) for t, p in zip(inv, payloads)],
                 str(tmp_path), 4096, 1 << 20, "toy")
    idx = sllm.Index.open(str(tmp_path / "index.bin"))
    comm = sllm.Comm.init_rank(sllm.Comm.unique_id(), 1, 0, 0)
    with pytest.raises(sllm.SllmError) as ex:   # strided chunks: pinned sources only
        sllm.load_files(idx, str(tmp_path), {0: 0}, sllm.LoadConfig(chunk_bytes=2 << 20, fanout="allgather"), comm=comm)
    assert ex.value.status == 1
    comm.free()
    L = idx.partitions[0].length
    base = torch.empty(L, dtype=torch.uint8, device="cuda")
    sig = torch.zeros(2, dtype=torch.int32, device="cuda")
    peers = sllm.Comm.peers(1, 0, 0, [base.data_ptr()], [sig.data_ptr()])
    idx2, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    with pytest.raises(sllm.SllmError) as ex:   # a peer group is not an NCCL communicator
        sllm.load(idx2, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=2 << 20, fanout="allgather"), comm=peers)
    assert ex.value.status == 1
    peers.free()


def test_opt67b_full_size_sampled():
    """BASELINE configs[1] at full size in bench.py's launch configuration: every block
    checksum equals the oracle's (sampled blocks recomputed by the oracle from the pinned
    source) and sampled tensors equal their payload regenerated by the oracle side."""
    inv, seed = models.model_inventory("opt-6.7b")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    src = bufs[0].numpy()
    rng = np.random.default_rng(0)
    blocks = sorted(set(rng.integers(0, idx.partitions[0].n_blocks, size=24).tolist()) | {idx.partitions[0].n_blocks - 1})
    table = idx.block_checksums(0)
    for j in blocks:
        assert int(table[j]) == fletcher.f64_closed(src[j << 20:(j + 1) << 20])
    for mode in ("ce", "zerocopy", "scatter_ce", "scatter_zc"):
        res = sllm.load(idx, bufs, {0: 0}, sllm.LoadConfig(mode=mode, chunk_bytes=64 << 20))
        cs = res.block_checksums(0)
        assert np.array_equal(cs, table), mode
        for e in sorted(set(rng.integers(0, len(inv), size=12).tolist()) | {0, 1, 2, len(inv) - 1}):
            t = inv[e]
            got = res.tensors[t.name].view(torch.uint8).reshape(-1)
            n = min(t.nbytes, 1 << 20)
            want = payload.payload_bytes(seed, e, t.nbytes)
            assert np.array_equal(got[:n].cpu().numpy(), want[:n]), (mode, t.name)
            assert np.array_equal(got[-n:].cpu().numpy(), want[-n:]), (mode, t.name)
        # every tensor, every byte, against its payload regenerated on the host (C generator
        # pinned to the NumPy definition), compared on the device
        big = max(t.nbytes for t in inv)
        host = torch.empty(big, dtype=torch.uint8, pin_memory=True)
        dev = torch.empty(big, dtype=torch.uint8, device="cuda")
        for e, t in enumerate(inv):
            payload.payload_into([host.data_ptr()], [t.nbytes], seed, [e])
            dev[:t.nbytes].copy_(host[:t.nbytes])
            assert torch.equal(res.tensors[t.name].reshape(-1).view(torch.uint8), dev[:t.nbytes]), (mode, t.name)
        del host, dev
        del res
        torch.cuda.empty_cache()


def test_auto_mode_picks_by_size():
    """SLLM_MODE_AUTO: zero-copy for a small checkpoint, the copy engine for one above the
    256 MiB crossover; both exact."""
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, payloads = oracle_of(inv, seed, 4096, 1 << 20)
    res = sllm.load(idx, bufs, {0: 0}, sllm.LoadConfig(mode="auto"))
    assert res.report["mode"] == 1  # ZEROCOPY
    check_against_oracle(res, idx, inv, lay, oparts, payloads, [0], sllm.LoadConfig(mode="zerocopy"))
    big = models.llama2(1024, 12, 4096, 1024, vocab=32000)  # ~0.4 GB, one partition
    idx2, bufs2 = workloads.build_pinned(big, 9, 4096, 1 << 20)
    res2 = sllm.load(idx2, bufs2, {0: 0}, sllm.LoadConfig(mode="auto", chunk_bytes=64 << 20))
    assert idx2.partitions[0].length >= 256 << 20 and res2.report["mode"] == 0  # CE
    assert np.array_equal(res2.block_checksums(0), idx2.block_checksums(0))
    for e in (0, len(big) - 1):
        t = big[e]
        got = res2.tensors[t.name].reshape(-1).view(torch.uint8)[:4096].cpu().numpy()
        assert np.array_equal(got, payload.payload_bytes(9, e, t.nbytes)[:4096])


@pytest.mark.parametrize("mode", MODES + ["auto"])
def test_lora_adapter_all_modes_bit_exact(mode):
    """the rank-32 LoRA adapter of LLaMA-2-70B (828 MB, 1,120 small
    tensors -- the paper's ~1 GB adapter) in every mode: every tensor byte-equal
    to its payload, every block checksum equal to the oracle's table, the whole partition
    (padding included) equal to the oracle's bytes in the contiguous modes."""
    inv, seed = models.model_inventory("lora-70b-r32")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, payloads = _lora_oracle()
    cfg = sllm.LoadConfig(chunk_bytes=16 << 20, mode=mode)
    res = sllm.load(idx, bufs, {0: 0}, cfg)
    assert len(res.tensors) == 1120
    check_against_oracle(res, idx, inv, lay, oparts, payloads, [0], cfg)
    if mode == "auto":   # < 256 MiB per job picks zero-copy; 828 MB stays on the copy engine
        assert res.report["mode"] == 0


_LORA = {}


def _lora_oracle():
    if not _LORA:
        inv, seed = models.model_inventory("lora-70b-r32")
        _LORA["v"] = oracle_of(inv, seed, 4096, 1 << 20)
    return _LORA["v"]
