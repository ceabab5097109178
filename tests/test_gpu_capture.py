"""GPU parity of captured loads (sllm_load_capture / sllm_load_replay, SURVEY §8(f) rank 3:
the latency-bound small-checkpoint path replayed as CUDA graphs).

A capture records the whole device work of a load (table upload, accumulator reset, copy
windows, verify / scatter launches, result read-back) and moves no byte; every replay must
then load the checkpoint bit-exact against the oracle (bytes, per-tensor payloads, block
checksums) in every mode, report a flipped source byte as the oracle's (partition, block)
and recover on the next replay (the result word is reset by the graph itself), keep its
destinations reserved, and order the caller's stream after the replay."""
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

MODES = ["ce", "zerocopy", "scatter_ce", "scatter_zc"]


def oracle_of(inv, seed, A=4096, B=1 << 20):
    payloads = [payload.payload_bytes(seed, e, t.nbytes) for e, t in enumerate(inv)]
    lay, parts = olayout.convert([(t.name, t.device, t.dtype, t.shape, p) for t, p in zip(inv, payloads)], A, B)
    return lay, parts, payloads


def _b(t):
    """The tensor's bytes as a flat uint8 view (rank-0 scalars included)."""
    return t.reshape(-1).view(torch.uint8)


def check(cap, inv, lay, oparts, payloads, cfg):
    for e, t in enumerate(inv):
        got = cap.tensors[t.name]
        got_b = got.contiguous().view(torch.uint8).reshape(-1).cpu().numpy() if got.dim() else \
            got.reshape(1).view(torch.uint8).cpu().numpy()
        assert np.array_equal(got_b, payloads[e]), t.name
    if not cfg.scatter:
        assert np.array_equal(cap._keep[2][0].cpu().numpy(), oparts[lay.devices()[0]])
    assert cap.block_checksums(0).tolist() == lay.checksums[lay.devices()[0]]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("chunk", [1 << 20, 4 << 20])
def test_capture_replays_bit_exact(mode, chunk):
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, payloads = oracle_of(inv, seed)
    cfg = sllm.LoadConfig(chunk_bytes=chunk, mode=mode)
    bases, per = sllm.allocate(idx, {0: 0}, cfg.scatter)
    for t in (bases.values() if not cfg.scatter else per.values()):
        _b(t).fill_(0xA5)
    torch.cuda.synchronize()
    cap = sllm.load_capture(idx, bufs, {0: 0}, cfg, bases, per)
    # the capture moves no byte
    for t in (bases.values() if not cfg.scatter else per.values()):
        assert bool((_b(t) == 0xA5).all())
    for r in range(3):
        for t in (bases.values() if not cfg.scatter else per.values()):
            _b(t).fill_(0x5A + r)
        torch.cuda.synchronize()
        rep = cap.replay().wait()
        assert rep["bad_partition"] == -1 and rep["payload_bytes"] == sum(t.nbytes for t in inv)
        assert rep["transferred_bytes"] == idx.partitions[0].length
        check(cap, inv, lay, oparts, payloads, cfg)
    cap.free()


@pytest.mark.parametrize("mode", ["ce", "scatter_ce", "zerocopy"])
def test_capture_multi_window_partition(mode):
    """A ~0.5 GB partition at 1 MiB chunks: several copy windows, verification spans, the
    scatter staging ring and ticketed work units all inside the graph."""
    inv = models.llama2(1024, 12, 4096, 1024, vocab=32000)
    seed = 9
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, payloads = oracle_of(inv, seed)
    cfg = sllm.LoadConfig(chunk_bytes=1 << 20, mode=mode)
    bases, per = sllm.allocate(idx, {0: 0}, cfg.scatter)
    cap = sllm.load_capture(idx, bufs, {0: 0}, cfg, bases, per)
    for r in range(2):
        for t in (bases.values() if not cfg.scatter else per.values()):
            _b(t).fill_(r)
        torch.cuda.synchronize()
        cap.replay().wait()
        check(cap, inv, lay, oparts, payloads, cfg)
    cap.free()


@pytest.mark.parametrize("mode", ["ce", "zerocopy", "scatter_ce"])
def test_capture_fault_reported_then_recovers(mode):
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, payloads = oracle_of(inv, seed)
    cfg = sllm.LoadConfig(chunk_bytes=1 << 20, mode=mode)
    bases, per = sllm.allocate(idx, {0: 0}, cfg.scatter)
    cap = sllm.load_capture(idx, bufs, {0: 0}, cfg, bases, per)
    src = bufs[0].numpy()
    pos = 5 * (1 << 20) + 12345          # inside tensor bytes of block 5
    src[pos] ^= 0x10
    try:
        cap.replay()
        with pytest.raises(sllm.SllmError) as ex:
            cap.wait()
        assert ex.value.status == 9 and cap.report["bad_partition"] == 0 and cap.report["bad_block"] == pos >> 20
    finally:
        src[pos] ^= 0x10
    cap.replay().wait()                  # the graph resets its result word: the next replay is clean
    check(cap, inv, lay, oparts, payloads, cfg)
    cap.free()


def test_capture_streams_busy_and_rejects():
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    lay, oparts, payloads = oracle_of(inv, seed)
    cfg = sllm.LoadConfig(chunk_bytes=1 << 20, mode="ce")
    bases, _ = sllm.allocate(idx, {0: 0})
    cap = sllm.load_capture(idx, bufs, {0: 0}, cfg, bases)
    # caller-stream ordering: work queued on the replay's stream sees the loaded bytes
    s = torch.cuda.Stream()
    bases[0].fill_(0)
    torch.cuda.synchronize()
    cap.replay({0: s})
    with torch.cuda.stream(s):
        copy = bases[0].clone()
    with pytest.raises(sllm.SllmError) as ex:   # one replay in flight at a time
        cap.replay()
    assert ex.value.status == 10
    cap.wait()
    s.synchronize()
    assert np.array_equal(copy.cpu().numpy(), oparts[lay.devices()[0]])
    with pytest.raises(sllm.SllmError) as ex:   # the destination stays reserved
        sllm.load_start(idx, bufs, {0: 0}, cfg, bases)
    assert ex.value.status == 10
    cap.free()
    res = sllm.load_start(idx, bufs, {0: 0}, cfg, bases)  # released with the captured load
    res.wait()
    res.free()
    with pytest.raises(sllm.SllmError) as ex:   # no fan-out in a captured load
        sllm.load_capture(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20, fanout="p2p"), bases)
    assert ex.value.status == 1
    plain = sllm.load_start(idx, bufs, {0: 0}, cfg, bases)
    plain.wait()
    with pytest.raises(sllm.SllmError) as ex:   # replay needs a captured load
        sllm.CapturedLoad.replay(plain)
    assert ex.value.status == 1
    plain.free()
