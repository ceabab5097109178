"""Pinned whole-model LRU cache (sllm_cache_*; SPEC
S:102-108).  CPU tests run the cache with pin=0 (plain page-aligned memory):
the policy -- hits, misses, LRU eviction of unheld models only, capacity errors, one
read for concurrent acquirers -- and the resident bytes, which must equal the oracle
converter's partitions byte for byte.  The GPU test loads straight from a pinned entry."""
import threading

import numpy as np
import pytest

import paper_2401_14351_b200 as sllm
from oracle import layout as olayout
from synth import models, payload

MiB = 1 << 20


def make_model(tmp_path, name, seed, total):
    rng = np.random.default_rng(seed)
    inv = models.random_inventory(rng, 40, 2, total, dtypes=("f16", "f32"))
    data = [payload.payload_bytes(seed, e, t.nbytes) for e, t in enumerate(inv)]
    d = str(tmp_path / name)
    sllm.convert([(t.name, t.device, t.dtype, t.shape, a.ctypes.data) for t, a in zip(inv, data)], d, 4096, 64 << 10)
    lay, parts = olayout.convert([(t.name, t.device, t.dtype, t.shape, a) for t, a in zip(inv, data)], 4096, 64 << 10)
    return d, lay, parts


def footprint(lay):  # the cache rounds every partition up to 2 MiB
    return sum(-(-L // (2 * MiB)) * 2 * MiB for L in lay.partitions.values())


def resident_equals_oracle(index, bufs, lay, parts):
    import ctypes
    for p, d in enumerate(lay.devices()):
        L = index.partitions[p].length
        got = np.ctypeslib.as_array((ctypes.c_uint8 * L).from_address(bufs[p]))
        if not np.array_equal(got, parts[d]):
            return False
    return True


def test_hits_misses_and_lru_eviction(tmp_path):
    A = make_model(tmp_path, "a", 1, 6 * MiB)
    B = make_model(tmp_path, "b", 2, 6 * MiB)
    C = make_model(tmp_path, "c", 3, 6 * MiB)
    fa, fb, fc = (footprint(m[1]) for m in (A, B, C))
    cache = sllm.PinnedCache(max(fa + fb, fa + fc, fb + fc), pin=False)  # room for two models, not three
    for m in (A, B):
        idx, bufs, hit = cache.acquire(m[0])
        assert not hit and resident_equals_oracle(idx, bufs, m[1], m[2])
        cache.release(m[0])
    idx, bufs, hit = cache.acquire(A[0])          # A becomes most recently used
    assert hit and resident_equals_oracle(idx, bufs, A[1], A[2])
    cache.release(A[0])
    idx, bufs, hit = cache.acquire(C[0])          # must evict B (LRU), not A
    assert not hit and resident_equals_oracle(idx, bufs, C[1], C[2])
    cache.release(C[0])
    st = cache.stats()
    assert (st["hits"], st["misses"], st["evictions"], st["models"]) == (1, 3, 1, 2)
    assert st["used"] == fa + fc
    _, _, hit = cache.acquire(A[0])
    assert hit
    cache.release(A[0])
    _, _, hit = cache.acquire(B[0])               # B was evicted: a miss again (evicts C)
    assert not hit
    cache.release(B[0])
    assert cache.stats()["evictions"] == 2
    cache.close()


def test_held_models_are_never_evicted(tmp_path):
    A = make_model(tmp_path, "a", 4, 5 * MiB)
    B = make_model(tmp_path, "b", 5, 5 * MiB)
    cache = sllm.PinnedCache(max(footprint(A[1]), footprint(B[1])) + MiB, pin=False)  # one model at a time
    idx, bufs, _ = cache.acquire(A[0])
    with pytest.raises(sllm.SllmError) as ex:     # A is held: B cannot make room
        cache.acquire(B[0])
    assert ex.value.status == 5
    assert resident_equals_oracle(idx, bufs, A[1], A[2])   # A untouched by the failed miss
    cache.release(A[0])
    idx, bufs, hit = cache.acquire(B[0])          # now A is evictable
    assert not hit and resident_equals_oracle(idx, bufs, B[1], B[2])
    cache.release(B[0])
    with pytest.raises(sllm.SllmError) as ex:     # releasing what is not held
        cache.release(A[0])
    assert ex.value.status == 4
    cache.close()


def test_model_larger_than_capacity_and_missing_dir(tmp_path):
    A = make_model(tmp_path, "a", 6, 8 * MiB)
    cache = sllm.PinnedCache(2 * MiB, pin=False)
    with pytest.raises(sllm.SllmError) as ex:
        cache.acquire(A[0])
    assert ex.value.status == 5
    with pytest.raises(sllm.SllmError) as ex:
        cache.acquire(str(tmp_path / "nowhere"))
    assert ex.value.status == 6
    assert cache.stats()["used"] == 0 and cache.stats()["models"] == 0
    cache.close()


def test_concurrent_acquirers_share_one_read(tmp_path):
    A = make_model(tmp_path, "a", 7, 24 * MiB)
    cache = sllm.PinnedCache(64 * MiB, pin=False)
    out, errs = [], []

    def worker():
        try:
            idx, bufs, hit = cache.acquire(A[0], io_threads=2)
            out.append((hit, resident_equals_oracle(idx, bufs, A[1], A[2])))
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=worker) for _ in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs and len(out) == 6 and all(ok for _, ok in out)
    assert sum(1 for hit, _ in out if not hit) == 1        # exactly one read from storage
    st = cache.stats()
    assert (st["misses"], st["hits"]) == (1, 5)
    for _ in range(6):
        cache.release(A[0])
    cache.close()


@pytest.mark.gpu
def test_load_from_pinned_cache_entry(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    A = make_model(tmp_path, "a", 8, 16 * MiB)
    cache = sllm.PinnedCache(64 * MiB, gpu=0, pin=True)
    idx, bufs, hit = cache.acquire(A[0])
    assert not hit
    n = len(idx.partitions)
    for mode in ("ce", "zerocopy", "scatter_ce"):
        res = sllm.load(idx, bufs, {p: 0 for p in range(n)}, sllm.LoadConfig(chunk_bytes=1 << 20, mode=mode))
        for p, d in enumerate(A[1].devices()):
            assert res.block_checksums(p).tolist() == A[1].checksums[d]
        for e, ent in enumerate(A[1].entries):
            got = res.tensors[ent.name].reshape(-1).view(torch.uint8).cpu().numpy()
            assert np.array_equal(got, A[2][ent.device][ent.offset:ent.offset + ent.size])
        del res
    cache.release(A[0])
    cache.close()
