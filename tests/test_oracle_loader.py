"""Pins of oracle.loader: every loaded tensor equals the payload
regenerated independently from (seed, e) (O10), random checkpoints round-trip,
and a flipped source byte in block j is reported as exactly (partition, j)."""
import numpy as np
import pytest

from oracle import index, layout as L, loader
from oracle.errors import ChecksumError
from synth import models, payload


def _convert(inv, seed, A=4096, B=1 << 20):
    tensors = [(t.name, t.device, t.dtype, t.shape, payload.payload_bytes(seed, e, t.nbytes))
               for e, t in enumerate(inv)]
    lay, parts = L.convert(tensors, A, B, "m")
    return tensors, index.write(lay), parts


def test_toy_load_matches_payload():
    inv = models.toy()
    tensors, blob, parts = _convert(inv, 0)
    res = loader.load(blob, parts)
    assert res.payload_bytes == 13_569_860 and res.transferred_bytes == 13_594_624
    for e, t in enumerate(inv):
        assert res.tensors[t.name].tobytes() == payload.payload_bytes(0, e, t.nbytes).tobytes()
    res2 = loader.load(blob, parts, scatter=True)
    for t in inv:
        assert res2.tensors[t.name].tobytes() == res.tensors[t.name].tobytes()


@pytest.mark.parametrize("seed", range(20))
def test_random_checkpoints_roundtrip(seed):
    rng = np.random.default_rng(1000 + seed)
    inv = models.random_inventory(rng, int(rng.integers(1, 500)), int(rng.integers(1, 5)), 2 << 20)
    tensors, blob, parts = _convert(inv, seed, A=int(rng.choice([16, 4096])), B=1 << 14)
    res = loader.load(blob, parts)
    for t in tensors:
        assert res.tensors[t[0]].tobytes() == t[4].tobytes()


def test_fault_injection_names_block():
    inv = models.toy()
    _, blob, parts = _convert(inv, 0)
    rng = np.random.default_rng(5)
    for _ in range(10):
        pos = int(rng.integers(0, parts[0].size))
        bad = {0: parts[0].copy()}
        bad[0][pos] ^= np.uint8(1 << int(rng.integers(0, 8)))
        with pytest.raises(ChecksumError) as ex:
            loader.load(blob, bad)
        assert (ex.value.partition, ex.value.block) == (0, pos // (1 << 20))


def test_padding_flip_detected():
    # a flipped padding byte (outside every tensor) still fails its block (checksums
    # cover partition bytes, padding included -- O8)
    inv = models.toy()
    _, blob, parts = _convert(inv, 0)
    lay = index.read(blob)
    last = lay.entries[-1]
    pos = last.offset + last.size + 5
    bad = {0: parts[0].copy()}
    bad[0][pos] = 0x5A
    with pytest.raises(ChecksumError) as ex:
        loader.load(blob, bad)
    assert ex.value.block == pos // (1 << 20)


def test_multi_partition_fault_partition_index():
    inv = models.llama2(64, 2, 128, 32, vocab=256, tp=2)
    _, blob, parts = _convert(inv, 9, B=4096)
    bad = {d: p.copy() for d, p in parts.items()}
    bad[1][5000] ^= 0xFF
    with pytest.raises(ChecksumError) as ex:
        loader.load(blob, bad)
    assert (ex.value.partition, ex.value.block) == (1, 1)


def _whole_tensor_bytes_by_ownership(inv, A, B, hi_of):
    """Brute force, independent of the layout code: convert a copy of the checkpoint whose
    tensor e is filled with the marker byte pattern of e (so every partition byte names its
    owner), then count, per partition, the tensors ALL of whose bytes lie in the sampled
    prefix [0, hi_of(d)) -- the payload a sample of that prefix materialises."""
    assert len(inv) < 255
    marks = [(t.name, t.device, t.dtype, t.shape, np.full(t.nbytes, e + 1, np.uint8)) for e, t in enumerate(inv)]
    total = 0
    _, parts = L.convert(marks, A, B, "m")
    for d in parts:
        # owner of every byte read off the partition bytes themselves (0 = padding)
        counts_in = np.bincount(parts[d][:hi_of(d)], minlength=256)
        for e, t in enumerate(inv):
            if t.device == d and counts_in[e + 1] == t.nbytes:
                total += t.nbytes
    return total


@pytest.mark.parametrize("budget", [1, 1 << 20, (1 << 20) + 1, 4 << 20, 13 << 20, 64 << 20])
def test_sample_loader_payload_exact(budget):
    """load_sample (what cpu_baseline and `bench.py --impl reference` time) materialises
    exactly the tensors lying wholly inside the sampled prefix: the prefix is the budget
    rounded up to whole 1 MiB blocks (all of the partition once the budget exceeds it)."""
    inv = models.toy()
    _, blob, parts = _convert(inv, 0)
    got = loader.load_sample(blob, parts, budget)
    B = 1 << 20
    hi = min(13_594_624, -(-budget // B) * B)
    assert got == _whole_tensor_bytes_by_ownership(inv, 4096, B, lambda d: hi)
    if budget >= 13_594_624:
        assert got == 13_569_860            # the toy's whole payload


def test_sample_loader_multi_partition_budget_spans_partitions():
    inv = models.llama2(64, 2, 128, 32, vocab=256, tp=2)
    _, blob, parts = _convert(inv, 9, B=4096)
    lay = index.read(blob)
    L0 = lay.partitions[0]
    budget = L0 + 3 * 4096 + 1   # all of partition 0, then 4 blocks of partition 1
    got = loader.load_sample(blob, parts, budget)
    assert got == _whole_tensor_bytes_by_ownership(inv, 4096, 4096, lambda d: L0 if d == 0 else 4 * 4096)


def test_sample_loader_verifies_what_it_samples():
    """A flipped byte inside the sample raises ChecksumError(partition, block); one past the
    sampled prefix is never read, so the sample passes."""
    inv = models.toy()
    _, blob, parts = _convert(inv, 0)
    for pos in (5, (1 << 20) + 7, (2 << 20) - 1):
        bad = {0: parts[0].copy()}
        bad[0][pos] ^= 0x40
        with pytest.raises(ChecksumError) as ex:
            loader.load_sample(blob, bad, 2 << 20)
        assert (ex.value.partition, ex.value.block) == (0, pos // (1 << 20))
    bad = {0: parts[0].copy()}
    bad[0][(2 << 20) + 3] ^= 0x40
    assert loader.load_sample(blob, bad, 2 << 20) == loader.load_sample(blob, parts, 2 << 20)
