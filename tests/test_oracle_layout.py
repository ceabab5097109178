"""Pins of oracle.layout (c3): SPEC worked examples,
invariants, brute-force order independence and closed-form model inventories."""
import itertools
import math

import numpy as np
import pytest

from oracle import layout as L
from oracle.errors import ConversionError, InvalidError, OracleLookupError
from synth import models, payload


def _t(name, dev, n, dt="u8"):
    w = L.WIDTH[dt]
    return (name, dev, dt, (n,), bytes(n * w))


def test_spec_example_two_tensors():
    # sizes 10 B and 6 B on device 0, align 4096 -> offsets 0 and 4096, length 8192
    lay = L.plan([_t("a", 0, 10), _t("b", 0, 6)], 4096, 0)
    assert [e.offset for e in lay.entries] == [0, 4096]
    assert lay.partitions == {0: 8192}


def test_empty_checkpoint():
    lay = L.plan([], 4096, 1 << 20)
    assert lay.partitions == {} and lay.entries == []


def test_first_tensor_is_base():
    lay = L.plan([_t("x", 3, 100)], 4096, 0)
    assert lay.entries[0].offset == 0
    assert L.address(lay, "x", {3: 1_000_000}) == (3, 1_000_000)


def test_spec_address_example():
    # base 1,000,000 + offset 4096 = 1,004,096
    lay = L.plan([_t("a", 0, 10), _t("b", 0, 6)], 4096, 0)
    assert L.address(lay, "b", {0: 1_000_000}) == (0, 1_004_096)
    with pytest.raises(OracleLookupError):
        L.address(lay, "nope", {0: 0})


def test_alignment_variants():
    lay = L.plan([_t("a", 0, 10), _t("b", 0, 6)], 16, 0)
    assert [e.offset for e in lay.entries] == [0, 16] and lay.partitions == {0: 32}


def test_validation_errors():
    with pytest.raises(ConversionError):
        L.plan([_t("a", 0, 4), _t("a", 0, 4)], 4096, 0)            # duplicate name
    with pytest.raises(ConversionError):
        L.convert([("a", 0, "f16", (3,), bytes(5))], 4096, 0)      # payload != shape*width
    with pytest.raises(ConversionError):
        L.plan([("", 0, "u8", (1,), bytes(1))], 4096, 0)           # empty name
    with pytest.raises(ConversionError):
        L.plan([("a", 0, "u8", (0,), bytes(0))], 4096, 0)          # zero dimension (Q16)
    with pytest.raises(ConversionError):
        L.plan([("a", -1, "u8", (1,), bytes(1))], 4096, 0)
    with pytest.raises(ConversionError):
        L.plan([("a", 0, "c64", (1,), bytes(8))], 4096, 0)
    for a, b in [(8, 0), (48, 0), (4096, 2048), (4096, 3 << 20)]:
        with pytest.raises(InvalidError):
            L.plan([_t("a", 0, 1)], a, b)


def test_scalar_tensor():
    lay = L.plan([("s", 0, "f16", (), bytes(2))], 4096, 0)
    assert lay.entries[0].size == 2 and lay.partitions[0] == 4096


def _check_invariants(tensors, lay, A):
    # alignment, disjointness, coverage, payload sum, padding bound (Q5)
    assert lay.payload_bytes == sum(len(t[4]) for t in tensors)
    for d, Ld in lay.partitions.items():
        es = sorted((e for e in lay.entries if e.device == d), key=lambda e: e.offset)
        assert Ld % A == 0
        for e in es:
            assert e.offset % A == 0 and e.offset + e.size <= Ld
        for a, b in zip(es, es[1:]):
            assert b.offset >= a.offset + a.size
        pad = Ld - sum(e.size for e in es)
        assert 0 <= pad < A * (len(es) + 1)


@pytest.mark.parametrize("seed", range(10))
def test_random_invariants_and_roundtrip(seed):
    rng = np.random.default_rng(seed)
    inv = models.random_inventory(rng, int(rng.integers(1, 300)), int(rng.integers(1, 5)), 4 << 20)
    tensors = [(t.name, t.device, t.dtype, t.shape, payload.payload_bytes(seed, e, t.nbytes))
               for e, t in enumerate(inv)]
    A = int(rng.choice([16, 256, 4096]))
    lay, parts = L.convert(tensors, A, 1 << 16)
    _check_invariants(tensors, lay, A)
    for e, t in zip(lay.entries, tensors):
        assert parts[e.device][e.offset:e.offset + e.size].tobytes() == t[4].tobytes()
    # bytes outside tensors are zero (Q3)
    for d, P in parts.items():
        mask = np.ones(P.size, bool)
        for e in lay.entries:
            if e.device == d:
                mask[e.offset:e.offset + e.size] = False
        assert not P[mask].any()


def test_order_independence_bruteforce():
    """every permutation of <= 6 tensors over 1-3 devices round-trips."""
    rng = np.random.default_rng(0)
    base = [(f"t{i}", int(rng.integers(0, 3)), "u8", (int(rng.integers(1, 40)),)) for i in range(6)]
    base = [(n, d, dt, s, rng.integers(0, 256, size=s[0], dtype=np.uint8).tobytes()) for n, d, dt, s in base]
    for k in (1, 3, 6):
        for perm in itertools.permutations(base[:k]):
            lay, parts = L.convert(list(perm), 16, 0)
            for e, t in zip(lay.entries, perm):
                assert e.name == t[0]
                assert parts[e.device][e.offset:e.offset + e.size].tobytes() == bytes(t[4])
            _check_invariants(list(perm), lay, 16)


def _bytes_of(inv):
    return sum(t.nbytes for t in inv)


def test_model_inventories_closed_form():
    """Closed forms from the public configs."""
    inv, _ = models.model_inventory("opt-6.7b")
    d, f, v, p, nl = 4096, 16384, 50272, 2050, 32
    per_layer = 4 * (d * d + d) + 2 * 2 * d + (f * d + f) + (d * f + d)
    assert len(inv) == 516
    assert _bytes_of(inv) == 2 * (v * d + p * d + 2 * d + nl * per_layer) == 13_316_947_968
    inv70 = models.llama2(8192, 80, 28672, 1024, tp=1)
    assert len(inv70) == 723
    assert _bytes_of(inv70) == 137_953_296_384
    inv70tp8, _ = models.model_inventory("llama2-70b-tp8")
    assert len(inv70tp8) == 8 * 723
    # shards cover the full model once, plus 7 extra copies of the replicated norms
    assert _bytes_of(inv70tp8) == 137_953_296_384 + 7 * (2 * 80 + 1) * 8192 * 2
    toy = models.toy()
    assert len(toy) == 22 and _bytes_of(toy) == 13_569_860
    lay = L.plan([(t.name, t.device, t.dtype, t.shape, t.nbytes) for t in toy], 4096, 1 << 20)
    assert lay.partitions == {0: 13_594_624}
    lay16 = L.plan([(t.name, t.device, t.dtype, t.shape, t.nbytes) for t in toy], 16, 1 << 20)
    assert lay16.partitions == {0: 13_569_888}
    # OPT-6.7B has no padding at A=4096 (every size is a multiple of 4096)
    lay = L.plan([(t.name, t.device, t.dtype, t.shape, t.nbytes) for t in inv], 4096, 1 << 20)
    assert lay.partitions == {0: 13_316_947_968}


def test_under_1mib_fractions():
    """62.4% of OPT tensors and 22.3% of LLaMA-2 tensors are < 1 MiB."""
    inv, _ = models.model_inventory("opt-6.7b")
    frac = sum(t.nbytes < (1 << 20) for t in inv) / len(inv)
    assert math.isclose(frac, 0.624, abs_tol=0.001)
    inv = models.llama2(8192, 80, 28672, 1024)
    frac = sum(t.nbytes < (1 << 20) for t in inv) / len(inv)
    assert math.isclose(frac, 0.223, abs_tol=0.001)


@pytest.mark.parametrize("Ld,C", [(0, 16), (16, 16), (17, 16), (100, 7), (13_594_624, 1 << 20), (1 << 30, 16 << 20)])
def test_chunks(Ld, C):
    ch = L.chunks(Ld, C)
    assert len(ch) == -(-Ld // C)
    assert sum(hi - lo for lo, hi in ch) == Ld
    for k, (lo, hi) in enumerate(ch):
        assert lo == k * C
        assert hi - lo == C or k == len(ch) - 1
