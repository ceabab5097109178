"""Pins of oracle.fletcher: textbook vectors, the sequential
definition against the closed form, the ordered combine, special cases, and brute-force
single-byte-change detection."""
import os

import numpy as np
import pytest

from oracle import fletcher

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "fletcher64_vectors.txt")


def _vectors():
    out = []
    for line in open(GOLDEN):
        line = line.strip()
        if line and not line.startswith("#"):
            msg, hx = line.split()
            out.append((msg.encode(), int(hx, 16)))
    return out


@pytest.mark.parametrize("msg,expect", _vectors())
def test_textbook_vectors(msg, expect):
    assert fletcher.f64_sequential(msg) == expect
    assert fletcher.f64_closed(msg) == expect


def test_hand_computed_two_words():
    # w0 = 1, w1 = 2: s1 = 3, s2 = 1 + 3 = 4
    x = (1).to_bytes(4, "little") + (2).to_bytes(4, "little")
    assert fletcher.f64_sequential(x) == (4 << 32) | 3
    assert fletcher.f64_closed(x) == (4 << 32) | 3


@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 63, 4096 * 4, 4096 * 4 + 12, 3 * 4096 * 4 + 7, 65536])
def test_closed_form_equals_sequential(n):
    rng = np.random.default_rng(n)
    x = rng.integers(0, 256, size=n, dtype=np.uint8).tobytes()
    assert fletcher.f64_closed(x) == fletcher.f64_sequential(x)


def test_closed_form_high_words():
    # all words = M-1 (max residue) stress the uint64 bounds of the closed form
    x = np.full(3 * 4096 + 5, 0xFFFFFFFE, dtype="<u4").tobytes()
    assert fletcher.f64_closed(x) == fletcher.f64_sequential(x)


def test_zero_and_all_ones_blind_spot():
    assert fletcher.f64_closed(bytes(4096)) == 0
    # 0xFFFFFFFF == 0 (mod M): the known Fletcher blind spot (Q8)
    assert fletcher.f64_closed(b"\xff" * 4096) == 0
    assert fletcher.f64_sequential(b"\xff" * 64) == 0


def test_ordered_combine_random_splits():
    rng = np.random.default_rng(7)
    x = rng.integers(0, 256, size=4 * 3000, dtype=np.uint8).tobytes()
    whole = fletcher.f64_sequential(x)
    for _ in range(200):
        k = int(rng.integers(0, 3001)) * 4
        fx = fletcher.f64_closed(x[:k])
        fy = fletcher.f64_closed(x[k:])
        assert fletcher.combine(fx, fy, (len(x) - k) // 4) == whole


def test_block_checksums_and_chunk_combine():
    rng = np.random.default_rng(3)
    B = 4096
    part = rng.integers(0, 256, size=5 * B + 2048, dtype=np.uint8)
    cs = fletcher.block_checksums(part, B)
    assert len(cs) == 6
    for j, c in enumerate(cs):
        assert c == fletcher.f64_sequential(part[j * B:(j + 1) * B].tobytes())
    # chunk of blocks 1..3 via combine == direct
    chunk = fletcher.chunk_checksum(cs[1:4], [B // 4] * 3)
    assert chunk == fletcher.f64_sequential(part[B:4 * B].tobytes())


def test_every_single_byte_change_detected():
    """Brute force: each single-byte change of a random 64-byte message is
    detected (delta = D*256^k with 0 < |delta| < M cannot vanish mod M)."""
    rng = np.random.default_rng(11)
    x = bytearray(rng.integers(0, 256, size=64, dtype=np.uint8).tobytes())
    ref = fletcher.f64_closed(bytes(x))
    misses = 0
    for i in range(len(x)):
        orig = x[i]
        for v in range(256):
            if v == orig:
                continue
            x[i] = v
            misses += fletcher.f64_closed(bytes(x)) == ref
        x[i] = orig
    assert misses == 0


@pytest.mark.parametrize("nbytes,fill", [(1 << 20, None), ((1 << 20) + 12, None), (3 << 20, None),
                                         (1 << 20, 0xFFFFFFFE), (1 << 20, 0xFFFFFFFF)])
def test_closed_form_equals_sequential_at_block_size(nbytes, fill):
    """block_checksums applies f64_closed to whole 1 MiB blocks (64 of its 4096-word
    sub-blocks): pin it there against the literal sequential definition, including the
    largest residue words (0xFFFFFFFE) that maximise every uint64 partial sum and the
    0xFFFFFFFF == 0 words of the blind spot."""
    if fill is None:
        x = np.random.default_rng(nbytes).integers(0, 256, size=nbytes, dtype=np.uint8).tobytes()
    else:
        x = np.full(nbytes // 4, fill, dtype="<u4").tobytes()
    assert fletcher.f64_closed(x) == fletcher.f64_sequential(x)
