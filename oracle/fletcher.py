"""Fletcher-64 over 32-bit words -- SURVEY.md §8(c) O7/O8 (reading Q8 in DESIGN.md).

The paper has no integrity check ("the paper is silent"); the
north star requires "a fused per-chunk checksum ... to verify integrity".  The
build's reading is the textbook Fletcher-64:

    words  w_i = little-endian u32 at byte 4i (tail zero-padded), n = ceil(|x|/4),
    M = 2**32 - 1
    sequential:   s1 = s2 = 0; for i: s1 = (s1 + w_i) mod M; s2 = (s2 + s1) mod M
    result:       (s2 << 32) | s1
    closed form:  s1 = sum w_i mod M;  s2 = sum (n - i) * w_i mod M
    combine X||Y: s1 = s1X + s1Y;  s2 = s2X + nY*s1X + s2Y   (mod M)

Both halves are canonical residues in [0, M-1] (so 0xFFFFFFFF never appears).
Block checksums (O8): cs[j] = F64(P[j*B : min((j+1)*B, L)]).
"""
from __future__ import annotations

from typing import Iterable, List, Tuple

import numpy as np

M = 0xFFFFFFFF
SUB = 4096  # closed-form sub-block (words) so every uint64 partial sum is exact


def words(x) -> List[int]:
    """The u32 little-endian word sequence of O7 (tail zero-padded to 4 bytes)."""
    b = bytes(x)
    if len(b) % 4:
        b = b + b"\x00" * (4 - len(b) % 4)
    return [int.from_bytes(b[i:i + 4], "little") for i in range(0, len(b), 4)]


def f64_sequential(x) -> int:
    """O7 sequential form, literally.  Slow: for small inputs and as the pin of the others."""
    s1 = s2 = 0
    for w in words(x):
        s1 = (s1 + w) % M
        s2 = (s2 + s1) % M
    return (s2 << 32) | s1


def _as_words(x) -> np.ndarray:
    a = np.frombuffer(memoryview(x).cast("B"), dtype=np.uint8) if not isinstance(x, np.ndarray) else x.reshape(-1).view(np.uint8)
    if a.size % 4:
        a = np.concatenate([a, np.zeros(4 - a.size % 4, dtype=np.uint8)])
    return a.view("<u4")


def f64_closed(x) -> int:
    """O7 closed form: s1 = sum w_i, s2 = sum (n - i) w_i, both mod M.

    Evaluated over sub-blocks k of SUB words: with S_k = sum_j w_{k,j} and
    U_k = sum_j j * w_{k,j} (j local), sum_i (n - i) w_i = sum_k (n - SUB*k) S_k - U_k.
    Every uint64 intermediate is < 2**64 (S_k < 2**44, U_k < 2**56, residues < 2**32)."""
    w = _as_words(x)
    n = int(w.size)
    if n == 0:
        return 0
    nsub = (n + SUB - 1) // SUB
    W = np.zeros(nsub * SUB, dtype=np.uint64)
    W[:n] = w
    W = W.reshape(nsub, SUB)
    S = W.sum(axis=1, dtype=np.uint64)
    U = (W * np.arange(SUB, dtype=np.uint64)[None, :]).sum(axis=1, dtype=np.uint64)
    weight = (np.uint64(n) - np.uint64(SUB) * np.arange(nsub, dtype=np.uint64)) % np.uint64(M)
    s1 = int(S.sum(dtype=np.uint64)) % M
    t = int(((weight * (S % np.uint64(M))) % np.uint64(M)).sum(dtype=np.uint64))
    u = int((U % np.uint64(M)).sum(dtype=np.uint64))
    s2 = (t - u) % M
    return (s2 << 32) | s1


def split(f: int) -> Tuple[int, int]:
    return f & M, f >> 32


def combine(fx: int, fy: int, ny_words: int) -> int:
    """O7 ordered combine of F64(X) and F64(Y) for X||Y, Y having ny_words words."""
    s1x, s2x = split(fx)
    s1y, s2y = split(fy)
    s1 = (s1x + s1y) % M
    s2 = (s2x + ny_words * s1x + s2y) % M
    return (s2 << 32) | s1


def block_checksums(part, block: int) -> List[int]:
    """O8: one F64 per block of ``block`` bytes of a partition (last block may be short)."""
    a = part if isinstance(part, np.ndarray) else np.frombuffer(memoryview(part).cast("B"), dtype=np.uint8)
    a = a.reshape(-1).view(np.uint8)
    return [f64_closed(a[j:j + block]) for j in range(0, a.size, block)]


def chunk_checksum(block_cs: Iterable[int], block_words: Iterable[int]) -> int:
    """F64 of a chunk from its blocks' checksums, by the ordered combine (O8)."""
    acc = 0
    for f, nw in zip(block_cs, block_words):
        acc = combine(acc, f, nw)
    return acc
