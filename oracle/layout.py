"""Converter layout, partition bytes, addressing and chunk plan -- SURVEY.md §8(c) O1-O3, O5, O6.

PAPER.md P:545-547 (§Loading-Optimized Checkpoints): "tensors for each GPU are grouped
in partitions ... These files contain only the binary data of model parameters and
exclude metadata ...  a tensor index file ... maps tensor names to a tuple of GPU id,
offset, and size ...  The tensors are aligned with memory word sizes, facilitating
direct computation of memory address."  Readings: alignment A (Q1),
source order within a partition (Q2), zero padding (Q3), L_d = align_up(last
end, A) (Q4), devices ascending.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple

import numpy as np

from .errors import ConversionError, InvalidError, OracleLookupError

# Oracle's own copy of the dtype table; deliberately not imported.
# (Q12: SPEC's F16/F32/I8/I64 plus BF16/U8, and the remaining safetensors dtypes I32, F64, I16,
# BOOL, F8_E4M3, F8_E5M2 -- the dtype only fixes the element width)
WIDTH = {"f16": 2, "bf16": 2, "f32": 4, "i8": 1, "u8": 1, "i64": 8,
         "i32": 4, "f64": 8, "i16": 2, "bool": 1, "f8e4m3": 1, "f8e5m2": 1}
CODE = {"f16": 0, "bf16": 1, "f32": 2, "i8": 3, "u8": 4, "i64": 5,
        "i32": 6, "f64": 7, "i16": 8, "bool": 9, "f8e4m3": 10, "f8e5m2": 11}
NAME_OF_CODE = {v: k for k, v in CODE.items()}
MAX_NDIM = 8
# DESIGN.md Q8 (build limit): alignment and checksum block are at most 256 MiB
MAX_BLOCK = 1 << 28


def is_pow2(x: int) -> bool:
    return x > 0 and (x & (x - 1)) == 0


def align_up(x: int, a: int) -> int:
    return (x + a - 1) // a * a


@dataclass
class Entry:
    name: str
    device: int
    dtype: str
    shape: Tuple[int, ...]
    offset: int
    size: int


@dataclass
class Layout:
    align: int
    block: int
    model_id: str
    partitions: Dict[int, int]            # device id -> L_d  (ascending when iterated via devices())
    entries: List[Entry]                  # global source order
    checksums: Dict[int, List[int]] = field(default_factory=dict)  # device -> block table

    def devices(self) -> List[int]:
        return sorted(self.partitions)

    @property
    def payload_bytes(self) -> int:
        return sum(e.size for e in self.entries)


def validate_params(align: int, block: int) -> None:
    """O1: A is a power of two >= 16; B is 0 (no checksums) or a power of two multiple of A."""
    if not (is_pow2(align) and align >= 16):
        raise InvalidError(f"alignment {align} must be a power of two >= 16")
    if block != 0 and not (is_pow2(block) and block % align == 0):
        raise InvalidError(f"block {block} must be a power of two multiple of the alignment")
    if align > MAX_BLOCK or block > MAX_BLOCK:
        raise InvalidError("alignment / block size above 256 MiB (DESIGN.md Q8)")


def validate_source(tensors: Sequence) -> None:
    """O1: unique non-empty names, known dtype, device >= 0, positive dims,
    rank <= 8, payload length == prod(shape) * width."""
    seen = set()
    for t in tensors:
        name, dev, dt, shape, payload = t
        if not isinstance(name, str) or name == "":
            raise ConversionError("empty tensor name")
        try:
            name.encode("utf-8")
        except UnicodeEncodeError as ex:
            raise ConversionError(f"name not UTF-8: {name!r}") from ex
        if name in seen:
            raise ConversionError(f"duplicate tensor name {name!r}")
        seen.add(name)
        if dt not in WIDTH:
            raise ConversionError(f"unknown dtype {dt!r}")
        if dev < 0:
            raise ConversionError(f"negative device id for {name!r}")
        if len(shape) > MAX_NDIM or any(int(s) <= 0 for s in shape):
            raise ConversionError(f"bad shape {shape} for {name!r}")
        if len(payload) != math.prod(shape) * WIDTH[dt]:
            raise ConversionError(f"payload of {name!r} has {len(payload)} bytes, shape needs "
                                  f"{math.prod(shape) * WIDTH[dt]}")


def plan(tensors: Sequence, align: int, block: int, model_id: str = "") -> Layout:
    """O2 layout algorithm, literally: for each device d ascending, cursor = 0; for each
    tensor of d in source order: off = align_up(cursor, A); cursor = off + size.
    L_d = align_up(cursor, A).  ``tensors`` items: (name, device, dtype, shape, payload_or_size)."""
    validate_params(align, block)
    validate_source([t if not isinstance(t[4], int) else (t[0], t[1], t[2], t[3], _Len(t[4]))
                     for t in tensors])
    offsets: Dict[int, int] = {}
    partitions: Dict[int, int] = {}
    for d in sorted({t[1] for t in tensors}):
        cursor = 0
        for i, t in enumerate(tensors):
            if t[1] != d:
                continue
            size = _size(t)
            off = align_up(cursor, align)
            offsets[i] = off
            cursor = off + size
        partitions[d] = align_up(cursor, align)
    entries = [Entry(t[0], t[1], t[2], tuple(int(s) for s in t[3]), offsets[i], _size(t))
               for i, t in enumerate(tensors)]
    return Layout(align, block, model_id, partitions, entries)


class _Len:
    """Stand-in payload of a given length (plan() needs sizes only)."""

    def __init__(self, n):
        self.n = n

    def __len__(self):
        return self.n


def _size(t) -> int:
    p = t[4]
    return p if isinstance(p, int) else len(p)


def partition_bytes(layout: Layout, payloads: Sequence) -> Dict[int, np.ndarray]:
    """O3: P_d[off_e : off_e + size_e] = payload_e; every other byte is 0x00 (Q3)."""
    parts = {d: np.zeros(L, dtype=np.uint8) for d, L in layout.partitions.items()}
    for e, p in zip(layout.entries, payloads):
        parts[e.device][e.offset:e.offset + e.size] = np.frombuffer(memoryview(p).cast("B"), dtype=np.uint8) \
            if not isinstance(p, np.ndarray) else p.reshape(-1).view(np.uint8)
    return parts


def convert(tensors: Sequence, align: int = 4096, block: int = 1 << 20, model_id: str = ""):
    """O1-O4 + O8: validate, lay out, build partitions, fill block checksums.
    Returns (layout, {device: partition bytes}).  Index bytes: oracle.index.write(layout)."""
    from . import fletcher
    layout = plan(tensors, align, block, model_id)
    parts = partition_bytes(layout, [t[4] for t in tensors])
    if block:
        layout.checksums = {d: fletcher.block_checksums(parts[d], block) for d in layout.devices()}
    return layout, parts


def address(layout: Layout, name: str, bases: Dict[int, int]) -> Tuple[int, int]:
    """O5 ("base + offset"): (device, base_device + offset)."""
    for e in layout.entries:
        if e.name == name:
            return e.device, bases[e.device] + e.offset
    raise OracleLookupError(name)


def chunks(length: int, chunk: int) -> List[Tuple[int, int]]:
    """O6 ("divides each partition into chunks with equal size (except for the last
    one)"): chunk k covers [k*C, min((k+1)*C, L)) for k < ceil(L/C)."""
    if chunk <= 0:
        raise InvalidError("chunk size must be positive")
    return [(k * chunk, min((k + 1) * chunk, length)) for k in range((length + chunk - 1) // chunk)]
