"""Tensor index writer/reader -- SURVEY.md §8(c) O4 and its binary format (reading Q6/Q7).

PAPER.md P:546-547: "a tensor index file ... maps tensor names to a tuple of GPU id,
offset, and size".  SPEC.md S:79: "self-describing little-endian binary record stream
with a magic number and format_version=1".  The record layout (all little-endian):

  header : "SLLMIDX1" | u32 version=1 | u32 flags(bit0 = has block checksums) | u64 A
           | u64 B (0 iff no checksums) | u32 n_partitions | u32 n_tensors | u64 payload_bytes
           | u32 model_id_len | model_id | zero pad to 8
  parts  : n_partitions x { i32 device | u32 0 | u64 L_d | u64 n_tensors_d | u64 n_blocks }
           (strictly ascending device id)
  tensors: n_tensors x { u32 name_len | name | i32 device | u8 dtype | u8 ndim | u16 0
           | u64 offset | u64 size | ndim x i64 shape | zero pad to 8 }   (global source order)
  cksums : per partition, in order: n_blocks x u64 Fletcher-64
  trailer: u64 Fletcher-64(every preceding byte) | u64 total index length

Every read-side check of SURVEY §8(c) raises FormatError; with the trailer length and
the "records end exactly at len-16" rule every truncation is detectable.
"""
from __future__ import annotations

import math
import struct
from typing import Dict, List

from . import fletcher
from .errors import FormatError
from .layout import CODE, NAME_OF_CODE, WIDTH, MAX_NDIM, MAX_BLOCK, Entry, Layout, is_pow2

MAGIC = b"SLLMIDX1"
VERSION = 1
FLAG_CHECKSUMS = 1


def _pad8(buf: bytearray) -> None:
    buf += b"\x00" * ((-len(buf)) % 8)


def write(layout: Layout) -> bytes:
    """O4 writer: the index bytes of a layout (checksums must be filled when B != 0)."""
    devs = layout.devices()
    has_cs = layout.block != 0
    mid = layout.model_id.encode("utf-8")
    out = bytearray()
    out += MAGIC
    out += struct.pack("<IIQQIIQI", VERSION, FLAG_CHECKSUMS if has_cs else 0, layout.align, layout.block,
                       len(devs), len(layout.entries), layout.payload_bytes, len(mid))
    out += mid
    _pad8(out)
    for d in devs:
        L = layout.partitions[d]
        nt = sum(1 for e in layout.entries if e.device == d)
        nb = (L + layout.block - 1) // layout.block if has_cs else 0
        out += struct.pack("<iIQQQ", d, 0, L, nt, nb)
    for e in layout.entries:
        nm = e.name.encode("utf-8")
        out += struct.pack("<I", len(nm)) + nm
        out += struct.pack("<iBBHQQ", e.device, CODE[e.dtype], len(e.shape), 0, e.offset, e.size)
        out += struct.pack(f"<{len(e.shape)}q", *e.shape)
        _pad8(out)
    if has_cs:
        for d in devs:
            cs = layout.checksums[d]
            out += struct.pack(f"<{len(cs)}Q", *cs)
    out += struct.pack("<Q", fletcher.f64_closed(bytes(out)))
    out += struct.pack("<Q", len(out) + 8)
    return bytes(out)


class _Reader:
    def __init__(self, blob: bytes, limit: int):
        self.b = blob
        self.p = 0
        self.limit = limit

    def take(self, n: int) -> bytes:
        if n < 0 or self.p + n > self.limit:
            raise FormatError(f"truncated index: need {n} bytes at {self.p}, records end at {self.limit}")
        v = self.b[self.p:self.p + n]
        self.p += n
        return v

    def unpack(self, fmt: str):
        return struct.unpack(fmt, self.take(struct.calcsize(fmt)))

    def pad8(self) -> None:
        pad = self.take((-self.p) % 8)
        if any(pad):
            raise FormatError("non-zero padding")


def read(blob: bytes) -> Layout:
    """O4 reader with the full read-side validation list of SURVEY §8(c)."""
    blob = bytes(blob)
    n = len(blob)
    if n < 16 + 56:
        raise FormatError(f"index too short ({n} bytes)")
    if n % 8:
        raise FormatError("index length not a multiple of 8")
    cs_stored, total = struct.unpack("<QQ", blob[n - 16:])
    if total != n:
        raise FormatError(f"trailer length {total} != file length {n}")
    if fletcher.f64_closed(blob[:n - 16]) != cs_stored:
        raise FormatError("index self-checksum mismatch")
    r = _Reader(blob, n - 16)
    if r.take(8) != MAGIC:
        raise FormatError("bad magic")
    version, flags, A, B, n_parts, n_tensors, payload, mid_len = r.unpack("<IIQQIIQI")
    if version != VERSION:
        raise FormatError(f"unsupported version {version}")
    if flags & ~FLAG_CHECKSUMS:
        raise FormatError(f"unknown flag bits {flags:#x}")
    if not (is_pow2(A) and A >= 16):
        raise FormatError(f"bad alignment {A}")
    has_cs = bool(flags & FLAG_CHECKSUMS)
    if has_cs:
        if not (is_pow2(B) and B % A == 0):
            raise FormatError(f"bad block size {B}")
    elif B != 0:
        raise FormatError("block size set without checksum flag")
    if A > MAX_BLOCK or B > MAX_BLOCK:
        raise FormatError("alignment / block size above 256 MiB (DESIGN.md Q8)")
    try:
        model_id = r.take(mid_len).decode("utf-8")
    except UnicodeDecodeError as ex:
        raise FormatError("model id not UTF-8") from ex
    r.pad8()
    parts: Dict[int, int] = {}
    part_nt: Dict[int, int] = {}
    part_nb: Dict[int, int] = {}
    prev = None
    for _ in range(n_parts):
        d, zero, L, nt, nb = r.unpack("<iIQQQ")
        if zero != 0:
            raise FormatError("non-zero reserved field")
        if d < 0 or (prev is not None and d <= prev):
            raise FormatError("partition device ids not strictly ascending / negative")
        prev = d
        if L % A != 0 or L == 0:
            raise FormatError(f"partition {d} length {L} not a positive multiple of A")
        exp_nb = (L + B - 1) // B if has_cs else 0
        if nb != exp_nb:
            raise FormatError(f"partition {d}: n_blocks {nb} != {exp_nb}")
        if nt == 0:
            raise FormatError(f"partition {d} has no tensors")
        parts[d], part_nt[d], part_nb[d] = L, nt, nb
    entries: List[Entry] = []
    names = set()
    for _ in range(n_tensors):
        (nl,) = r.unpack("<I")
        if nl == 0:
            raise FormatError("empty tensor name")
        try:
            name = r.take(nl).decode("utf-8")
        except UnicodeDecodeError as ex:
            raise FormatError("tensor name not UTF-8") from ex
        if name in names:
            raise FormatError(f"duplicate tensor name {name!r}")
        names.add(name)
        d, dt, ndim, zero, off, size = r.unpack("<iBBHQQ")
        if zero != 0:
            raise FormatError("non-zero reserved field")
        if d not in parts:
            raise FormatError(f"tensor {name!r} on unknown device {d}")
        if dt not in NAME_OF_CODE:
            raise FormatError(f"unknown dtype code {dt}")
        if ndim > MAX_NDIM:
            raise FormatError(f"ndim {ndim} > {MAX_NDIM}")
        shape = r.unpack(f"<{ndim}q")
        r.pad8()
        if any(s <= 0 for s in shape):
            raise FormatError(f"non-positive dimension in {name!r}")
        dtype = NAME_OF_CODE[dt]
        if size != math.prod(shape) * WIDTH[dtype]:
            raise FormatError(f"size of {name!r} != prod(shape) * width")
        if off % A != 0:
            raise FormatError(f"offset of {name!r} not aligned")
        if off + size > parts[d]:
            raise FormatError(f"{name!r} extends past its partition")
        entries.append(Entry(name, d, dtype, tuple(shape), off, size))
    for d in parts:
        es = sorted((e for e in entries if e.device == d), key=lambda e: e.offset)
        if len(es) != part_nt[d]:
            raise FormatError(f"partition {d}: tensor count mismatch")
        for a, b in zip(es, es[1:]):
            if b.offset < a.offset + a.size:
                raise FormatError(f"overlapping tensors {a.name!r} and {b.name!r}")
    if sum(e.size for e in entries) != payload:
        raise FormatError("payload_bytes mismatch")
    checksums: Dict[int, List[int]] = {}
    if has_cs:
        for d in sorted(parts):
            checksums[d] = list(r.unpack(f"<{part_nb[d]}Q"))
            if any((c & fletcher.M) == fletcher.M or (c >> 32) == fletcher.M for c in checksums[d]):
                raise FormatError(f"non-canonical block checksum in partition {d}")
    if r.p != n - 16:
        raise FormatError("records do not end at the trailer")
    return Layout(A, B, model_id, parts, entries, checksums)
