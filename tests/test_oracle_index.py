"""Pins of oracle.index: round trip, every truncation
rejected, crafted overlap / misalignment / corruption rejected, and the
committed golden index of the S:49 example."""
import copy
import os
import struct

import numpy as np
import pytest

from oracle import fletcher, index, layout as L
from oracle.errors import FormatError
from synth import models, payload

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def toy_layout():
    inv = models.toy()
    tensors = [(t.name, t.device, t.dtype, t.shape, payload.payload_bytes(0, e, t.nbytes))
               for e, t in enumerate(inv)]
    return L.convert(tensors, 4096, 1 << 20, "toy")


def test_roundtrip_toy():
    lay, _ = toy_layout()
    blob = index.write(lay)
    back = index.read(blob)
    assert back == lay
    assert len(blob) % 8 == 0


@pytest.mark.parametrize("seed", range(5))
def test_roundtrip_random(seed):
    rng = np.random.default_rng(100 + seed)
    inv = models.random_inventory(rng, 200, 3, 1 << 20)
    tensors = [(t.name, t.device, t.dtype, t.shape, payload.payload_bytes(seed, e, t.nbytes))
               for e, t in enumerate(inv)]
    lay, _ = L.convert(tensors, 256, 4096, f"rand{seed}")
    assert index.read(index.write(lay)) == lay
    lay0 = copy.deepcopy(lay)
    lay0.block = 0
    lay0.checksums = {}
    assert index.read(index.write(lay0)) == lay0


def test_every_truncation_rejected():
    lay, _ = toy_layout()
    blob = index.write(lay)
    for n in range(len(blob)):
        with pytest.raises(FormatError):
            index.read(blob[:n])


def _rewrite(lay):
    """write() does not validate, so a mutated layout yields a well-formed-looking file
    with a valid trailer -- the 'hand-crafted' corrupt index of S:60."""
    return index.write(lay)


def test_crafted_overlap_rejected():
    lay, _ = toy_layout()
    bad = copy.deepcopy(lay)
    bad.entries[1].offset = bad.entries[0].offset + 4096   # overlaps entry 0 (3 MiB long)
    with pytest.raises(FormatError, match="overlap"):
        index.read(_rewrite(bad))


def test_crafted_misaligned_rejected():
    lay, _ = toy_layout()
    bad = copy.deepcopy(lay)
    bad.entries[-1].offset += 8
    with pytest.raises(FormatError, match="aligned"):
        index.read(_rewrite(bad))


def test_crafted_out_of_partition_and_sizes():
    lay, _ = toy_layout()
    bad = copy.deepcopy(lay)
    bad.entries[-1].offset = lay.partitions[0]
    with pytest.raises(FormatError):
        index.read(_rewrite(bad))
    bad = copy.deepcopy(lay)
    bad.entries[3].shape = (1, 2)
    with pytest.raises(FormatError, match="size"):
        index.read(_rewrite(bad))
    bad = copy.deepcopy(lay)
    bad.partitions[0] += 8
    with pytest.raises(FormatError):
        index.read(_rewrite(bad))


def test_any_byte_flip_rejected():
    lay, _ = toy_layout()
    blob = bytearray(index.write(lay))
    rng = np.random.default_rng(1)
    for pos in rng.choice(len(blob), size=300, replace=False):
        b = bytearray(blob)
        b[pos] ^= 1 << int(rng.integers(0, 8))
        with pytest.raises(FormatError):
            index.read(bytes(b))


def test_header_checks_with_fixed_trailer():
    lay, _ = toy_layout()
    blob = bytearray(index.write(lay))

    def refix(b):
        b = bytearray(b)
        n = len(b)
        b[n - 16:n - 8] = struct.pack("<Q", fletcher.f64_closed(bytes(b[:n - 16])))
        return bytes(b)

    for off, val in [(0, b"X"), (8, b"\x02"), (12, b"\x02"), (16, b"\x08")]:
        b = bytearray(blob)
        b[off:off + len(val)] = val
        with pytest.raises(FormatError):
            index.read(refix(b))


def test_golden_spec_example_index():
    """tests/golden/spec_s49_index.hex is written by tests/golden/make_golden.py, which
    calls only oracle/ (S:49 example: u8[10] + u8[6], A = 4096, B = 4096)."""
    blob = bytes.fromhex(open(os.path.join(GOLDEN, "spec_s49_index.hex")).read().strip())
    lay = index.read(blob)
    assert [(e.name, e.offset, e.size) for e in lay.entries] == [("a", 0, 10), ("b", 4096, 6)]
    assert lay.partitions == {0: 8192}
    # block checksums of the all-bytes 0x01 / 0x02 payloads, computed by the sequential form
    part = bytearray(8192)
    part[0:10] = b"\x01" * 10
    part[4096:4102] = b"\x02" * 6
    assert lay.checksums[0] == [fletcher.f64_sequential(bytes(part[:4096])),
                                fletcher.f64_sequential(bytes(part[4096:]))]


def test_golden_index_field_offsets():
    """Decode tests/golden/spec_s49_index.hex field by field at the byte offsets of the
    record layout in SURVEY §8(c) ("Proposed index binary format") -- without the oracle's
    reader -- and check every value against the S:49 worked example (u8[10] "a" + u8[6] "b",
    A = 4096, B = 4096, L = 8192).  Pins the writer's layout against the spec rather than
    against its own reader."""
    import struct
    blob = bytes.fromhex(open(os.path.join(GOLDEN, "spec_s49_index.hex")).read().strip())
    u32 = lambda o: struct.unpack_from("<I", blob, o)[0]  # noqa: E731
    u64 = lambda o: struct.unpack_from("<Q", blob, o)[0]  # noqa: E731
    i32 = lambda o: struct.unpack_from("<i", blob, o)[0]  # noqa: E731
    # header: char[8] | u32 version | u32 flags | u64 A | u64 B | u32 n_partitions |
    #         u32 n_tensors | u64 payload | u32 model_id_len | model_id | pad->8
    assert blob[0:8] == b"SLLMIDX1"
    assert (u32(8), u32(12), u64(16), u64(24), u32(32), u32(36), u64(40), u32(48)) == \
        (1, 1, 4096, 4096, 1, 2, 16, 8)
    assert blob[52:60] == b"spec-s49" and blob[60:64] == bytes(4)        # 60 -> pad to 64
    # parts: i32 device | u32 0 | u64 L | u64 n_tensors_d | u64 n_blocks
    assert (i32(64), u32(68), u64(72), u64(80), u64(88)) == (0, 0, 8192, 2, 2)
    # tensors: u32 name_len | name | i32 device | u8 dtype | u8 ndim | u16 0 | u64 offset |
    #          u64 size | ndim x i64 shape | pad->8   (dtype code 4 = U8)
    o = 96
    for name, off, size in ((b"a", 0, 10), (b"b", 4096, 6)):
        assert u32(o) == 1 and blob[o + 4:o + 5] == name
        o += 5
        assert (i32(o), blob[o + 4], blob[o + 5], struct.unpack_from("<H", blob, o + 6)[0]) == (0, 4, 1, 0)
        assert (u64(o + 8), u64(o + 16), struct.unpack_from("<q", blob, o + 24)[0]) == (off, size, size)
        o += 32
        pad = (-o) % 8
        assert blob[o:o + pad] == bytes(pad)
        o += pad
    # checksum table: 2 blocks of 1024 words; closed form written out with Python ints:
    # s1 = sum w_i, s2 = sum (n - i) w_i (mod 2^32 - 1)
    M = 0xFFFFFFFF

    def f64_words(ws, n):
        s1 = sum(ws) % M
        s2 = sum((n - i) * w for i, w in enumerate(ws)) % M
        return (s2 << 32) | s1
    block0 = f64_words([0x01010101, 0x01010101, 0x00000101], 1024)   # ten 0x01 bytes
    block1 = f64_words([0x02020202, 0x00000202], 1024)               # six 0x02 bytes
    assert (u64(o), u64(o + 8)) == (block0, block1)
    o += 16
    # trailer: u64 F64(all preceding bytes) | u64 total length
    assert u64(o + 8) == len(blob) == o + 16
    ws = list(struct.unpack_from(f"<{o // 4}I", blob, 0))
    assert u64(o) == f64_words(ws, len(ws))
