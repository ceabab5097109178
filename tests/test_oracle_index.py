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
