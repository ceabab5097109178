"""The native converter / index codec / host Fletcher-64 against the oracle (CPU only).

Acceptance criterion 1 of SPEC.md S:570 adapted to the converter: 200 randomized
checkpoints (1-4 devices, up to 10k tensors, <= 256 MiB total -- here smaller totals
keep the CPU suite fast) convert to partitions and an index that are BYTE-IDENTICAL to
the oracle's.  The native side never sees the oracle's output: both start from the same
synth inventory + payloads."""
import copy
import os

import numpy as np
import pytest

import paper_2401_14351_b200 as sllm
from oracle import fletcher, index as oindex, layout as olayout
from synth import models, payload


def _native_convert(inv, payloads, A, B, model_id="m"):
    tensors = [(t.name, t.device, t.dtype, t.shape) for t in inv]
    idx = sllm.Index.plan(tensors, A, B, model_id)
    parts = [np.empty(p.length, dtype=np.uint8) for p in idx.partitions]
    for b in parts:
        b.fill(0xA5)  # garbage: the converter must zero padding itself
    srcs = [(t.name, t.device, t.dtype, t.shape, p.ctypes.data) for t, p in zip(inv, payloads)]
    idx.convert_into(srcs, [b.ctypes.data for b in parts])
    return idx, parts


def _oracle_convert(inv, payloads, A, B, model_id="m"):
    lay, parts = olayout.convert([(t.name, t.device, t.dtype, t.shape, p) for t, p in zip(inv, payloads)],
                                 A, B, model_id)
    return lay, parts


def _case(seed, n_max=400, total=1 << 20):
    rng = np.random.default_rng(seed)
    inv = models.random_inventory(rng, int(rng.integers(1, n_max)), int(rng.integers(1, 5)), total)
    payloads = [payload.payload_bytes(seed, e, t.nbytes) for e, t in enumerate(inv)]
    A = int(rng.choice([16, 64, 4096]))
    B = int(rng.choice([0, A, 4096 * 4, 1 << 16])) if A <= 4096 else 0
    if B and B % A:
        B = 0
    return inv, payloads, A, B


def test_toy_byte_identical():
    inv = models.toy()
    payloads = [payload.payload_bytes(0, e, t.nbytes) for e, t in enumerate(inv)]
    idx, parts = _native_convert(inv, payloads, 4096, 1 << 20, "toy")
    lay, oparts = _oracle_convert(inv, payloads, 4096, 1 << 20, "toy")
    assert idx.serialize() == oindex.write(lay)
    assert [p.length for p in idx.partitions] == [13_594_624]
    assert np.array_equal(parts[0], oparts[0])


@pytest.mark.parametrize("seed", range(200))
def test_random_checkpoints_byte_identical(seed):
    inv, payloads, A, B = _case(seed, n_max=300 if seed % 10 else 3000, total=(1 << 20) if seed % 10 else (4 << 20))
    idx, parts = _native_convert(inv, payloads, A, B)
    lay, oparts = _oracle_convert(inv, payloads, A, B)
    assert idx.serialize() == oindex.write(lay)
    devs = lay.devices()
    assert len(parts) == len(devs)
    for p, d in zip(parts, devs):
        assert np.array_equal(p, oparts[d])


def test_native_parses_oracle_index_and_back():
    for seed in range(20):
        inv, payloads, A, B = _case(1000 + seed)
        lay, _ = _oracle_convert(inv, payloads, A, B, f"model-{seed}")
        blob = oindex.write(lay)
        idx = sllm.Index.from_bytes(blob)
        assert idx.serialize() == blob
        info = idx.info()
        assert info["model_id"] == f"model-{seed}" and info["payload_bytes"] == lay.payload_bytes
        assert idx.counts() == (len(lay.entries), len(lay.devices()))
        for t, e in zip(idx.tensors, lay.entries):
            assert (t.name, t.device, t.dtype, t.shape, t.offset, t.nbytes) == \
                (e.name, e.device, e.dtype, e.shape, e.offset, e.size)
        for p, d in enumerate(lay.devices()):
            if B:
                assert idx.block_checksums(p).tolist() == lay.checksums[d]


def test_native_rejects_every_truncation_and_crafted_errors():
    inv = models.toy()
    payloads = [payload.payload_bytes(0, e, t.nbytes) for e, t in enumerate(inv)]
    lay, _ = _oracle_convert(inv, payloads, 4096, 1 << 20, "toy")
    blob = oindex.write(lay)
    for n in range(len(blob)):
        with pytest.raises(sllm.SllmError) as ex:
            sllm.Index.from_bytes(blob[:n])
        assert ex.value.status == 3
    for mutate in (lambda L: setattr(L.entries[1], "offset", L.entries[0].offset + 4096),
                   lambda L: setattr(L.entries[-1], "offset", L.entries[-1].offset + 16),
                   lambda L: setattr(L.entries[3], "shape", (7,)),
                   lambda L: L.partitions.__setitem__(0, L.partitions[0] + 16),
                   lambda L: setattr(L.entries[2], "name", L.entries[1].name)):
        bad = copy.deepcopy(lay)
        mutate(bad)
        with pytest.raises(sllm.SllmError) as ex:
            sllm.Index.from_bytes(oindex.write(bad))
        assert ex.value.status == 3
    rng = np.random.default_rng(2)
    for pos in rng.choice(len(blob), size=200, replace=False):
        b = bytearray(blob)
        b[pos] ^= 0x10
        with pytest.raises(sllm.SllmError):
            sllm.Index.from_bytes(bytes(b))


def test_conversion_errors():
    with pytest.raises(sllm.SllmError) as ex:
        sllm.Index.plan([("a", 0, "u8", (4,)), ("a", 0, "u8", (4,))])
    assert ex.value.status == 2
    with pytest.raises(sllm.SllmError) as ex:
        sllm.Index.plan([("a", 0, "u8", (0,))])
    assert ex.value.status == 2
    with pytest.raises(sllm.SllmError) as ex:
        sllm.Index.plan([("a", 0, "u8", (4,))], align=8)
    assert ex.value.status == 1
    idx = sllm.Index.plan([], 4096, 1 << 20)
    assert idx.partitions == [] and idx.info()["n_tensors"] == 0


def test_spec_examples_native():
    idx = sllm.Index.plan([("a", 0, "u8", (10,)), ("b", 0, "u8", (6,))], 4096, 0)
    assert [t.offset for t in idx.tensors] == [0, 4096] and idx.partitions[0].length == 8192
    assert idx.address("b", [1_000_000]) == (0, 1_004_096)
    with pytest.raises(sllm.SllmError) as ex:
        idx.address("zz", [0])
    assert ex.value.status == 4


@pytest.mark.parametrize("n", [0, 1, 5, 64, 4095, 65536 * 4 + 3, 1 << 20])
def test_host_fletcher_matches_oracle(n):
    rng = np.random.default_rng(n)
    x = rng.integers(0, 256, size=n, dtype=np.uint8)
    ref = fletcher.f64_sequential(x.tobytes()) if n <= 4096 else fletcher.f64_closed(x)
    assert sllm.fletcher64(x) == ref


def test_host_fletcher_textbook():
    assert sllm.fletcher64(b"abcde") == 0xC8C6C527646362C6
    assert sllm.fletcher64(b"abcdefgh") == 0x312E2B28CCCAC8C6
    assert sllm.fletcher64(b"\xff" * 4096) == 0


def test_convert_to_files_and_read_partition(tmp_path):
    inv = models.llama2(256, 2, 512, 64, vocab=1024, tp=2)
    payloads = [payload.payload_bytes(7, e, t.nbytes) for e, t in enumerate(inv)]
    srcs = [(t.name, t.device, t.dtype, t.shape, p.ctypes.data) for t, p in zip(inv, payloads)]
    sllm.convert(srcs, str(tmp_path), 4096, 1 << 16, "tp2")
    lay, oparts = _oracle_convert(inv, payloads, 4096, 1 << 16, "tp2")
    assert open(tmp_path / "index.bin", "rb").read() == oindex.write(lay)
    idx = sllm.Index.open(str(tmp_path / "index.bin"))
    for p, d in enumerate(lay.devices()):
        assert open(tmp_path / f"part_{d}.bin", "rb").read() == oparts[d].tobytes()
        L = idx.partitions[p].length
        raw = np.zeros(L + 8192, np.uint8)
        off = (-raw.ctypes.data) % 4096
        dst = raw[off:off + L]
        sllm.lib()  # loaded
        from paper_2401_14351_b200 import _abi
        import ctypes
        _abi.check(sllm.lib().sllm_host_read_partition(str(tmp_path).encode(), idx.handle, p,
                                                       ctypes.c_void_p(dst.ctypes.data), 3))
        assert np.array_equal(dst, oparts[d])


def _reseal(b: bytearray) -> bytes:
    """Recompute the index trailer (self-checksum) after a crafted edit -- the edit must be
    caught by the structural checks, not by the checksum."""
    import struct
    n = len(b)
    b[n - 16:n - 8] = struct.pack("<Q", fletcher.f64_closed(bytes(b[:n - 16])))
    return bytes(b)


def test_native_rejects_crafted_counts_before_sizing_by_them():
    """A crafted (re-sealed) index whose tensor count or partition length promises more
    records / checksum tables than the blob holds is rejected with SLLM_E_FORMAT before
    anything is allocated by those counts (no multi-GB resize on bad input)."""
    import struct
    import time
    inv = models.toy()
    payloads = [payload.payload_bytes(0, e, t.nbytes) for e, t in enumerate(inv)]
    lay, _ = _oracle_convert(inv, payloads, 4096, 1 << 20, "toy")
    blob = oindex.write(lay)
    # header: magic 8 | version 4 | flags 4 | A 8 | B 8 | n_parts 4 | n_tensors 4 @36
    b = bytearray(blob)
    b[36:40] = struct.pack("<I", 0xFFFFFFFF)
    t0 = time.perf_counter()
    with pytest.raises(sllm.SllmError) as ex:
        sllm.Index.from_bytes(_reseal(b))
    assert ex.value.status == 3 and "tensor count" in str(ex.value)
    # partition record at 56 (header 52 B + "toy" padded to 8): L_d @64, n_blocks @80;
    # L_d = 2^50 with the consistent n_blocks = 2^30 would need an 8 GiB checksum table
    b = bytearray(blob)
    b[64:72] = struct.pack("<Q", 1 << 50)
    b[80:88] = struct.pack("<Q", (1 << 50) >> 20)
    with pytest.raises(sllm.SllmError) as ex:
        sllm.Index.from_bytes(_reseal(b))
    assert ex.value.status == 3 and "checksum tables" in str(ex.value)
    assert time.perf_counter() - t0 < 5


@pytest.mark.parametrize("block", [1 << 28, 1 << 29])
def test_block_size_cap_both_sides(block):
    """DESIGN.md Q8 build limit: alignment and checksum block at most 256 MiB, in the oracle
    and in the library alike (plan -> INVALID, a crafted index -> FORMAT)."""
    from oracle.errors import FormatError, InvalidError
    t = [("a", 0, "u8", (64,))]
    if block <= 1 << 28:
        assert sllm.Index.plan(t, 4096, block).info()["block"] == block
        olayout.plan([(*x, 64) for x in t], 4096, block)
        return
    with pytest.raises(sllm.SllmError) as ex:
        sllm.Index.plan(t, 4096, block)
    assert ex.value.status == 1
    with pytest.raises(InvalidError):
        olayout.plan([(*x, 64) for x in t], 4096, block)
    # a sealed index at the cap, its B field raised past it and re-sealed
    import struct
    lay, _ = _oracle_convert([models.toy()[0]], [payload.payload_bytes(0, 0, models.toy()[0].nbytes)], 4096, 1 << 28)
    b = bytearray(oindex.write(lay))
    b[24:32] = struct.pack("<Q", block)
    with pytest.raises(sllm.SllmError) as ex:
        sllm.Index.from_bytes(_reseal(b))
    assert ex.value.status == 3
    with pytest.raises(FormatError):
        oindex.read(_reseal(b))
