"""Converter front-end for .safetensors checkpoints (paper_2401_14351_b200/formats.py).

The input files are written by the independent ``safetensors`` package; the converted
checkpoint is read back with the oracle's own index reader (oracle/index.py), the layout is
re-derived by the oracle's layout algorithm from the index's tensor order, and every
tensor's bytes are compared with what ``safetensors.safe_open`` reads -- padding must be
zero, block checksums must equal the oracle's."""
import os

import numpy as np
import pytest

st_numpy = pytest.importorskip("safetensors.numpy")
from safetensors import safe_open  # noqa: E402

from paper_2401_14351_b200 import _abi, formats  # noqa: E402
from oracle import fletcher, index as oindex, layout as olayout  # noqa: E402


def _tensors(seed):
    rng = np.random.default_rng(seed)
    return {
        "model.embed.weight": rng.standard_normal((300, 64)).astype(np.float16),
        "model.layers.0.q.weight": rng.standard_normal((64, 64)).astype(np.float32),
        "model.layers.0.norm.bias": rng.standard_normal((33,)).astype(np.float16),   # 66 B
        "model.scale": np.array(1.5, dtype=np.float16),                              # scalar, 2 B
        "model.ids": rng.integers(-2**40, 2**40, size=(17,), dtype=np.int64),
        "model.qweight": rng.integers(-128, 127, size=(40, 24), dtype=np.int8),
        "model.mask": rng.integers(0, 255, size=(9, 3), dtype=np.uint8),
        "model.pos": rng.integers(-2**31, 2**31 - 1, size=(11,), dtype=np.int32),     # I32
        "model.freq": rng.standard_normal((5, 3)),                                     # F64
        "model.idx16": rng.integers(-2**15, 2**15 - 1, size=(7,), dtype=np.int16),    # I16
        "model.flags": rng.integers(0, 2, size=(13,)).astype(bool),                    # BOOL
    }


def _check(out_dir, files, device_of, A, B):
    blob = open(os.path.join(out_dir, "index.bin"), "rb").read()
    lay = oindex.read(blob)                       # oracle reader: every FormatError check
    ref = olayout.plan([(e.name, e.device, e.dtype, e.shape, e.size) for e in lay.entries], A, B)
    assert [(e.name, e.offset) for e in ref.entries] == [(e.name, e.offset) for e in lay.entries]
    assert ref.partitions == lay.partitions
    arrays = {}
    for f in files:
        with safe_open(f, framework="numpy") as h:
            for k in h.keys():
                arrays[k] = h.get_tensor(k)
    assert sorted(arrays) == sorted(e.name for e in lay.entries)
    for d in lay.devices():
        part = np.fromfile(os.path.join(out_dir, f"part_{d}.bin"), dtype=np.uint8)
        assert part.size == lay.partitions[d]
        covered = np.zeros(part.size, bool)
        for e in lay.entries:
            if e.device != d:
                continue
            assert e.device == device_of(e.name)
            want = np.ascontiguousarray(arrays[e.name]).reshape(-1).view(np.uint8)
            assert tuple(e.shape) == tuple(arrays[e.name].shape)
            assert np.array_equal(part[e.offset:e.offset + e.size], want), e.name
            covered[e.offset:e.offset + e.size] = True
        assert not part[~covered].any()          # Q3: padding is 0x00
        assert lay.checksums[d] == fletcher.block_checksums(part, B)


def test_single_file(tmp_path):
    f = str(tmp_path / "model.safetensors")
    st_numpy.save_file(_tensors(0), f)
    out = str(tmp_path / "ckpt")
    n = formats.convert_safetensors([f], out, align=4096, block=1 << 16, model_id="st-test")
    assert n == 11
    _check(out, [f], lambda name: 0, 4096, 1 << 16)


def test_sharded_files_to_two_partitions(tmp_path):
    t = _tensors(1)
    names = sorted(t)
    f1, f2 = str(tmp_path / "model-00001-of-00002.safetensors"), str(tmp_path / "model-00002-of-00002.safetensors")
    st_numpy.save_file({k: t[k] for k in names[:4]}, f1)
    st_numpy.save_file({k: t[k] for k in names[4:]}, f2)
    dev = lambda name: 1 if "layers" in name or "mask" in name else 0  # noqa: E731
    out = str(tmp_path / "ckpt")
    formats.convert_safetensors([f1, f2], out, device_of=dev, align=256, block=1 << 12)
    _check(out, [f1, f2], dev, 256, 1 << 12)


def test_rejects_unsupported_dtype_and_duplicates(tmp_path):
    f = str(tmp_path / "u16.safetensors")
    st_numpy.save_file({"w": np.zeros((4,), np.uint16)}, f)
    with pytest.raises(_abi.SllmError) as ex:
        formats.convert_safetensors([f], str(tmp_path / "o1"))
    assert ex.value.status == _abi.E_CONVERSION
    g = str(tmp_path / "g.safetensors")
    st_numpy.save_file({"w": np.zeros((4,), np.float16)}, g)
    with pytest.raises(_abi.SllmError) as ex:        # the same name in two shards
        formats.convert_safetensors([g, g], str(tmp_path / "o2"))
    assert ex.value.status == _abi.E_CONVERSION


def test_cli_convert_and_info(tmp_path):
    import json
    import subprocess
    import sys
    f = str(tmp_path / "m.safetensors")
    st_numpy.save_file(_tensors(2), f)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {**os.environ, "PYTHONPATH": root}
    out = str(tmp_path / "ckpt")
    r = subprocess.run([sys.executable, "-m", "paper_2401_14351_b200", "convert", "--out", out, "--block", "65536", f],
                       capture_output=True, text=True, env=env)
    assert r.returncode == 0, r.stderr
    assert json.loads(r.stdout)["converted_tensors"] == 11
    _check(out, [f], lambda name: 0, 4096, 1 << 16)
    r = subprocess.run([sys.executable, "-m", "paper_2401_14351_b200", "info", out], capture_output=True, text=True,
                       env=env)
    assert r.returncode == 0, r.stderr
    info = json.loads(r.stdout)
    assert info["n_tensors"] == 11 and len(info["partitions"]) == 1


def test_state_dict_front_end(tmp_path):
    """sllm.convert of an in-memory state dict (torch CPU tensors incl. bf16 and a
    non-contiguous view, NumPy arrays) split over two partitions by a parallelism plan:
    read back by the oracle's index reader, layout re-derived by the oracle, every byte of
    every tensor equal to the source, padding zero, block checksums = oracle Fletcher-64."""
    torch = pytest.importorskip("torch")
    g = torch.Generator().manual_seed(3)
    base = torch.randn(64, 48, generator=g)
    sd = {
        "embed.weight@0": torch.randn(300, 64, generator=g).to(torch.float16),
        "q.weight@0": torch.randn(64, 64, generator=g).to(torch.bfloat16),
        "o.weight@1": base.t(),                                  # non-contiguous view (48 x 64 f32)
        "norm.bias@1": np.random.default_rng(1).standard_normal(33).astype(np.float16),
        "ids@1": torch.arange(17, dtype=torch.int64),
        "scale@0": torch.tensor(0.5, dtype=torch.float16),       # scalar
    }
    dev = lambda n: int(n.rsplit("@", 1)[1])  # noqa: E731
    from paper_2401_14351_b200 import formats
    assert formats.convert_state_dict(sd, str(tmp_path), dev, 4096, 1 << 16, "sd") == len(sd)
    lay = oindex.read(open(tmp_path / "index.bin", "rb").read())
    ref = olayout.plan([(e.name, e.device, e.dtype, e.shape, e.size) for e in lay.entries], 4096, 1 << 16)
    assert [(e.name, e.device, e.offset) for e in ref.entries] == [(e.name, e.device, e.offset) for e in lay.entries]
    assert [e.name for e in lay.entries] == list(sd)          # source order kept
    for d in lay.devices():
        part = np.fromfile(tmp_path / f"part_{d}.bin", dtype=np.uint8)
        covered = np.zeros(part.size, bool)
        for e in lay.entries:
            if e.device != d:
                continue
            t = sd[e.name]
            if hasattr(t, "detach"):
                t = t.contiguous()
                want = (t.view(torch.int16) if t.dtype == torch.bfloat16 else t).numpy()
            else:
                want = t
            want = np.ascontiguousarray(want).reshape(-1).view(np.uint8)
            assert np.array_equal(part[e.offset:e.offset + e.size], want), e.name
            covered[e.offset:e.offset + e.size] = True
        assert not part[~covered].any()
        assert lay.checksums[d] == fletcher.block_checksums(part, 1 << 16)
    with pytest.raises(_abi.SllmError) as ex:                  # unsupported dtype
        formats.convert_state_dict({"x": np.zeros(3, np.complex64)}, str(tmp_path / "bad"))
    assert ex.value.status == _abi.E_CONVERSION


def test_view_plan_matches_base_plus_offset():
    """The grouped-split views of a contiguous load are exactly base[off:off+size] as
    dtype/shape (P:549 base + offset), for random inventories with all twelve dtypes,
    scalars and padding -- checked on a CPU tensor standing in for the device base."""
    import numpy as np
    import torch
    import paper_2401_14351_b200 as sllm
    from paper_2401_14351_b200 import api
    from synth import models
    for seed in range(6):
        rng = np.random.default_rng(500 + seed)
        inv = models.random_inventory(rng, 150, 3, 1 << 20)
        idx = sllm.Index.plan([(t.name, t.device, t.dtype, t.shape) for t in inv], int(rng.choice([16, 4096])), 0)
        bases = {p: torch.from_numpy(rng.integers(0, 256, q.length, dtype=np.uint8))
                 for p, q in enumerate(idx.partitions)}
        views = api._views(idx, bases.keys(), bases, None, False)
        assert len(views) == len(inv)
        for t in idx.tensors:
            v = views[t.name]
            assert tuple(v.shape) == t.shape and v.dtype == api._torch_dtypes()[t.dtype]
            assert v.data_ptr() == bases[t.partition].data_ptr() + t.offset
            raw = v.reshape(-1).view(torch.uint8) if v.dim() else v.reshape(1).view(torch.uint8)
            assert torch.equal(raw, bases[t.partition][t.offset:t.offset + t.nbytes])


def test_derived_tables_shared_by_content():
    """Index objects parsed from the same bytes share their Python tensor table (a1 still
    parses and validates every time); different content gets its own."""
    import paper_2401_14351_b200 as sllm
    from synth import models
    inv = models.toy()
    blob = sllm.Index.plan([(t.name, t.device, t.dtype, t.shape) for t in inv], 4096, 0).serialize()
    a, b = sllm.Index.from_bytes(blob), sllm.Index.from_bytes(blob)
    assert a.tensors is b.tensors and a.handle.value != b.handle.value
    other = sllm.Index.from_bytes(sllm.Index.plan([(t.name, t.device, t.dtype, t.shape) for t in inv[:-1]],
                                                  4096, 0).serialize())
    assert other.tensors is not a.tensors and len(other.tensors) == len(inv) - 1
