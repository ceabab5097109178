"""The C-ABI library loads and exports every symbol include/sllm.h declares; host-only
entry points behave per the header (no GPU needed)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2401_14351_b200 as sllm
from paper_2401_14351_b200 import _abi

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "sllm.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"SLLM_API\s+[\w\s\*]+?\b(sllm_\w+)\s*\(", src)))


def test_every_declared_symbol_exported():
    lib = sllm.lib()
    names = declared_symbols()
    assert len(names) >= 35
    for n in names:
        assert hasattr(lib, n), n
        assert n in _abi.SIGNATURES, f"{n} not bound in _abi.SIGNATURES"
    assert set(_abi.SIGNATURES) == set(names)


def test_only_c_abi_exported():
    out = os.popen(f"nm -D --defined-only {_abi.LIB_PATH}").read()
    syms = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert syms and all(s.startswith("sllm_") for s in syms), sorted(s for s in syms if not s.startswith("sllm_"))[:10]


def test_abi_version_and_errors():
    lib = sllm.lib()
    assert lib.sllm_abi_version() == 1
    out = ctypes.c_void_p()
    st = lib.sllm_index_open(b"/nonexistent/index.bin", ctypes.byref(out))
    assert st == _abi.E_IO
    assert b"nonexistent" in lib.sllm_last_error()
    st = lib.sllm_index_from_memory(b"\x00" * 100, 100, ctypes.byref(out))
    assert st == _abi.E_FORMAT


def test_chunk_count_and_slices():
    assert sllm.chunk_count(0, 16) == 0
    assert sllm.chunk_count(17, 16) == 2
    assert sllm.chunk_count(13_316_947_968, 16 << 20) == 794
    for L, C, N in [(100 * 4096, 4096, 3), (13_594_624, 1 << 20, 8), (4096, 4096, 4), (0, 16, 2),
                    (59_949_920_256, 16 << 20, 8)]:
        sl = sllm.replica_slices(L, C, N)
        assert sl[0][0] == 0 and sl[-1][1] == L
        for (a, b), (c, d) in zip(sl, sl[1:]):
            assert b == c
        for a, b in sl:
            assert a <= b and a % C == 0
        sizes = [b - a for a, b in sl]
        assert max(sizes) - min(sizes) <= C


def test_host_alloc_fails_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(sllm.SllmError) as ex:
        sllm.HostBuffer(1 << 20)
    assert ex.value.status in (_abi.E_CUDA, _abi.E_NOMEM)


def test_load_rejects_bad_arguments():
    idx = sllm.Index.plan([("a", 0, "u8", (10,))], 4096, 4096)
    buf = np.zeros(4096, np.uint8)
    idx.seal([buf.ctypes.data])
    lib = sllm.lib()
    out = ctypes.c_void_p()
    cfg = _abi.LoadConfig(3 << 20 | 5, 2, 0, 0, 1, 0, 0, 0, 0)   # chunk not a multiple of the block
    gpu = (ctypes.c_int32 * 1)(0)
    src = (ctypes.c_void_p * 1)(buf.ctypes.data)
    dst = (ctypes.c_void_p * 1)(0x1000)
    st = lib.sllm_load_start(idx.handle, ctypes.byref(cfg), src, gpu, dst, None, None, None, ctypes.byref(out))
    assert st == _abi.E_INVALID
    cfg = _abi.LoadConfig(1 << 20, 9, 0, 0, 1, 0, 0, 0, 0)        # too many streams
    st = lib.sllm_load_start(idx.handle, ctypes.byref(cfg), src, gpu, dst, None, None, None, ctypes.byref(out))
    assert st == _abi.E_INVALID
    cfg = _abi.LoadConfig(1 << 20, 2, 7, 0, 1, 0, 0, 0, 0)        # unknown mode
    st = lib.sllm_load_start(idx.handle, ctypes.byref(cfg), src, gpu, dst, None, None, None, ctypes.byref(out))
    assert st == _abi.E_INVALID
    unsealed = sllm.Index.plan([("a", 0, "u8", (10,))], 4096, 4096)
    cfg = _abi.LoadConfig(1 << 20, 2, 0, 0, 1, 0, 0, 0, 0)
    st = lib.sllm_load_start(unsealed.handle, ctypes.byref(cfg), src, gpu, dst, None, None, None, ctypes.byref(out))
    assert st == _abi.E_INVALID
