"""Counter-based synthetic payload.

    splitmix64(z): z += 0x9E3779B97F4A7C15; z = (z ^ z>>30) * 0xBF58476D1CE4E5B9;
                   z = (z ^ z>>27) * 0x94D049BB133111EB; return z ^ z>>31
    key_e     = splitmix64(seed ^ splitmix64(e))          (e = global source-order index)
    word_k(e) = splitmix64(key_e + k * 0x9E3779B97F4A7C15)
    payload_e = little-endian concatenation of word_0, word_1, ... truncated to size_e

Uniform random bits, so every fp16 NaN/Inf/-0/subnormal pattern occurs (Q13: equality
is byte equality).  NumPy uint64 arithmetic wraps mod 2**64, so the vectorised form
below is exact.  ``payload_into`` uses the multi-threaded C twin in ``csynth.c`` when
it is built (pinned against this file by tests/test_synth.py).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(z):
    """Vectorised splitmix64 over a uint64 scalar or array (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = np.asarray(z, dtype=np.uint64) + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def tensor_key(seed: int, e: int) -> np.uint64:
    return splitmix64(np.uint64(seed) ^ splitmix64(np.uint64(e)))


def payload_bytes(seed: int, e: int, nbytes: int) -> np.ndarray:
    """Payload of tensor ``e`` as a fresh uint8 array (NumPy definition)."""
    nw = (nbytes + 7) // 8
    key = tensor_key(seed, e)
    with np.errstate(over="ignore"):
        k = np.arange(nw, dtype=np.uint64)
        words = splitmix64(key + k * GOLDEN)
    return words.astype("<u8").view(np.uint8)[:nbytes].copy()


_lib = None


def _csynth():
    global _lib
    if _lib is None:
        path = os.path.join(os.path.dirname(__file__), "libsynth.so")
        if not os.path.exists(path):
            return None
        lib = ctypes.CDLL(path)
        lib.synth_fill_many.argtypes = [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p),
                                        ctypes.POINTER(ctypes.c_uint64), ctypes.c_uint64,
                                        ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
        lib.synth_fill_many.restype = ctypes.c_int
        _lib = lib
    return _lib


def build_csynth(force: bool = False) -> str:
    """Compile csynth.c -> libsynth.so (plain gcc, pthreads)."""
    here = os.path.dirname(os.path.abspath(__file__))
    out = os.path.join(here, "libsynth.so")
    src = os.path.join(here, "csynth.c")
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        import subprocess
        tmp = f"{out}.tmp{os.getpid()}"  # several ranks may build at once: publish atomically
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v3", "-shared", "-fPIC", "-pthread",
                               "-o", tmp, src])
        os.replace(tmp, out)
    return out


def payload_into(ptrs, sizes, seed: int, es, threads: int = 0) -> None:
    """Fill raw host buffers ``ptrs[i]`` (ints) with ``sizes[i]`` payload bytes of
    tensor ``es[i]``.  Multi-threaded C when available, else NumPy."""
    n = len(ptrs)
    if n == 0:
        return
    lib = _csynth()
    if lib is not None:
        P = (ctypes.c_void_p * n)(*ptrs)
        S = (ctypes.c_uint64 * n)(*sizes)
        E = (ctypes.c_uint64 * n)(*es)
        rc = lib.synth_fill_many(n, P, S, seed, E, threads or (os.cpu_count() or 1))
        if rc != 0:
            raise RuntimeError(f"synth_fill_many failed rc={rc}")
        return
    for p, s, e in zip(ptrs, sizes, es):
        data = payload_bytes(seed, e, s)
        ctypes.memmove(p, data.ctypes.data, s)
