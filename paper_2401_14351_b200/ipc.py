"""Model manager <-> inference process handles.

The loading process exports, for every partition it loaded, a CUDA IPC handle of the
partition's device base (``export``); the inference process maps the bases, reads the
tensor index and builds every tensor as base + offset (``import_tensors``) without
copying a byte.  ``export`` is called after ``LoadResult.wait()`` (the paper's sync,
P:727) or before it, with the importer synchronising through the exporter.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, Tuple

from . import _abi
from ._abi import check, lib
from .api import Index, LoadResult, _torch_dtypes


def export(res: LoadResult) -> dict:
    """{"index": index bytes, "regions": {partition: 88-byte sllm_ipc_region}} for a
    contiguous-mode load (the partitions' device bases)."""
    bases = res._keep[3]
    if not bases:
        raise ValueError("IPC export needs a contiguous-mode load (one base per partition)")
    regions = {}
    for p, base in bases.items():
        r = _abi.IpcRegion()
        check(lib().sllm_ipc_export(C.c_void_p(base.data_ptr()), base.numel(), C.byref(r)))
        regions[int(p)] = bytes(r)
    return {"index": res.index.serialize(), "regions": regions}


class _CudaBuffer:
    """Minimal __cuda_array_interface__ producer so torch can wrap a mapped region."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


class Imported:
    """Mapped partitions of another process and the tensor views built on them."""

    def __init__(self, exported: dict):
        import torch
        self.index = Index.from_bytes(exported["index"])
        self.ptrs: Dict[int, int] = {}
        self.bases: Dict[int, object] = {}
        for p, blob in exported["regions"].items():
            r = _abi.IpcRegion.from_buffer_copy(blob)
            out = C.c_void_p()
            check(lib().sllm_ipc_open(C.byref(r), C.byref(out)))
            self.ptrs[int(p)] = out.value
            self.bases[int(p)] = torch.as_tensor(_CudaBuffer(out.value, r.nbytes), device=f"cuda:{r.gpu}")
        tdt = _torch_dtypes()
        self.tensors = {}
        for t in self.index.tensors:                      # base + offset per tensor
            if t.partition in self.bases:
                b = self.bases[t.partition]
                self.tensors[t.name] = b[t.offset:t.offset + t.nbytes].view(tdt[t.dtype]).view(t.shape)

    def close(self) -> None:
        self.tensors = {}
        self.bases = {}
        for p in list(self.ptrs):
            check(lib().sllm_ipc_close(C.c_void_p(self.ptrs.pop(p))))


def import_tensors(exported: dict) -> Imported:
    return Imported(exported)


def export_region(ptr: int, nbytes: int) -> bytes:
    """sllm_ipc_export of one device range (e.g. a P2P replica or signal array)."""
    r = _abi.IpcRegion()
    check(lib().sllm_ipc_export(C.c_void_p(ptr), nbytes, C.byref(r)))
    return bytes(r)


def open_region(blob: bytes, gpu: int) -> int:
    """Map an exported range into this process, in the context of CUDA device ``gpu`` (the
    importing GPU: a peer's memory is then reached over NVLink)."""
    r = _abi.IpcRegion.from_buffer_copy(blob)
    r.gpu = gpu
    out = C.c_void_p()
    check(lib().sllm_ipc_open(C.byref(r), C.byref(out)))
    return out.value


def close(ptr: int) -> None:
    check(lib().sllm_ipc_close(C.c_void_p(ptr)))
