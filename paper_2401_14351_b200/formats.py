"""Converter front-end for checkpoints in the wild: Hugging Face ``.safetensors`` files
(ServerlessLLM converts an uploaded checkpoint into its loading-optimized
format; SPEC S:43 convert(src, align)).

A safetensors file is ``u64 header length | JSON header | raw tensor bytes``; the header maps
every tensor name to ``{dtype, shape, data_offsets: [begin, end)}`` relative to the end of
the header.  The files are memory-mapped and every tensor is handed to ``sllm_convert`` as a
(name, device, dtype, shape, host pointer, nbytes) record -- no tensor is copied on the
Python side; the native converter packs them into aligned partitions and writes the index.
"""
from __future__ import annotations

import json
import mmap
import struct
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _abi
from .api import convert

# safetensors dtype tags -> the index's dtype names (include/sllm.h sllm_dtype)
ST_DTYPES = {"F16": "f16", "BF16": "bf16", "F32": "f32", "I8": "i8", "U8": "u8", "I64": "i64",
             "I32": "i32", "F64": "f64", "I16": "i16", "BOOL": "bool", "F8_E4M3": "f8e4m3", "F8_E5M2": "f8e5m2"}


def read_header(path: str) -> Tuple[dict, int]:
    """(header dict in file order, byte offset of the data section)."""
    with open(path, "rb") as f:
        raw = f.read(8)
        if len(raw) != 8:
            raise _abi.SllmError(_abi.E_FORMAT, f"{path}: not a safetensors file")
        (n,) = struct.unpack("<Q", raw)
        hdr = json.loads(f.read(n))
    return hdr, 8 + n


class SafetensorsSource:
    """Memory-mapped safetensors files as converter input records (keeps the maps alive)."""

    def __init__(self, paths: Sequence[str], device_of: Optional[Callable[[str], int]] = None):
        self._maps = []
        self.records: List[tuple] = []
        for path in paths:
            hdr, base = read_header(path)
            f = open(path, "rb")
            mm = mmap.mmap(f.fileno(), 0, access=mmap.ACCESS_READ)
            f.close()
            arr = np.frombuffer(mm, dtype=np.uint8)
            self._maps.append((mm, arr))
            for name, meta in hdr.items():
                if name == "__metadata__":
                    continue
                dt = ST_DTYPES.get(meta["dtype"])
                if dt is None:
                    raise _abi.SllmError(_abi.E_CONVERSION, f"{path}: tensor '{name}' has unsupported dtype "
                                                            f"{meta['dtype']}")
                b, e = (int(x) for x in meta["data_offsets"])
                if base + e > arr.size or b > e:
                    raise _abi.SllmError(_abi.E_FORMAT, f"{path}: tensor '{name}' lies outside the file")
                shape = tuple(int(s) for s in meta["shape"])
                ptr = arr[base + b:base + e].ctypes.data if e > b else 0
                dev = device_of(name) if device_of else 0
                self.records.append((name, dev, dt, shape, ptr, e - b))

    def close(self):
        self.records = []
        for mm, arr in self._maps:
            del arr
        self._maps = []


def convert_safetensors(paths: Sequence[str], out_dir: str, device_of: Optional[Callable[[str], int]] = None,
                        align: int = 4096, block: int = 1 << 20, model_id: str = "") -> int:
    """Convert safetensors files (tensors in file, then header order = the source order of
    the layout, Q2) into ``out_dir``/part_<d>.bin + index.bin.  ``device_of(name)`` gives
    each tensor's partition (default: everything on partition 0).  Returns the tensor
    count.  Errors as sllm_convert: duplicate names across files, payload != shape x width
    and zero-sized dimensions raise SLLM_E_CONVERSION."""
    src = SafetensorsSource(paths, device_of)
    try:
        convert(src.records, out_dir, align, block, model_id)
        return len(src.records)
    finally:
        src.close()


# torch / NumPy dtypes -> the index's dtype names (include/sllm.h sllm_dtype)
_NP_DTYPES = {np.dtype(np.float16): "f16", np.dtype(np.float32): "f32", np.dtype(np.int8): "i8",
              np.dtype(np.uint8): "u8", np.dtype(np.int64): "i64", np.dtype(np.int32): "i32",
              np.dtype(np.float64): "f64", np.dtype(np.int16): "i16", np.dtype(np.bool_): "bool"}


def convert_state_dict(state_dict, out_dir: str, device_of: Optional[Callable[[str], int]] = None,
                       align: int = 4096, block: int = 1 << 20, model_id: str = "") -> int:
    """Convert an in-memory state dict (name -> CPU torch tensor or NumPy array, in the
    dict's order = the layout's source order, Q2) into ``out_dir``/part_<d>.bin +
    index.bin -- SURVEY §8(b)'s ``sllm.convert(state_dict_like, ...)``.  ``device_of(name)``
    is the parallelism plan (which GPU each tensor goes to; default 0).  Tensors are
    passed to sllm_convert by host pointer (made contiguous first when they are not); bf16
    is supported for torch tensors.  Returns the tensor count; errors as sllm_convert."""
    keep, records = [], []
    for name, t in state_dict.items():
        if hasattr(t, "detach"):  # torch.Tensor
            import torch
            if t.device.type != "cpu":
                raise _abi.SllmError(_abi.E_INVALID, f"tensor '{name}' is on {t.device}; convert from host memory")
            t = t.detach().contiguous()
            raw = {torch.bfloat16: ("bf16", torch.int16), torch.float8_e4m3fn: ("f8e4m3", torch.uint8),
                   torch.float8_e5m2: ("f8e5m2", torch.uint8)}
            if t.dtype in raw:  # no NumPy twin: hand over the bytes under a same-width integer view
                dt = raw[t.dtype][0]
                arr = t.view(raw[t.dtype][1]).numpy()
            else:
                arr = t.numpy()
                dt = _NP_DTYPES.get(arr.dtype)
        else:
            arr = np.ascontiguousarray(np.asarray(t))
            dt = _NP_DTYPES.get(arr.dtype)
        if dt is None:
            raise _abi.SllmError(_abi.E_CONVERSION, f"tensor '{name}' has unsupported dtype {arr.dtype}")
        arr = np.ascontiguousarray(arr)
        keep.append(arr)
        records.append((name, device_of(name) if device_of else 0, dt, tuple(int(s) for s in arr.shape),
                        arr.ctypes.data if arr.size else 0, arr.nbytes))
    convert(records, out_dir, align, block, model_id)
    return len(records)
