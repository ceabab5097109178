"""ctypes declarations of include/sllm.h (argument marshalling only).

The library is REQUIRED: importing the binding without libsllm.so raises (there is no
CPU fallback).  Build it with ``python -m paper_2401_14351_b200.build``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SLLM_LIB_PATH: an A/B measurement build of the same sources (tools/build_variant.py);
# the product path is the in-tree libsllm.so
LIB_PATH = os.environ.get("SLLM_LIB_PATH") or os.path.join(HERE, "libsllm.so")

MAX_NDIM = 8

STATUS = {0: "OK", 1: "INVALID", 2: "CONVERSION", 3: "FORMAT", 4: "LOOKUP", 5: "CAPACITY", 6: "IO",
          7: "CUDA", 8: "NCCL", 9: "CHECKSUM", 10: "BUSY", 11: "NOMEM", 12: "PEER"}
(OK, E_INVALID, E_CONVERSION, E_FORMAT, E_LOOKUP, E_CAPACITY, E_IO, E_CUDA, E_NCCL, E_CHECKSUM, E_BUSY, E_NOMEM,
 E_PEER) = range(13)

MODE_CE, MODE_ZEROCOPY, MODE_SCATTER_CE, MODE_SCATTER_ZC, MODE_AUTO, MODE_GDS = range(6)
FANOUT_NONE, FANOUT_BCAST, FANOUT_P2P, FANOUT_ALLGATHER, FANOUT_NVLS = range(5)
DTYPE_CODE = {"f16": 0, "bf16": 1, "f32": 2, "i8": 3, "u8": 4, "i64": 5,
              "i32": 6, "f64": 7, "i16": 8, "bool": 9, "f8e4m3": 10, "f8e5m2": 11}
DTYPE_NAME = {v: k for k, v in DTYPE_CODE.items()}


class SrcTensor(C.Structure):
    _fields_ = [("name", C.c_char_p), ("device_id", C.c_int32), ("dtype", C.c_int32), ("ndim", C.c_int32),
                ("shape", C.POINTER(C.c_int64)), ("data", C.c_void_p), ("nbytes", C.c_uint64)]


class IndexInfo(C.Structure):
    _fields_ = [("align", C.c_uint64), ("block", C.c_uint64), ("payload_bytes", C.c_uint64),
                ("n_partitions", C.c_uint64), ("n_tensors", C.c_uint64), ("model_id", C.c_char_p)]


class TensorInfo(C.Structure):
    _fields_ = [("name", C.c_char_p), ("device_id", C.c_int32), ("partition", C.c_int32), ("dtype", C.c_int32),
                ("ndim", C.c_int32), ("shape", C.c_int64 * MAX_NDIM), ("offset", C.c_uint64), ("nbytes", C.c_uint64)]


class LoadConfig(C.Structure):
    _fields_ = [("chunk_bytes", C.c_uint64), ("n_streams", C.c_int32), ("mode", C.c_int32), ("fanout", C.c_int32),
                ("verify", C.c_int32), ("ctas", C.c_int32), ("profile", C.c_int32),
                ("engine", C.c_int32), ("reserved", C.c_int32)]


class LoadReport(C.Structure):
    _fields_ = [("payload_bytes", C.c_uint64), ("transferred_bytes", C.c_uint64), ("fanout_bytes", C.c_uint64),
                ("chunks", C.c_uint64), ("kernel_launches", C.c_uint64), ("copy_calls", C.c_uint64),
                ("t_total_ns", C.c_uint64), ("t_issue_ns_max", C.c_uint64), ("t_device_ms_max", C.c_double),
                ("t_kernel_ms_sum", C.c_double), ("t_copy_ms_sum", C.c_double), ("kernel_bytes", C.c_uint64),
                ("bad_partition", C.c_int32), ("mode", C.c_int32), ("bad_block", C.c_uint64),
                ("storage_bytes", C.c_uint64), ("t_storage_wait_ns_max", C.c_uint64),
                ("t_kernel_span_ms_sum", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class TensorHandle(C.Structure):
    _fields_ = [("gpu", C.c_int32), ("dtype", C.c_int32), ("ndim", C.c_int32), ("reserved", C.c_int32),
                ("shape", C.c_int64 * MAX_NDIM), ("ptr", C.c_void_p), ("nbytes", C.c_uint64)]


class IpcRegion(C.Structure):
    _fields_ = [("handle", C.c_uint8 * 64), ("offset", C.c_uint64), ("nbytes", C.c_uint64), ("gpu", C.c_int32),
                ("reserved", C.c_int32)]


class CacheStats(C.Structure):
    _fields_ = [("capacity", C.c_uint64), ("used", C.c_uint64), ("models", C.c_uint64), ("hits", C.c_uint64),
                ("misses", C.c_uint64), ("evictions", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


P = C.c_void_p
PP = C.POINTER(C.c_void_p)
U64 = C.c_uint64
S = C.c_int  # sllm_status
# name -> (restype, argtypes): every entry point of include/sllm.h
SIGNATURES = {
    "sllm_last_error": (C.c_char_p, []),
    "sllm_abi_version": (C.c_int32, []),
    "sllm_plan": (S, [C.POINTER(SrcTensor), C.c_size_t, U64, U64, C.c_char_p, PP]),
    "sllm_convert_into": (S, [C.POINTER(SrcTensor), C.c_size_t, P, PP]),
    "sllm_index_seal": (S, [P, PP]),
    "sllm_convert": (S, [C.POINTER(SrcTensor), C.c_size_t, U64, U64, C.c_char_p, C.c_char_p]),
    "sllm_index_serialize": (S, [P, P, C.c_size_t, C.POINTER(C.c_size_t)]),
    "sllm_index_open": (S, [C.c_char_p, PP]),
    "sllm_index_from_memory": (S, [P, C.c_size_t, PP]),
    "sllm_index_close": (None, [P]),
    "sllm_index_get_info": (S, [P, C.POINTER(IndexInfo)]),
    "sllm_index_counts": (S, [P, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "sllm_index_partition": (S, [P, C.c_size_t, C.POINTER(C.c_int32), C.POINTER(U64), C.POINTER(U64), C.POINTER(U64)]),
    "sllm_index_block_checksums": (S, [P, C.c_size_t, C.POINTER(C.POINTER(U64))]),
    "sllm_index_tensor": (S, [P, C.c_size_t, C.POINTER(TensorInfo)]),
    "sllm_index_find": (S, [P, C.c_char_p, C.POINTER(C.c_size_t)]),
    "sllm_tensor_address": (S, [P, C.c_char_p, C.POINTER(U64), C.POINTER(C.c_int32), C.POINTER(U64)]),
    "sllm_fletcher64_host": (S, [P, U64, C.POINTER(U64)]),
    "sllm_chunk_count": (S, [U64, U64, C.POINTER(U64)]),
    "sllm_replica_slices": (S, [U64, U64, C.c_int32, C.POINTER(U64)]),
    "sllm_replica_round": (S, [U64, U64, C.c_int32, U64, C.POINTER(U64), C.POINTER(U64)]),
    "sllm_device_trim": (S, [C.c_int32, U64]),
    "sllm_allgather_round": (S, [U64, U64, C.c_int32, U64, C.POINTER(U64), C.POINTER(U64), C.POINTER(C.c_int32)]),
    "sllm_fanout_unit": (S, [U64, C.c_int32, C.POINTER(U64)]),
    "sllm_gpu_numa_node": (S, [C.c_int32, C.POINTER(C.c_int32)]),
    "sllm_host_numa_node": (S, [P, C.POINTER(C.c_int32)]),
    "sllm_host_alloc": (S, [U64, C.c_int32, PP]),
    "sllm_host_free": (None, [P]),
    "sllm_host_register": (S, [P, U64]),
    "sllm_host_unregister": (S, [P]),
    "sllm_host_read_partition": (S, [C.c_char_p, P, C.c_size_t, P, C.c_int32]),
    "sllm_comm_unique_id": (S, [P]),
    "sllm_comm_init_rank": (S, [P, C.c_int32, C.c_int32, C.c_int32, PP]),
    "sllm_comm_init_all": (S, [C.POINTER(C.c_int32), C.c_int32, PP]),
    "sllm_comm_init_peers": (S, [C.c_int32, C.c_int32, C.c_int32, PP, PP, U64, PP]),
    "sllm_comm_init_nvls": (S, [C.POINTER(C.c_int32), C.c_int32, U64, U64, PP]),
    "sllm_comm_replica": (S, [P, PP, C.POINTER(U64)]),
    "sllm_comm_free": (None, [P]),
    "sllm_cache_create": (S, [U64, C.c_int32, C.c_int32, PP]),
    "sllm_cache_acquire": (S, [P, C.c_char_p, C.c_int32, PP, C.POINTER(PP), C.POINTER(C.c_int32)]),
    "sllm_cache_release": (S, [P, C.c_char_p]),
    "sllm_cache_get_stats": (S, [P, C.POINTER(CacheStats)]),
    "sllm_cache_destroy": (None, [P]),
    "sllm_load_start": (S, [P, C.POINTER(LoadConfig), PP, C.POINTER(C.c_int32), PP, PP, PP, P, PP]),
    "sllm_load_files_start": (S, [P, C.POINTER(LoadConfig), C.c_char_p, C.POINTER(C.c_int32), PP, PP, PP, C.c_int32,
                                  P, PP]),
    "sllm_load_capture": (S, [P, C.POINTER(LoadConfig), PP, C.POINTER(C.c_int32), PP, PP, PP]),
    "sllm_load_replay": (S, [P, PP]),
    "sllm_load_wait": (S, [P, C.POINTER(LoadReport)]),
    "sllm_load_tensor": (S, [P, C.c_char_p, C.POINTER(TensorHandle)]),
    "sllm_load_block_checksums": (S, [P, C.c_size_t, C.POINTER(C.POINTER(U64))]),
    "sllm_load_free": (None, [P]),
    "sllm_ipc_export": (S, [P, U64, C.POINTER(IpcRegion)]),
    "sllm_ipc_open": (S, [C.POINTER(IpcRegion), PP]),
    "sllm_ipc_close": (S, [P]),
    "sllm_block_checksums_device": (S, [P, U64, U64, P, C.c_int32, P]),
    "sllm_materialise_device": (S, [P, C.c_size_t, P, PP, C.c_int32, P, C.POINTER(U64), C.POINTER(C.c_float)]),
}

_lib = None


def lib():
    """The loaded libsllm.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2401_14351_b200.build` "
                              "(the CUDA library is required; there is no CPU fallback)")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class SllmError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"SLLM_E_{STATUS.get(status, status)}: {message}")
        self.status = status
        self.message = message


def check(status: int) -> None:
    if status != OK:
        raise SllmError(status, lib().sllm_last_error().decode("utf-8", "replace"))
