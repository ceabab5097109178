"""B200-native loading-optimized checkpoint loader (ServerlessLLM, arXiv 2401.14351).

The product is the C-ABI library ``libsllm.so`` (include/sllm.h): converter, index
codec, pinned DRAM tier, the chunked host->HBM pipeline (copy engine or sm_100a
zero-copy kernels), the index-driven scatter kernel, the fused Fletcher-64 block
verification, the replicated fan-out (fused NVLink peer stores or NCCL), the file tier,
the pinned whole-model LRU cache and cross-process handles.  This package is the thin
ctypes binding over it; see ``api`` for the Python surface.
"""
from ._abi import SllmError, lib, LIB_PATH  # noqa: F401
from .api import (Index, HostBuffer, LoadConfig, LoadResult, CapturedLoad, Comm, PinnedCache, TensorInfo, PartitionInfo,  # noqa: F401
                  allocate, block_checksums_device, chunk_count, convert, fletcher64, load, load_capture, load_files, load_start,
                  materialise_device, replica_slices, replica_schedule, allgather_schedule, trim_device_cache,
                  fanout_unit)

open_index = Index.open  # SURVEY §8(b) Python surface: sllm.open_index(path)

__all__ = ["open_index", "SllmError", "lib", "Index", "HostBuffer", "LoadConfig", "LoadResult", "CapturedLoad", "load_capture", "Comm", "PinnedCache", "allocate", "load",
           "load_start", "convert", "fletcher64", "chunk_count", "replica_slices", "block_checksums_device",
           "materialise_device", "load_files", "replica_schedule", "allgather_schedule", "trim_device_cache", "fanout_unit"]
