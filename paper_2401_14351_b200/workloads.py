"""Synthetic checkpoints packed straight into pinned DRAM with the library's converter.

plan (libsllm) -> fill every tensor's slot with the seeded payload (synth, O10) -> seal
(libsllm computes the block checksums).  Padding stays 0x00 (pinned buffers are zeroed
at allocation).  Used by bench.py, smoke() and the GPU tests to build multi-GB inputs
in seconds without disk; the oracle never sees anything produced here except the index
checksums, which the CPU suite pins to the oracle (tests/test_format_parity.py).
"""
from __future__ import annotations

import os
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

from synth import models, payload

from .api import HostBuffer, Index


def plan_inventory(inv: Sequence[models.TensorSpec], align: int = 4096, block: int = 1 << 20,
                   model_id: str = "") -> Index:
    return Index.plan([(t.name, t.device, t.dtype, t.shape) for t in inv], align, block, model_id)


def build_pinned(inv: Sequence[models.TensorSpec], seed: int, align: int = 4096, block: int = 1 << 20,
                 model_id: str = "", partitions: Optional[Iterable[int]] = None, gpu_of: Optional[Dict[int, int]] = None,
                 threads: int = 0) -> Tuple[Index, Dict[int, HostBuffer]]:
    """Pinned partitions for ``partitions`` (default: all), sealed index.  Tensor e of the
    inventory gets payload (seed, e)."""
    idx = plan_inventory(inv, align, block, model_id)
    parts = idx.partitions
    sel = list(range(len(parts))) if partitions is None else sorted(partitions)
    bufs: Dict[int, HostBuffer] = {}
    for p in sel:
        gpu = -1 if gpu_of is None else gpu_of.get(p, -1)
        bufs[p] = HostBuffer(parts[p].length, gpu)
    ptrs, sizes, es = [], [], []
    for e, t in enumerate(idx.tensors):
        if t.partition in bufs:
            ptrs.append(bufs[t.partition].ptr + t.offset)
            sizes.append(t.nbytes)
            es.append(e)
    if not threads:  # ranks of one node share its cores (8 ranks each building 17 GB at once)
        threads = max(1, len(os.sched_getaffinity(0)) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1"))))
    payload.payload_into(ptrs, sizes, seed, es, threads)
    idx.seal([bufs[p].ptr if p in bufs else None for p in range(len(parts))])
    return idx, bufs


def build_config(config: str, partitions: Optional[Iterable[int]] = None, gpu_of: Optional[Dict[int, int]] = None,
                 align: int = 4096, block: int = 1 << 20) -> Tuple[Index, Dict[int, HostBuffer], List[models.TensorSpec], int]:
    inv, seed = models.model_inventory(config)
    idx, bufs = build_pinned(inv, seed, align, block, config, partitions, gpu_of)
    return idx, bufs, inv, seed
