"""The plain CPU loader -- SURVEY.md §8(c) O9 and c4 ("what counts as the oracle loader").

PAPER.md P:549: the model manager "allocates memory on GPUs and loads the binary data
of the checkpoint"; the inference process computes each tensor's address as
*base + offset* from the index; a synchronization returns once everything is loaded
(P:727).  The oracle does the same on the host, as slowly and plainly as possible:

  1. parse the index with its own reader (oracle.index.read);
  2. "allocate" one fresh host buffer per partition (the SPEC's device stub);
  3. copy the partition's bytes into it (P:680's chunks are a transfer detail: the
     result is the same bytes, O6 "never changes the result");
  4. recompute every block's Fletcher-64 (O8) and compare with the index (O9(d));
  5. materialise every tensor as the view base[off : off+size] (O9(a)); for scatter
     mode (O9(b)) copy each tensor's bytes into its own fresh buffer.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Iterable, Optional

import numpy as np

from . import fletcher, index
from .errors import ChecksumError


@dataclass
class OracleLoad:
    layout: index.Layout
    partitions: Dict[int, np.ndarray]      # device -> loaded bytes (contiguous mode)
    tensors: Dict[str, np.ndarray]         # name -> uint8 bytes (views or scatter copies)
    payload_bytes: int
    transferred_bytes: int


def _u8(buf) -> np.ndarray:
    if isinstance(buf, np.ndarray):
        return buf.reshape(-1).view(np.uint8)
    return np.frombuffer(memoryview(buf).cast("B"), dtype=np.uint8)


def verify_partition(layout: index.Layout, p: int, device: int, data: np.ndarray,
                     blocks: Optional[Iterable[int]] = None) -> None:
    """O9(d): recompute cs[d][j] and compare; raise ChecksumError(partition p, block j)
    for the first mismatch in block order."""
    B = layout.block
    if B == 0:
        return
    table = layout.checksums[device]
    js = range(len(table)) if blocks is None else blocks
    for j in js:
        if fletcher.f64_closed(data[j * B:(j + 1) * B]) != table[j]:
            raise ChecksumError(p, j)


def load(index_blob: bytes, sources: Dict[int, object], scatter: bool = False,
         verify: bool = True) -> OracleLoad:
    """Load every partition from ``sources[device]`` (host buffers holding the partition
    bytes) and return the materialised tensors.  Raises ChecksumError(p, j)."""
    layout = index.read(index_blob)
    parts: Dict[int, np.ndarray] = {}
    for p, d in enumerate(layout.devices()):
        src = _u8(sources[d])[:layout.partitions[d]]
        dst = np.empty(layout.partitions[d], dtype=np.uint8)
        dst[:] = src
        if verify:
            verify_partition(layout, p, d, dst)
        parts[d] = dst
    tensors = {}
    for e in layout.entries:
        view = parts[e.device][e.offset:e.offset + e.size]
        tensors[e.name] = view.copy() if scatter else view
    return OracleLoad(layout, parts, tensors, layout.payload_bytes, sum(layout.partitions.values()))


def load_sample(index_blob: bytes, sources: Dict[int, object], byte_budget: int) -> int:
    """Bounded sample of ``load`` for bench.py's cpu_baseline: parse the index, then copy
    and verify whole blocks in partition order until ``byte_budget`` bytes are done, and
    copy every tensor fully contained in them (scatter materialisation).  Returns the
    payload bytes materialised."""
    layout = index.read(index_blob)
    done = 0
    payload = 0
    B = layout.block or (1 << 20)
    for p, d in enumerate(layout.devices()):
        L = layout.partitions[d]
        hi = min(L, (max(byte_budget - done, 0) + B - 1) // B * B)
        if hi <= 0:
            break
        if d not in sources:  # a partition this process does not hold (sharded runs)
            continue
        src = _u8(sources[d])
        dst = np.empty(hi, dtype=np.uint8)
        dst[:] = src[:hi]
        if layout.block:
            verify_partition(layout, p, d, dst, range((hi + B - 1) // B))
        for e in layout.entries:
            if e.device == d and e.offset + e.size <= hi:
                _ = dst[e.offset:e.offset + e.size].copy()
                payload += e.size
        done += hi
    return payload
