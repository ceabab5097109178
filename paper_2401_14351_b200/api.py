"""Python surface of the loader (SURVEY §8(b) "Python surface").  Argument marshalling
only: every byte the load path moves is moved by libsllm.so (copy engine or its sm_100a
kernels).  PyTorch provides device memory, streams and the process group.

    idx = Index.open("ckpt/index.bin")                       # S:52 read_index
    src = {p: HostBuffer.read_partition("ckpt", idx, p) ...}  # file -> pinned DRAM tier
    res = load(idx, src, gpus={0: 0}, config=LoadConfig())   # P:549 load + P:727 sync
    res.tensors["model.layers.0.mlp.up_proj.weight"]          # torch view, base + offset
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

import numpy as np

from . import _abi
from ._abi import check, lib

_TORCH_DTYPE = None


def _torch_dtypes():
    global _TORCH_DTYPE
    if _TORCH_DTYPE is None:
        import torch
        _TORCH_DTYPE = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32, "i8": torch.int8,
                        "u8": torch.uint8, "i64": torch.int64, "i32": torch.int32, "f64": torch.float64,
                        "i16": torch.int16, "bool": torch.bool, "f8e4m3": torch.float8_e4m3fn,
                        "f8e5m2": torch.float8_e5m2}
    return _TORCH_DTYPE


WIDTH = {"f16": 2, "bf16": 2, "f32": 4, "i8": 1, "u8": 1, "i64": 8,
         "i32": 4, "f64": 8, "i16": 2, "bool": 1, "f8e4m3": 1, "f8e5m2": 1}


@dataclass(frozen=True)
class TensorInfo:
    name: str
    device: int
    partition: int
    dtype: str
    shape: Tuple[int, ...]
    offset: int
    nbytes: int


@dataclass(frozen=True)
class PartitionInfo:
    device: int
    length: int
    n_blocks: int
    n_tensors: int


def _src_array(tensors: Sequence) -> Tuple[C.Array, list]:
    """tensors: (name, device, dtype, shape[, data_ptr, nbytes]) -> SrcTensor[] (+ keepalive)."""
    arr = (_abi.SrcTensor * max(len(tensors), 1))()
    keep = []
    for i, t in enumerate(tensors):
        name, dev, dt, shape = t[0], t[1], t[2], tuple(int(s) for s in t[3])
        nm = name.encode("utf-8")
        shp = (C.c_int64 * max(len(shape), 1))(*shape)
        keep += [nm, shp]
        nbytes = math.prod(shape) * WIDTH[dt] if len(t) < 6 else int(t[5])
        arr[i] = _abi.SrcTensor(nm, int(dev), _abi.DTYPE_CODE[dt], len(shape), shp,
                                C.c_void_p(int(t[4])) if len(t) > 4 and t[4] else None, nbytes)
    return arr, keep


def _ptr_array(ptrs: Iterable[Optional[int]]) -> C.Array:
    ptrs = list(ptrs)
    return (C.c_void_p * max(len(ptrs), 1))(*[C.c_void_p(int(p)) if p else None for p in ptrs])


# Python-side tables derived from an index's content (TensorInfo list, per-partition view
# plans), shared by every Index parsed from the same bytes: the C parse and validation (a1)
# still run for every Index, but the per-tensor Python objects are built once per content
# instead of once per load (a latency-bound load of a 1,120-tensor LoRA adapter otherwise
# spends ~1 ms per step creating and tearing them down).  Keyed by the index bytes
# themselves (a checksum key could map two different indexes to one table: Fletcher-64 does
# not tell a 0x00000000 word from 0xFFFFFFFF); the hash of a bytes object is cached on it,
# so a caller re-opening the same blob pays one hash; bounded LRU.
_DERIVED: "Dict[bytes, dict]" = {}
_DERIVED_MAX = 16


def _derived_for(key: Optional[bytes]) -> dict:
    if key is None:
        return {}
    d = _DERIVED.pop(key, None)
    if d is None:
        d = {}
        if len(_DERIVED) >= _DERIVED_MAX:
            _DERIVED.pop(next(iter(_DERIVED)))
    _DERIVED[key] = d  # most recently used last
    return d


class Index:
    """Owned handle to a parsed or planned index (sllm_index*)."""

    def __init__(self, handle: int, owned: bool = True, key: Optional[bytes] = None):
        self._h = C.c_void_p(handle)
        self._owned = owned  # False: borrowed from another owner (e.g. a PinnedCache entry)
        self._derived = _derived_for(key)
        self._tensors: Optional[List[TensorInfo]] = self._derived.get("tensors")
        self._by_name: Optional[Dict[str, int]] = self._derived.get("by_name")

    # -- constructors ------------------------------------------------------------------
    @classmethod
    def plan(cls, tensors: Sequence, align: int = 4096, block: int = 1 << 20, model_id: str = "") -> "Index":
        """Layout only.  tensors: (name, device, dtype, shape)."""
        arr, keep = _src_array(tensors)
        out = C.c_void_p()
        check(lib().sllm_plan(arr, len(tensors), align, block, model_id.encode(), C.byref(out)))
        return cls(out.value)

    @classmethod
    def open(cls, path: str) -> "Index":
        out = C.c_void_p()
        check(lib().sllm_index_open(path.encode(), C.byref(out)))
        return cls(out.value)

    @classmethod
    def from_bytes(cls, blob: bytes) -> "Index":
        blob = bytes(blob)
        out = C.c_void_p()
        check(lib().sllm_index_from_memory(blob, len(blob), C.byref(out)))
        return cls(out.value, key=blob)

    def close(self) -> None:
        if self._h and self._h.value:
            if self._owned:
                lib().sllm_index_close(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    # -- filling -----------------------------------------------------------------------
    def seal(self, part_ptrs: Sequence[int]) -> None:
        check(lib().sllm_index_seal(self._h, _ptr_array(part_ptrs)))

    def convert_into(self, tensors: Sequence, part_ptrs: Sequence[int]) -> None:
        """tensors: (name, device, dtype, shape, data_ptr) in plan order."""
        arr, keep = _src_array(tensors)
        check(lib().sllm_convert_into(arr, len(tensors), self._h, _ptr_array(part_ptrs)))

    def serialize(self) -> bytes:
        n = C.c_size_t()
        check(lib().sllm_index_serialize(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(lib().sllm_index_serialize(self._h, buf, n.value, C.byref(n)))
        return buf.raw[:n.value]

    # -- queries -----------------------------------------------------------------------
    def counts(self) -> Tuple[int, int]:
        """(n_tensors, n_partitions) -- sllm_index_counts."""
        nt, npart = C.c_size_t(), C.c_size_t()
        check(lib().sllm_index_counts(self.handle, C.byref(nt), C.byref(npart)))
        return nt.value, npart.value

    def info(self) -> dict:
        i = _abi.IndexInfo()
        check(lib().sllm_index_get_info(self._h, C.byref(i)))
        return {"align": i.align, "block": i.block, "payload_bytes": i.payload_bytes,
                "n_partitions": i.n_partitions, "n_tensors": i.n_tensors, "model_id": i.model_id.decode()}

    @property
    def partitions(self) -> List[PartitionInfo]:
        out = []
        for p in range(self.info()["n_partitions"]):
            d, L, nb, nt = C.c_int32(), C.c_uint64(), C.c_uint64(), C.c_uint64()
            check(lib().sllm_index_partition(self._h, p, C.byref(d), C.byref(L), C.byref(nb), C.byref(nt)))
            out.append(PartitionInfo(d.value, L.value, nb.value, nt.value))
        return out

    @property
    def tensors(self) -> List[TensorInfo]:
        if self._tensors is None and "tensors" in self._derived:  # built by another Index of this content
            self._tensors, self._by_name = self._derived["tensors"], self._derived["by_name"]
        if self._tensors is None:
            out = []
            for i in range(self.info()["n_tensors"]):
                t = _abi.TensorInfo()
                check(lib().sllm_index_tensor(self._h, i, C.byref(t)))
                out.append(TensorInfo(t.name.decode("utf-8"), t.device_id, t.partition, _abi.DTYPE_NAME[t.dtype],
                                      tuple(t.shape[:t.ndim]), t.offset, t.nbytes))
            self._tensors = out
            self._by_name = {t.name: i for i, t in enumerate(out)}
            self._derived["tensors"], self._derived["by_name"] = self._tensors, self._by_name
        return self._tensors

    def view_plan(self, p: int):
        """Per dtype of partition p: (dtype, split sizes in elements over the whole partition,
        [(name, piece index, shape)]) -- tensors as pieces of one typed split of the base,
        padding as the pieces in between (cached per index content)."""
        plans = self._derived.setdefault("view_plans", {})
        if p not in plans:
            L = self.partitions[p].length
            by_dt: Dict[str, list] = {}
            for t in self.tensors:
                if t.partition == p:
                    by_dt.setdefault(t.dtype, []).append(t)
            plan = []
            for dt, ts in by_dt.items():
                w = WIDTH[dt]
                ts.sort(key=lambda t: t.offset)
                sizes, items, cur = [], [], 0
                for t in ts:   # offsets are multiples of A >= 16, sizes of the width
                    o, n = t.offset // w, t.nbytes // w
                    if o > cur:
                        sizes.append(o - cur)
                    items.append((t.name, len(sizes), t.shape))
                    sizes.append(n)
                    cur = o + n
                if L // w > cur:
                    sizes.append(L // w - cur)
                plan.append((dt, sizes, items))
            plans[p] = plan
        return plans[p]

    def find(self, name: str) -> int:
        i = C.c_size_t()
        check(lib().sllm_index_find(self._h, name.encode("utf-8"), C.byref(i)))
        return i.value

    def address(self, name: str, bases: Sequence[int]) -> Tuple[int, int]:
        """P:549 base + offset; bases[p] = base address of partition p."""
        arr = (C.c_uint64 * max(len(bases), 1))(*bases)
        d, a = C.c_int32(), C.c_uint64()
        check(lib().sllm_tensor_address(self._h, name.encode("utf-8"), arr, C.byref(d), C.byref(a)))
        return d.value, a.value

    def block_checksums(self, p: int) -> np.ndarray:
        t = C.POINTER(C.c_uint64)()
        check(lib().sllm_index_block_checksums(self._h, p, C.byref(t)))
        n = self.partitions[p].n_blocks
        return np.ctypeslib.as_array(t, shape=(n,)).copy() if n else np.zeros(0, np.uint64)


def convert(tensors: Sequence, out_dir: str, align: int = 4096, block: int = 1 << 20, model_id: str = "") -> None:
    """SPEC S:43 convert() to <out_dir>/part_<d>.bin + index.bin.  tensors:
    (name, device, dtype, shape, data_ptr) with host pointers."""
    arr, keep = _src_array(tensors)
    check(lib().sllm_convert(arr, len(tensors), align, block, model_id.encode(), out_dir.encode()))


def fletcher64(data) -> int:
    a = np.ascontiguousarray(np.frombuffer(memoryview(data).cast("B"), dtype=np.uint8)) \
        if not isinstance(data, np.ndarray) else np.ascontiguousarray(data.reshape(-1).view(np.uint8))
    out = C.c_uint64()
    check(lib().sllm_fletcher64_host(C.c_void_p(a.ctypes.data), a.size, C.byref(out)))
    return out.value


def chunk_count(length: int, chunk: int) -> int:
    out = C.c_uint64()
    check(lib().sllm_chunk_count(length, chunk, C.byref(out)))
    return out.value


def replica_slices(length: int, chunk: int, nranks: int) -> List[Tuple[int, int]]:
    arr = (C.c_uint64 * (2 * nranks))()
    check(lib().sllm_replica_slices(length, chunk, nranks, arr))
    return [(arr[2 * r], arr[2 * r + 1]) for r in range(nranks)]


def fanout_unit(chunk: int, fanout: str) -> int:
    """sllm_fanout_unit: the slice / round unit a load with this chunk size and fan-out uses
    (NCCL fan-outs: a whole >= 64 MiB window of chunks)."""
    out = C.c_uint64()
    check(lib().sllm_fanout_unit(chunk, {"none": 0, "bcast": 1, "p2p": 2, "allgather": 3, "nvls": 4}[fanout],
                                 C.byref(out)))
    return out.value


def replica_schedule(length: int, chunk: int, nranks: int) -> List[List[Tuple[int, int]]]:
    """The fan-out rounds the replicated load executes: rounds[r][q] = (lo, hi) that rank
    q broadcasts in round r (lo == hi: nothing)."""
    arr = (C.c_uint64 * (2 * nranks))()
    n = C.c_uint64()
    if length == 0:
        return []
    check(lib().sllm_replica_round(length, chunk, nranks, 0, arr, C.byref(n)))
    out = []
    for r in range(n.value):
        check(lib().sllm_replica_round(length, chunk, nranks, r, arr, None))
        out.append([(arr[2 * q], arr[2 * q + 1]) for q in range(nranks)])
    return out


def allgather_schedule(length: int, chunk: int, nranks: int) -> List[Tuple[bool, List[Tuple[int, int]]]]:
    """The rounds of fanout="allgather": (full, [(lo, hi) of rank q's chunk]) per round --
    chunk k belongs to rank k % nranks; a full round is one in-place all-gather of `chunk`
    bytes per rank, the ragged last round grouped broadcasts."""
    arr = (C.c_uint64 * (2 * nranks))()
    n = C.c_uint64()
    full = C.c_int32()
    if length == 0:
        return []
    check(lib().sllm_allgather_round(length, chunk, nranks, 0, arr, C.byref(n), None))
    out = []
    for r in range(n.value):
        check(lib().sllm_allgather_round(length, chunk, nranks, r, arr, None, C.byref(full)))
        out.append((bool(full.value), [(arr[2 * q], arr[2 * q + 1]) for q in range(nranks)]))
    return out


class HostBuffer:
    """Pinned, device-mapped host memory from sllm_host_alloc (the DRAM tier)."""

    def __init__(self, nbytes: int, gpu: int = -1):
        p = C.c_void_p()
        check(lib().sllm_host_alloc(int(nbytes), gpu, C.byref(p)))
        self.ptr = p.value
        self.nbytes = int(nbytes)

    @classmethod
    def read_partition(cls, directory: str, index: Index, p: int, gpu: int = -1, threads: int = 0) -> "HostBuffer":
        buf = cls(index.partitions[p].length, gpu)
        check(lib().sllm_host_read_partition(directory.encode(), index.handle, p, C.c_void_p(buf.ptr), threads))
        return buf

    def numpy(self) -> np.ndarray:
        return np.ctypeslib.as_array((C.c_uint8 * self.nbytes).from_address(self.ptr))

    def torch(self):
        import torch
        return torch.from_numpy(self.numpy())

    def free(self) -> None:
        if self.ptr:
            lib().sllm_host_free(C.c_void_p(self.ptr))
            self.ptr = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class PinnedCache:
    """The pinned DRAM tier as a whole-model LRU cache (sllm_cache_*; PAPER.md P:578-579,
    P:692).  ``acquire(dir)`` -> (Index, {partition: host pointer}) usable as
    ``sllm.load`` sources; the model stays resident and unevictable until ``release(dir)``."""

    def __init__(self, capacity: int, gpu: int = -1, pin: bool = True):
        out = C.c_void_p()
        check(lib().sllm_cache_create(int(capacity), gpu, int(pin), C.byref(out)))
        self._h = out

    def acquire(self, directory: str, io_threads: int = 0) -> Tuple["Index", Dict[int, int], bool]:
        idx, bufs, hit = C.c_void_p(), C.POINTER(C.c_void_p)(), C.c_int32()
        check(lib().sllm_cache_acquire(self._h, directory.encode(), io_threads, C.byref(idx), C.byref(bufs),
                                       C.byref(hit)))
        index = Index(idx.value, owned=False)
        return index, {p: bufs[p] for p in range(len(index.partitions))}, bool(hit.value)

    def release(self, directory: str) -> None:
        check(lib().sllm_cache_release(self._h, directory.encode()))

    def stats(self) -> dict:
        st = _abi.CacheStats()
        check(lib().sllm_cache_get_stats(self._h, C.byref(st)))
        return st.as_dict()

    def close(self) -> None:
        if self._h and self._h.value:
            lib().sllm_cache_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class LoadConfig:
    chunk_bytes: int = 16 << 20   # P:1279 "16MB" (read as MiB, Q9)
    n_streams: int = 2
    mode: str = "ce"              # ce | zerocopy | scatter_ce | scatter_zc | auto (ce or zerocopy by size) | gds (files)
    fanout: str = "none"          # none | bcast / allgather (NCCL) | p2p (fused NVLink stores) | nvls (multicast)
    verify: bool = True
    ctas: int = 0
    profile: int = 0              # 1 per-launch CUDA events (bench roofline), 2 + copies, 3 + in-kernel spans
    engine: str = "tma"           # tma (bulk-load smem ring) | tma_store (+ bulk stores) | ldg (register tiles)

    def to_c(self) -> _abi.LoadConfig:
        modes = {"ce": _abi.MODE_CE, "zerocopy": _abi.MODE_ZEROCOPY, "scatter_ce": _abi.MODE_SCATTER_CE,
                 "scatter_zc": _abi.MODE_SCATTER_ZC, "auto": _abi.MODE_AUTO, "gds": _abi.MODE_GDS}
        fan = {"none": _abi.FANOUT_NONE, "bcast": _abi.FANOUT_BCAST, "p2p": _abi.FANOUT_P2P,
               "allgather": _abi.FANOUT_ALLGATHER, "nvls": _abi.FANOUT_NVLS}
        return _abi.LoadConfig(self.chunk_bytes, self.n_streams, modes[self.mode], fan[self.fanout],
                               int(self.verify), self.ctas, int(self.profile),
                               {"tma": 1, "ldg": 2, "tma_store": 3}[self.engine], 0)

    @property
    def scatter(self) -> bool:
        return self.mode.startswith("scatter")


class Comm:
    """NCCL communicator for the replicated fan-out (sllm_comm*)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().sllm_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def init_rank(cls, uid: bytes, nranks: int, rank: int, gpu: int) -> "Comm":
        buf = C.create_string_buffer(bytes(uid), 128)
        out = C.c_void_p()
        check(lib().sllm_comm_init_rank(buf, nranks, rank, gpu, C.byref(out)))
        return cls(out.value)

    @classmethod
    def init_all(cls, gpus: Sequence[int]) -> List["Comm"]:
        """sllm_comm_init_all: one process driving several GPUs (ncclCommInitAll); handle i
        belongs to gpus[i] and is rank i of the group."""
        n = len(gpus)
        arr = (C.c_int32 * n)(*[int(g) for g in gpus])
        out = (C.c_void_p * n)()
        check(lib().sllm_comm_init_all(arr, n, out))
        return [cls(out[i]) for i in range(n)]

    @classmethod
    def from_process_group(cls, gpu: int, group=None) -> "Comm":
        """Build the communicator over a torch.distributed group (id exchanged through it)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls.init_rank(obj[0], world, rank, gpu)

    @classmethod
    def peers(cls, nranks: int, rank: int, gpu: int, peer_bases: Sequence[int], peer_signals: Sequence[int],
              timeout_ms: int = 0, keep: Optional[list] = None) -> "Comm":
        """Peer group for fanout="p2p" (sllm_comm_init_peers): device pointers, valid in
        this process, to every rank's replica and zero-filled signal array (2*nranks int32)."""
        out = C.c_void_p()
        check(lib().sllm_comm_init_peers(nranks, rank, gpu, _ptr_array(peer_bases), _ptr_array(peer_signals),
                                         timeout_ms, C.byref(out)))
        c = cls(out.value)
        c._keep = keep or []
        return c

    @classmethod
    def peers_from_process_group(cls, base, group=None, timeout_ms: int = 0) -> "Comm":
        """Collective over a torch.distributed group: export this rank's replica ``base`` (a
        CUDA uint8 tensor) and a fresh signal array with CUDA IPC, exchange the handles
        through the group, map the peers' and build the peer group."""
        import torch
        import torch.distributed as dist
        from . import ipc
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        gpu = base.device.index
        sig = torch.zeros(2 * world, dtype=torch.int32, device=base.device)
        torch.cuda.synchronize(gpu)
        mine = (ipc.export_region(base.data_ptr(), base.numel()), ipc.export_region(sig.data_ptr(), sig.numel() * 4))
        regions = [None] * world
        dist.all_gather_object(regions, mine, group=group)
        bases, sigs, opened = [], [], []
        for q, (rb, rs) in enumerate(regions):
            if q == rank:
                bases.append(base.data_ptr())
                sigs.append(sig.data_ptr())
            else:
                pb, ps = ipc.open_region(rb, gpu), ipc.open_region(rs, gpu)
                opened += [pb, ps]
                bases.append(pb)
                sigs.append(ps)
        c = cls.peers(world, rank, gpu, bases, sigs, timeout_ms, keep=[base, sig])
        c._opened = opened
        return c

    @classmethod
    def nvls(cls, gpus: Sequence[int], nbytes: int, timeout_ms: int = 0) -> List["Comm"]:
        """sllm_comm_init_nvls: an NVLink-SHARP multicast group over ``gpus`` driven by this
        process (handle i = rank i on gpus[i]) with library-owned replicas of >= ``nbytes``
        bound to it.  Raises SllmError(SLLM_E_INVALID) where the platform cannot create
        multicast objects (no NVSwitch fabric)."""
        n = len(gpus)
        arr = (C.c_int32 * n)(*[int(g) for g in gpus])
        out = (C.c_void_p * n)()
        check(lib().sllm_comm_init_nvls(arr, n, int(nbytes), int(timeout_ms), out))
        comms = [cls(out[i]) for i in range(n)]
        for i, c in enumerate(comms):
            c._gpu = int(gpus[i])
            c._group = comms          # the replicas live while any handle of the group does
        return comms

    def replica(self):
        """The replica a P2P / NVLS handle is bound to, as a zero-copy torch uint8 tensor
        (NVLS: library-owned memory, valid while the group's handles live)."""
        import torch
        base, n = C.c_void_p(), C.c_uint64()
        check(lib().sllm_comm_replica(self._h, C.byref(base), C.byref(n)))

        class _Mem:  # __cuda_array_interface__ view of the library's allocation
            __cuda_array_interface__ = {"shape": (n.value,), "typestr": "|u1", "data": (base.value, False),
                                        "version": 3, "strides": None}
        t = torch.as_tensor(_Mem(), device=f"cuda:{getattr(self, '_gpu', 0)}")
        return t

    @property
    def handle(self):
        return self._h

    def free(self):
        if self._h and self._h.value:
            lib().sllm_comm_free(self._h)
            self._h = C.c_void_p()
        from . import ipc
        for p in getattr(self, "_opened", []):
            ipc.close(p)
        self._opened = []

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class LoadResult:
    """An in-flight or finished load.  ``tensors`` are usable as addresses immediately
     and hold the checkpoint's bytes once ``wait()`` returned (Q17)."""

    def __init__(self, handle, index: Index, tensors: Dict[str, object], keep: list):
        self._h = handle
        self.index = index
        self.tensors = tensors
        self._keep = keep
        self.report: Optional[dict] = None

    def wait(self) -> dict:
        rep = _abi.LoadReport()
        st = lib().sllm_load_wait(self._h, C.byref(rep))
        self.report = rep.as_dict()
        check(st)
        return self.report

    def block_checksums(self, p: int) -> np.ndarray:
        t = C.POINTER(C.c_uint64)()
        check(lib().sllm_load_block_checksums(self._h, p, C.byref(t)))
        n = self.index.partitions[p].n_blocks
        return np.ctypeslib.as_array(t, shape=(n,)).copy() if n else np.zeros(0, np.uint64)

    def handle_of(self, name: str) -> dict:
        h = _abi.TensorHandle()
        check(lib().sllm_load_tensor(self._h, name.encode("utf-8"), C.byref(h)))
        return {"gpu": h.gpu, "ptr": h.ptr, "dtype": _abi.DTYPE_NAME[h.dtype], "shape": tuple(h.shape[:h.ndim]),
                "nbytes": h.nbytes}

    def free(self):
        if self._h is not None and self._h.value:
            lib().sllm_load_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _views(index: Index, parts, bases, per_tensor, scatter: bool) -> Dict[str, object]:
    """{name: torch tensor} of a load: scatter -> the caller's per-tensor buffers; contiguous
    -> zero-copy views base + offset, made with one typed split of each
    partition's base per dtype (the view plan) and a reshape per tensor."""
    tensors: Dict[str, object] = {}
    parts = set(parts)
    if scatter:
        for t in index.tensors:
            if t.partition in parts:
                tensors[t.name] = per_tensor[t.name]
        return tensors
    tdt = _torch_dtypes()
    for p in sorted(parts):
        base = bases[p]
        for dt, sizes, items in index.view_plan(p):
            pieces = base.view(tdt[dt]).split(sizes)
            for name, k, shape in items:
                tensors[name] = pieces[k].view(shape)
    return tensors


def allocate(index: Index, gpus: Dict[int, int], scatter: bool = False, partitions: Optional[Iterable[int]] = None):
    """Destination memory through PyTorch's allocator: one uint8 base of L_p bytes per
    partition (contiguous) or one tensor per index entry (scatter)."""
    import torch
    parts = index.partitions
    sel = sorted(gpus) if partitions is None else sorted(partitions)
    bases: Dict[int, object] = {}
    per_tensor: Dict[str, object] = {}
    tdt = _torch_dtypes()
    if not scatter:
        for p in sel:
            bases[p] = torch.empty(parts[p].length, dtype=torch.uint8, device=f"cuda:{gpus[p]}")
    else:
        for t in index.tensors:
            if t.partition in sel:
                per_tensor[t.name] = torch.empty(t.shape, dtype=tdt[t.dtype], device=f"cuda:{gpus[t.partition]}")
    return bases, per_tensor


def load_start(index: Index, sources: Dict[int, object], gpus: Dict[int, int], config: Optional[LoadConfig] = None,
               bases: Optional[Dict[int, object]] = None, per_tensor: Optional[Dict[str, object]] = None,
               streams: Optional[Dict[int, object]] = None, comm: Optional[Comm] = None) -> LoadResult:
    """sllm_load_start over preallocated destinations.  sources[p]: HostBuffer or an int
    host pointer (pinned); gpus[p]: CUDA ordinal; bases[p]: torch uint8 tensor (contiguous)
    or per_tensor[name]: torch tensor (scatter)."""
    import torch
    cfg = config or LoadConfig()
    parts = index.partitions
    n = len(parts)
    src = [None] * n
    gpu = (C.c_int32 * max(n, 1))()
    for p, s in sources.items():
        src[p] = s.ptr if isinstance(s, HostBuffer) else int(s)
        gpu[p] = int(gpus[p])
    dst_base = None
    dst_tensor = None
    if not cfg.scatter:
        dst_base = _ptr_array([bases[p].data_ptr() if p in (bases or {}) else None for p in range(n)])
    else:
        dst_tensor = _ptr_array([per_tensor[t.name].data_ptr() if t.partition in sources else None
                                 for t in index.tensors])
    st = None
    if streams:
        st = _ptr_array([streams[p].cuda_stream if p in streams else None for p in range(n)])
    out = C.c_void_p()
    ccfg = cfg.to_c()
    check(lib().sllm_load_start(index.handle, C.byref(ccfg), _ptr_array(src), gpu, dst_base, dst_tensor, st,
                                comm.handle if comm else None, C.byref(out)))
    # The tensor objects are built while the transfer runs (the inference
    # process sets base + offset pointers before the data has arrived).
    tensors = _views(index, sources.keys(), bases, per_tensor, cfg.scatter)
    return LoadResult(out, index, tensors, [dst_base, dst_tensor, st, bases, per_tensor, sources])


class CapturedLoad(LoadResult):
    """sllm_load_capture: the load recorded once as one CUDA graph per partition; every
    ``replay()`` loads the checkpoint again into the same destinations (one graph launch per
    partition) and ``wait()`` reports that replay's verification."""

    def replay(self, streams: Optional[Dict[int, object]] = None) -> "CapturedLoad":
        n = len(self.index.partitions)
        st = None
        if streams:
            st = _ptr_array([streams[p].cuda_stream if p in streams else None for p in range(n)])
        check(lib().sllm_load_replay(self._h, st))
        return self


def load_capture(index: Index, sources: Dict[int, object], gpus: Dict[int, int], config: Optional[LoadConfig] = None,
                 bases: Optional[Dict[int, object]] = None, per_tensor: Optional[Dict[str, object]] = None
                 ) -> CapturedLoad:
    """sllm_load_capture over preallocated destinations (arguments as ``load_start``; no
    fan-out, no streams: each ``replay`` takes them)."""
    cfg = config or LoadConfig()
    parts = index.partitions
    n = len(parts)
    src = [None] * n
    gpu = (C.c_int32 * max(n, 1))()
    for p, s in sources.items():
        src[p] = s.ptr if isinstance(s, HostBuffer) else int(s)
        gpu[p] = int(gpus[p])
    dst_base = dst_tensor = None
    if not cfg.scatter:
        dst_base = _ptr_array([bases[p].data_ptr() if p in (bases or {}) else None for p in range(n)])
    else:
        dst_tensor = _ptr_array([per_tensor[t.name].data_ptr() if t.partition in sources else None
                                 for t in index.tensors])
    out = C.c_void_p()
    ccfg = cfg.to_c()
    check(lib().sllm_load_capture(index.handle, C.byref(ccfg), _ptr_array(src), gpu, dst_base, dst_tensor,
                                  C.byref(out)))
    tensors = _views(index, sources.keys(), bases, per_tensor, cfg.scatter)
    return CapturedLoad(out, index, tensors, [dst_base, dst_tensor, bases, per_tensor, sources])


def load_files(index: Index, directory: str, gpus: Dict[int, int], config: Optional[LoadConfig] = None,
               io_threads: int = 0, wait: bool = True, stream_of_caller: bool = True,
               bases: Optional[Dict[int, object]] = None, per_tensor: Optional[Dict[str, object]] = None,
               comm: Optional[Comm] = None) -> LoadResult:
    """The full multi-tier pipeline from <directory>/part_<device>.bin (sllm_load_files_start):
    O_DIRECT readers -> pinned slot ring -> GPU, for the partitions listed in ``gpus``.  With
    a fan-out config and ``comm`` (replicated checkpoint) this rank reads only its slice."""
    import torch
    cfg = config or LoadConfig()
    if bases is None and per_tensor is None:
        bases, per_tensor = allocate(index, gpus, cfg.scatter, partitions=gpus.keys())
    parts = index.partitions
    n = len(parts)
    gpu = (C.c_int32 * max(n, 1))(*([-1] * max(n, 1)))
    for p, g in gpus.items():
        gpu[p] = int(g)
    dst_base = dst_tensor = None
    if not cfg.scatter:
        dst_base = _ptr_array([bases[p].data_ptr() if p in bases else None for p in range(n)])
    else:
        dst_tensor = _ptr_array([per_tensor[t.name].data_ptr() if t.partition in gpus else None for t in index.tensors])
    streams = {p: torch.cuda.current_stream(gpus[p]) for p in gpus} if stream_of_caller else {}
    st = _ptr_array([streams[p].cuda_stream if p in streams else None for p in range(n)]) if streams else None
    out = C.c_void_p()
    ccfg = cfg.to_c()
    check(lib().sllm_load_files_start(index.handle, C.byref(ccfg), directory.encode(), gpu, dst_base, dst_tensor, st,
                                      io_threads, comm.handle if comm else None, C.byref(out)))
    tensors = _views(index, gpus.keys(), bases, per_tensor, cfg.scatter)
    res = LoadResult(out, index, tensors, [dst_base, dst_tensor, st, bases, per_tensor, None])
    if wait:
        res.wait()
    return res


def load(index: Index, sources: Dict[int, object], gpus: Dict[int, int], config: Optional[LoadConfig] = None,
         wait: bool = True, comm: Optional[Comm] = None, stream_of_caller: bool = True) -> LoadResult:
    """Allocate destinations with torch, start the load and (by default) wait for it --
    the whole "time-to-loaded-model" path (Q19)."""
    import torch
    cfg = config or LoadConfig()
    bases, per_tensor = allocate(index, gpus, cfg.scatter, partitions=sources.keys())
    streams = {p: torch.cuda.current_stream(gpus[p]) for p in sources} if stream_of_caller else None
    res = load_start(index, sources, gpus, cfg, bases, per_tensor, streams, comm)
    if wait:
        res.wait()
    return res


def trim_device_cache(gpu: int, keep_bytes: int = 0) -> None:
    """sllm_device_trim: hand the library's idle cached device memory (scratch, SCATTER_CE
    staging) on ``gpu`` back to the driver, down to ``keep_bytes``."""
    check(lib().sllm_device_trim(gpu, keep_bytes))


def block_checksums_device(src_ptr: int, length: int, block: int, out_ptr: int, ctas: int = 0, stream=None) -> None:
    check(lib().sllm_block_checksums_device(C.c_void_p(src_ptr), length, block, C.c_void_p(out_ptr), ctas,
                                            C.c_void_p(stream.cuda_stream if stream is not None else 0)))


def materialise_device(index: Index, p: int, src_ptr: int, per_tensor: Dict[str, object], ctas: int = 0,
                       stream=None, timed: bool = False) -> Optional[float]:
    """K3 over a device-resident partition image.  timed=True returns the launch's device
    time in ms (CUDA events around the launch only)."""
    infos = index.tensors
    arr = _ptr_array([per_tensor[t.name].data_ptr() if t.partition == p else None for t in infos])
    bad = C.c_uint64()
    ms = C.c_float(-1.0)
    check(lib().sllm_materialise_device(index.handle, p, C.c_void_p(src_ptr), arr, ctas,
                                        C.c_void_p(stream.cuda_stream if stream is not None else 0), C.byref(bad),
                                        C.byref(ms) if timed else None))
    return float(ms.value) if timed else None
