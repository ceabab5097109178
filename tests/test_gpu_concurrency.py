"""Concurrent loads from several host threads into one GPU (a serving process loading
several models at once; P:721 requests arrive independently): every thread runs its own
sequence of loads of its own random checkpoint in its own mode, engine, chunk size and
stream count, with and without the caller-stream gate, while the others are in flight.
Every result is checked byte for byte against the oracle; the library's per-GPU stream
sets, stream gates and stream-ordered scratch must keep the loads independent."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2401_14351_b200 as sllm  # noqa: E402
from paper_2401_14351_b200 import workloads  # noqa: E402
from oracle import layout as olayout  # noqa: E402
from synth import models, payload  # noqa: E402

MODES = ["ce", "zerocopy", "scatter_ce", "scatter_zc"]


def _worker(t, reps, errors):
    try:
        torch.cuda.set_device(0)
        stream = torch.cuda.Stream()  # each thread gates its own stream
        rng = np.random.default_rng(9000 + t)
        inv = models.random_inventory(rng, int(rng.integers(50, 600)), int(rng.integers(1, 3)), 48 << 20)
        A, B = 4096, 1 << 20
        seed = 100 + t
        idx, bufs = workloads.build_pinned(inv, seed, A, B)
        payloads = [payload.payload_bytes(seed, e, x.nbytes) for e, x in enumerate(inv)]
        lay, oparts = olayout.convert([(x.name, x.device, x.dtype, x.shape, p) for x, p in zip(inv, payloads)], A, B)
        n = len(idx.partitions)
        for r in range(reps):
            mode = MODES[(t + r) % 4]
            cfg = sllm.LoadConfig(chunk_bytes=int(rng.choice([1, 2, 4])) << 20, n_streams=int(rng.integers(1, 4)),
                                  mode=mode, engine=["tma", "tma_store"][r % 2])
            with torch.cuda.stream(stream):
                res = sllm.load(idx, bufs, {p: 0 for p in range(n)}, cfg, stream_of_caller=bool(r % 2))
            stream.synchronize()
            for e, x in enumerate(inv):
                got = res.tensors[x.name]
                b = got.contiguous().view(torch.uint8).reshape(-1) if got.dim() else got.reshape(1).view(torch.uint8)
                if not np.array_equal(b.cpu().numpy(), payloads[e]):
                    errors.append((t, r, mode, x.name))
                    return
            for p, d in enumerate(lay.devices()):
                if res.block_checksums(p).tolist() != lay.checksums[d]:
                    errors.append((t, r, mode, "checksums", p))
                    return
            del res
    except Exception as ex:  # noqa: BLE001
        errors.append((t, repr(ex)))


def test_concurrent_loads_from_threads():
    errors = []
    threads = [threading.Thread(target=_worker, args=(t, 10, errors)) for t in range(8)]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=600)
    assert not any(th.is_alive() for th in threads), "a loader thread hung"
    assert not errors, errors


def _file_worker(t, tmpdir, reps, errors):
    try:
        torch.cuda.set_device(0)
        stream = torch.cuda.Stream()
        rng = np.random.default_rng(9500 + t)
        inv = models.random_inventory(rng, int(rng.integers(50, 400)), int(rng.integers(1, 3)), 40 << 20)
        seed = 300 + t
        payloads = [payload.payload_bytes(seed, e, x.nbytes) for e, x in enumerate(inv)]
        d = f"{tmpdir}/ckpt{t}"
        sllm.convert([(x.name, x.device, x.dtype, x.shape, p.ctypes.data) for x, p in zip(inv, payloads)], d,
                     4096, 1 << 20, f"t{t}")
        idx = sllm.Index.open(f"{d}/index.bin")
        n = len(idx.partitions)
        for r in range(reps):
            mode = ["ce", "zerocopy", "scatter_ce", "scatter_zc"][(t + r) % 4]
            with torch.cuda.stream(stream):
                res = sllm.load_files(idx, d, {p: 0 for p in range(n)},
                                      sllm.LoadConfig(chunk_bytes=2 << 20, mode=mode), io_threads=2,
                                      stream_of_caller=bool(r % 2))
            stream.synchronize()
            for e, x in enumerate(inv):
                got = res.tensors[x.name]
                b = got.contiguous().view(torch.uint8).reshape(-1) if got.dim() else got.reshape(1).view(torch.uint8)
                if not np.array_equal(b.cpu().numpy(), payloads[e]):
                    errors.append((t, r, mode, x.name))
                    return
            del res
    except Exception as ex:  # noqa: BLE001
        errors.append((t, repr(ex)))


def test_concurrent_file_and_pinned_loads(tmp_path):
    """File-tier loads (caller stream ordered at wait) and pinned loads (ordered at start)
    in flight together from separate threads."""
    errors = []
    threads = [threading.Thread(target=_worker, args=(t, 6, errors)) for t in range(3)] + \
              [threading.Thread(target=_file_worker, args=(t, str(tmp_path), 4, errors)) for t in range(3)]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=600)
    assert not any(th.is_alive() for th in threads), "a loader thread hung"
    assert not errors, errors
