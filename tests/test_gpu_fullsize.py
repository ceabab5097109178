"""Full-size parity for the multi-partition configs (BASELINE configs[2], configs[3]):
every partition of LLaMA-2-13B TP2 (2 x 13.0 GB) and of the north star's target checkpoint,
LLaMA-2-70B TP8 (8 x 17.25 GB = 138 GB), loaded in the bench launch configuration (CE,
64 MiB chunks, verification on).  Only one GPU is available, so every partition goes to
cuda:0 -- eight worker threads, eight pipelines, one PCIe link.

Checked: every block checksum the GPU computes equals the index table (all 16,448 blocks
of every partition), the index tables equal the oracle's Fletcher-64 on sampled blocks of
the pinned source, every byte of every tensor equals its payload regenerated on the host,
and the report's byte counts equal the oracle layout's.  Skipped when the box lacks the host RAM
or HBM to hold the checkpoint."""
import os
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2401_14351_b200 as sllm  # noqa: E402
from paper_2401_14351_b200 import workloads  # noqa: E402
from oracle import fletcher, layout as olayout  # noqa: E402
from synth import models, payload  # noqa: E402


def host_ram():
    return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")


def every_tensor_equals_payload(tensors, inv, seed):
    """Every byte of every loaded tensor against its payload regenerated on the host (O10,
    the multi-threaded C generator pinned to the NumPy definition in test_synth.py), one
    tensor at a time through a pinned scratch buffer; the comparison is torch.equal on the
    device.  Returns the bytes compared."""
    big = max(t.nbytes for t in inv)
    host = torch.empty(big, dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(big, dtype=torch.uint8, device="cuda")
    total = 0
    for e, t in enumerate(inv):
        n = t.nbytes
        payload.payload_into([host.data_ptr()], [n], seed, [e])
        dev[:n].copy_(host[:n])
        got = tensors[t.name].reshape(-1).view(torch.uint8)
        assert got.numel() == n and torch.equal(got, dev[:n]), t.name
        total += n
    del host, dev
    return total


@pytest.mark.parametrize("config,need", [("llama2-13b-tp2", 27e9), ("llama2-70b-tp8", 138e9)])
def test_partitioned_checkpoint_full_size(config, need):
    free, total = torch.cuda.mem_get_info(0)
    if host_ram() < need * 1.25 or free < need * 1.05:
        pytest.skip(f"{config} needs {need / 1e9:.0f} GB of host RAM and HBM")
    inv, seed = models.model_inventory(config)
    lay = olayout.plan([(t.name, t.device, t.dtype, t.shape, t.nbytes) for t in inv], 4096, 1 << 20)
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20, config, gpu_of={p: 0 for p in range(8)}, threads=0)
    try:
        parts = sorted(bufs)
        assert [idx.partitions[p].length for p in parts] == [lay.partitions[d] for d in lay.devices()]
        assert [(t.name, t.offset, t.nbytes) for t in idx.tensors] == [(e.name, e.offset, e.size) for e in lay.entries]
        rng = np.random.default_rng(7)
        for p in parts:  # index tables vs the oracle's Fletcher-64 on sampled blocks of the source
            src, table = bufs[p].numpy(), idx.block_checksums(p)
            nb = idx.partitions[p].n_blocks
            for j in sorted(set(rng.integers(0, nb, size=6).tolist()) | {0, nb - 1}):
                assert int(table[j]) == fletcher.f64_closed(src[j << 20:(j + 1) << 20]), (p, j)
        cfg = sllm.LoadConfig(chunk_bytes=64 << 20, mode="ce")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = sllm.load(idx, bufs, {p: 0 for p in parts}, cfg)
        dt = time.perf_counter() - t0
        rep = res.report
        assert rep["bad_partition"] == -1
        assert rep["payload_bytes"] == lay.payload_bytes
        assert rep["transferred_bytes"] == sum(lay.partitions.values())
        print(f"{config}: {rep['payload_bytes'] / 1e9:.2f} GB on one GPU in {dt:.3f} s "
              f"({rep['payload_bytes'] / dt / 1e9:.1f} GB/s incl. allocation)")
        for p in parts:  # every block verified on the GPU, equal to the index table
            assert np.array_equal(res.block_checksums(p), idx.block_checksums(p)), p
        for e in sorted(set(rng.integers(0, len(inv), size=16).tolist()) | {0, len(inv) - 1}):
            t = inv[e]  # sampled heads and tails against the NumPy definition itself
            n = min(t.nbytes, 1 << 20)
            got = res.tensors[t.name].reshape(-1).view(torch.uint8)[:n].cpu().numpy()
            assert np.array_equal(got, payload.payload_bytes(seed, e, t.nbytes)[:n]), t.name
            tail = res.tensors[t.name].reshape(-1).view(torch.uint8)[-n:].cpu().numpy()
            assert np.array_equal(tail, payload.payload_bytes(seed, e, t.nbytes)[-n:]), t.name
        t0 = time.perf_counter()
        checked = every_tensor_equals_payload(res.tensors, inv, seed)  # every tensor, every byte
        assert checked == lay.payload_bytes
        print(f"{config}: all {len(inv)} tensors ({checked / 1e9:.2f} GB) byte-equal to their payload "
              f"({time.perf_counter() - t0:.1f} s)")
        del res
    finally:
        for b in bufs.values():
            b.free()
        torch.cuda.empty_cache()


def test_replicated_opt30b_full_size_p2p():
    """BASELINE configs[4] at full size: the OPT-30B-shaped replicated checkpoint (one
    59.95 GB partition) loaded by a 2-rank P2P fan-out group whose replicas
    share the one GPU -- rank r reads slice r over PCIe, its kernel stores every vector into
    both replicas.  Checked: each rank moved exactly its slice (Σ = L, every byte crossed
    PCIe once), every block checksum of both replicas equals the index table, the index
    table equals the oracle's Fletcher-64 on sampled source blocks, the replicas are equal
    (compared 1 GiB at a time on the device), and sampled tensors of both replicas equal
    their regenerated payload."""
    need = 59.95e9
    free, total = torch.cuda.mem_get_info(0)
    if host_ram() < need * 1.3 or free < 2 * need * 1.03:
        pytest.skip("the replicated OPT-30B check needs 60 GB of host RAM and 120 GB of HBM")
    inv, seed = models.model_inventory("opt-30b")
    lay = olayout.plan([(t.name, t.device, t.dtype, t.shape, t.nbytes) for t in inv], 4096, 1 << 20)
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20, "opt-30b", gpu_of={0: 0}, threads=0)
    bases = sigs = comms = None
    try:
        L = idx.partitions[0].length
        assert L == lay.partitions[0] and idx.info()["payload_bytes"] == lay.payload_bytes
        rng = np.random.default_rng(11)
        src, table = bufs[0].numpy(), idx.block_checksums(0)
        nb = idx.partitions[0].n_blocks
        for j in sorted(set(rng.integers(0, nb, size=6).tolist()) | {0, nb - 1}):
            assert int(table[j]) == fletcher.f64_closed(src[j << 20:(j + 1) << 20]), j
        R, chunk = 2, 64 << 20
        bases = [torch.empty(L, dtype=torch.uint8, device="cuda") for _ in range(R)]
        sigs = [torch.zeros(2 * R, dtype=torch.int32, device="cuda") for _ in range(R)]
        comms = [sllm.Comm.peers(R, r, 0, [b.data_ptr() for b in bases], [s.data_ptr() for s in sigs], 60000)
                 for r in range(R)]
        slices = sllm.replica_slices(L, chunk, R)
        cfg = sllm.LoadConfig(chunk_bytes=chunk, mode="ce", fanout="p2p")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        results = [sllm.load_start(idx, bufs, {0: 0}, cfg, {0: bases[r]}, None, None, comms[r]) for r in range(R)]
        reports, errs = [], []
        for r, res in enumerate(results):  # wait for every rank: the first error is the one to report
            try:
                reports.append(res.wait())
            except sllm.SllmError as ex:
                errs.append((r, str(ex)))
        dt = time.perf_counter() - t0
        assert not errs, errs
        print(f"opt-30b replicated x{R} (P2P, one GPU, one PCIe link): {L / 1e9:.2f} GB per replica, "
              f"{R} replicas in {dt:.3f} s; PCIe bytes {sum(r['transferred_bytes'] for r in reports) / 1e9:.2f} GB")
        for r, rep in enumerate(reports):
            lo, hi = slices[r]
            assert rep["bad_partition"] == -1
            assert rep["transferred_bytes"] == hi - lo and rep["fanout_bytes"] == L - (hi - lo)
            assert np.array_equal(results[r].block_checksums(0), table), r
        assert sum(rep["transferred_bytes"] for rep in reports) == L
        step = 1 << 30
        for o in range(0, L, step):
            assert torch.equal(bases[0][o:o + step], bases[1][o:o + step]), o
        for e in sorted(set(rng.integers(0, len(inv), size=12).tolist()) | {0, len(inv) - 1}):
            t = inv[e]
            n = min(t.nbytes, 1 << 20)
            want = payload.payload_bytes(seed, e, t.nbytes)
            for r in range(R):
                v = results[r].tensors[t.name].reshape(-1).view(torch.uint8)
                assert np.array_equal(v[:n].cpu().numpy(), want[:n]), (r, t.name)
                assert np.array_equal(v[-n:].cpu().numpy(), want[-n:]), (r, t.name)
        # every tensor of replica 0, every byte (replica 1 equals replica 0, checked above)
        assert every_tensor_equals_payload(results[0].tensors, inv, seed) == lay.payload_bytes
        del results
    finally:
        if comms:
            for c in comms:
                c.free()
        del bases, sigs
        for b in bufs.values():
            b.free()
        torch.cuda.empty_cache()
