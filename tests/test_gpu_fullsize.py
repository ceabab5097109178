"""Full-size parity for the multi-partition configs (BASELINE configs[2], configs[3]):
every partition of LLaMA-2-13B TP2 (2 x 13.0 GB) and of the north star's target checkpoint,
LLaMA-2-70B TP8 (8 x 17.25 GB = 138 GB), loaded in the bench launch configuration (CE,
64 MiB chunks, verification on).  Only one GPU is available, so every partition goes to
cuda:0 -- eight worker threads, eight pipelines, one PCIe link.

Checked: every block checksum the GPU computes equals the index table (all 16,448 blocks
of every partition), the index tables equal the oracle's Fletcher-64 on sampled blocks of
the pinned source, sampled tensors equal their payload regenerated on the host, and the
report's byte counts equal the oracle layout's.  Skipped when the box lacks the host RAM
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
            t = inv[e]
            n = min(t.nbytes, 1 << 20)
            got = res.tensors[t.name].reshape(-1).view(torch.uint8)[:n].cpu().numpy()
            assert np.array_equal(got, payload.payload_bytes(seed, e, t.nbytes)[:n]), t.name
            tail = res.tensors[t.name].reshape(-1).view(torch.uint8)[-n:].cpu().numpy()
            assert np.array_equal(tail, payload.payload_bytes(seed, e, t.nbytes)[-n:]), t.name
        del res
    finally:
        for b in bufs.values():
            b.free()
        torch.cuda.empty_cache()
