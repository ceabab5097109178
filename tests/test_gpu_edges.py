"""GPU parity on the degenerate and boundary cases of the method:
an empty checkpoint (no partitions), a checkpoint holding one 2-byte scalar
(partition = one alignment unit, one short block), a partition shorter than one chunk and
one exactly one chunk long, a tensor straddling every chunk boundary of a 1 MiB-chunk
load, sparse device ids mapped onto one GPU (Q15), and checksum blocks of 16 bytes (the
smallest block the format allows at A = 16).  Every mode, every byte against the oracle."""
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


def load_and_check(inv, seed, A, B, chunk, mode, gpus=None):
    payloads = [payload.payload_bytes(seed, e, t.nbytes) for e, t in enumerate(inv)]
    lay, oparts = olayout.convert([(t.name, t.device, t.dtype, t.shape, p) for t, p in zip(inv, payloads)], A, B)
    idx, bufs = workloads.build_pinned(inv, seed, A, B)
    gpus = gpus or {p: 0 for p in bufs}
    res = sllm.load(idx, bufs, gpus, sllm.LoadConfig(chunk_bytes=chunk, mode=mode))
    rep = res.report
    assert rep["bad_partition"] == -1
    assert rep["payload_bytes"] == lay.payload_bytes
    assert rep["transferred_bytes"] == sum(lay.partitions.values())
    for e, t in enumerate(inv):
        got = res.tensors[t.name]
        b = got.contiguous().view(torch.uint8).reshape(-1) if got.dim() else got.reshape(1).view(torch.uint8)
        assert np.array_equal(b.cpu().numpy(), payloads[e]), (mode, t.name)
    for p, d in enumerate(lay.devices()):
        if not mode.startswith("scatter"):
            assert np.array_equal(res._keep[3][p].cpu().numpy(), oparts[d]), (mode, p)
        assert res.block_checksums(p).tolist() == lay.checksums[d], (mode, p)
    return res


@pytest.mark.parametrize("mode", MODES)
def test_empty_checkpoint(mode):
    idx = workloads.plan_inventory([], 4096, 1 << 20)
    idx.seal([])
    assert len(idx.partitions) == 0
    res = sllm.load(idx, {}, {}, sllm.LoadConfig(mode=mode))
    assert res.report["payload_bytes"] == 0 and res.report["transferred_bytes"] == 0 and res.tensors == {}


@pytest.mark.parametrize("mode", MODES)
def test_single_scalar(mode):
    inv = [models.TensorSpec("s", 0, "f16", ())]
    load_and_check(inv, 5, 4096, 1 << 20, 1 << 20, mode)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("n_bytes", [(1 << 20) - 4096, 1 << 20, (2 << 20) + 8192])
def test_partition_vs_one_chunk(mode, n_bytes):
    """L shorter than and equal to one 1 MiB chunk, and one 2 MiB chunk plus an 8 KiB tail."""
    inv = [models.TensorSpec("a", 0, "u8", (n_bytes - 4096 - 16,)), models.TensorSpec("b", 0, "u8", (16,))]
    assert workloads.plan_inventory(inv, 4096, 1 << 20).partitions[0].length == n_bytes
    load_and_check(inv, 6, 4096, 1 << 20, 2 << 20 if n_bytes > (2 << 20) else 1 << 20, mode)


@pytest.mark.parametrize("mode", MODES)
def test_tensor_straddles_every_chunk(mode):
    """One 7.5 MiB tensor after a 3-byte one: with 1 MiB chunks and A = 16 every chunk and
    block boundary falls inside it at an offset that is not a multiple of 4 KiB."""
    inv = [models.TensorSpec("tiny", 0, "u8", (3,)), models.TensorSpec("big", 0, "u8", ((15 << 19) + 5,)),
           models.TensorSpec("tail", 0, "f32", (7,))]
    load_and_check(inv, 7, 16, 1 << 20, 1 << 20, mode)


@pytest.mark.parametrize("mode", MODES)
def test_sparse_device_ids_on_one_gpu(mode):
    """Partitions of logical devices 3 and 9 (Q15), both on cuda:0."""
    inv = [models.TensorSpec("x@3", 3, "bf16", (1000, 33)), models.TensorSpec("y@9", 9, "i64", (12345,)),
           models.TensorSpec("z@3", 3, "i8", (1,))]
    load_and_check(inv, 8, 4096, 1 << 20, 1 << 20, mode)


@pytest.mark.parametrize("mode", MODES)
def test_smallest_blocks(mode):
    """B = A = 16: one checksum per 16-byte vector (the kernels' unit is one block)."""
    inv, seed = models.model_inventory("toy")
    inv = inv[:6] + inv[-2:]
    load_and_check(inv, seed, 16, 16, 64 << 10, mode)


def test_device_trim_releases_staging():
    """A finished SCATTER_CE load returns its staging ring to the stream-ordered pool (cached
    for the next load); sllm_device_trim hands that idle memory back to the driver."""
    mid = models.llama2(1024, 12, 4096, 1024, vocab=32000)  # ~0.53 GB, 3 staging windows
    idx, bufs = workloads.build_pinned(mid, 9, 4096, 1 << 20)
    res = sllm.load(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=64 << 20, mode="scatter_ce"))
    assert np.array_equal(res.block_checksums(0), idx.block_checksums(0))
    torch.cuda.synchronize()
    before = torch.cuda.mem_get_info(0)[0]
    sllm.trim_device_cache(0)
    after = torch.cuda.mem_get_info(0)[0]
    assert after - before >= 256 << 20, (before, after)
    res2 = sllm.load(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=64 << 20, mode="scatter_ce"))  # regrows
    assert np.array_equal(res2.block_checksums(0), idx.block_checksums(0))
    with pytest.raises(sllm.SllmError):
        sllm.trim_device_cache(-1)
