"""File tier: partition files -> O_DIRECT readers
-> pinned slot ring -> GPU, exact against the oracle for every mode, with slot reuse
(more windows than ring slots), several partitions, corruption and I/O errors."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2401_14351_b200 as sllm  # noqa: E402
from oracle import layout as olayout  # noqa: E402
from synth import models, payload  # noqa: E402

MODES = ["ce", "zerocopy", "scatter_ce", "scatter_zc"]


def write_ckpt(tmp_path, inv, seed, A=4096, B=1 << 20):
    payloads = [payload.payload_bytes(seed, e, t.nbytes) for e, t in enumerate(inv)]
    srcs = [(t.name, t.device, t.dtype, t.shape, p.ctypes.data) for t, p in zip(inv, payloads)]
    sllm.convert(srcs, str(tmp_path), A, B, "files")
    lay, parts = olayout.convert([(t.name, t.device, t.dtype, t.shape, p) for t, p in zip(inv, payloads)], A, B)
    return sllm.Index.open(str(tmp_path / "index.bin")), lay, parts, payloads


def check(res, inv, payloads, lay, parts_loaded):
    for e, t in enumerate(inv):
        if lay.devices().index(t.device) in parts_loaded:
            got = res.tensors[t.name].reshape(-1).view(torch.uint8).cpu().numpy()
            assert np.array_equal(got, payloads[e]), t.name
    for p in parts_loaded:
        assert res.block_checksums(p).tolist() == lay.checksums[lay.devices()[p]]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("io_threads", [1, 3])
def test_toy_from_files(tmp_path, mode, io_threads):
    inv, seed = models.model_inventory("toy")
    idx, lay, parts, payloads = write_ckpt(tmp_path, inv, seed)
    res = sllm.load_files(idx, str(tmp_path), {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20, mode=mode),
                          io_threads=io_threads)
    assert res.report["transferred_bytes"] == 13_594_624
    assert res.report["storage_bytes"] == 13_594_624  # every partition byte read from storage once
    check(res, inv, payloads, lay, [0])


@pytest.mark.parametrize("mode", ["ce", "zerocopy", "scatter_ce"])
def test_ring_reuse_and_partitions(tmp_path, mode):
    """~1.1 GB over two partitions: 9 windows per partition against a 4-slot ring
    (io_threads=2), A = 16 so the tail of each file needs a buffered read."""
    inv = models.llama2(1024, 36, 4096, 256, vocab=8192, tp=2)
    inv = [models.TensorSpec(t.name, t.device, t.dtype, t.shape) for t in inv] + \
          [models.TensorSpec("odd@0", 0, "u8", (33,)), models.TensorSpec("odd@1", 1, "f16", ())]
    idx, lay, parts, payloads = write_ckpt(tmp_path, inv, 77, A=16, B=1 << 20)
    assert all(p.length > 5 * (64 << 20) for p in idx.partitions)
    res = sllm.load_files(idx, str(tmp_path), {0: 0, 1: 0}, sllm.LoadConfig(chunk_bytes=4 << 20, mode=mode),
                          io_threads=2)
    check(res, inv, payloads, lay, [0, 1])


def test_file_corruption_names_block(tmp_path):
    inv, seed = models.model_inventory("toy")
    idx, lay, parts, payloads = write_ckpt(tmp_path, inv, seed)
    path = tmp_path / "part_0.bin"
    data = bytearray(open(path, "rb").read())
    pos = 5 * (1 << 20) + 12345
    data[pos] ^= 0x40
    open(path, "wb").write(bytes(data))
    with pytest.raises(sllm.SllmError) as ex:
        sllm.load_files(idx, str(tmp_path), {0: 0}, sllm.LoadConfig(chunk_bytes=2 << 20))
    assert ex.value.status == 9 and "block 5" in ex.value.message


def test_missing_file_is_io_error(tmp_path):
    inv, seed = models.model_inventory("toy")
    idx, lay, parts, payloads = write_ckpt(tmp_path, inv, seed)
    os.remove(tmp_path / "part_0.bin")
    with pytest.raises(sllm.SllmError) as ex:
        sllm.load_files(idx, str(tmp_path), {0: 0}, sllm.LoadConfig())
    assert ex.value.status == 6
    # the pinned pool and stream gate survive the failure: a good load still works
    idx2, lay2, _, payloads2 = write_ckpt(tmp_path, inv, seed)
    res = sllm.load_files(idx2, str(tmp_path), {0: 0}, sllm.LoadConfig())
    check(res, inv, payloads2, lay2, [0])


# ---- GPUDirect Storage variant (SLLM_MODE_GDS: cuFileRead straight into HBM) ----------
# cuFileDriverOpen never returns on the VMs this build runs on (no nvidia-fs; the
# compatibility mode hangs probing the PCI topology: profiles/r01/gds_probe.log), so the
# mode is opt-in (SLLM_ENABLE_GDS=1) and the read tests run only where it is set.

GDS = os.environ.get("SLLM_ENABLE_GDS") == "1"


def test_gds_is_opt_in_and_file_only(tmp_path, monkeypatch):
    inv, seed = models.model_inventory("toy")
    idx, lay, parts, payloads = write_ckpt(tmp_path, inv, seed)
    monkeypatch.delenv("SLLM_ENABLE_GDS", raising=False)
    with pytest.raises(sllm.SllmError) as ex:   # fails fast, never touches cuFile
        sllm.load_files(idx, str(tmp_path), {0: 0}, sllm.LoadConfig(mode="gds"))
    assert ex.value.status == 1 and "SLLM_ENABLE_GDS" in ex.value.message
    from paper_2401_14351_b200 import workloads
    idx2, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    monkeypatch.setenv("SLLM_ENABLE_GDS", "1")
    with pytest.raises(sllm.SllmError) as ex:   # GDS reads files: not a pinned-source mode
        sllm.load(idx2, bufs, {0: 0}, sllm.LoadConfig(mode="gds"))
    assert ex.value.status == 1


@pytest.mark.skipif(not GDS, reason="SLLM_ENABLE_GDS=1 not set (needs a host where cuFile opens)")
@pytest.mark.parametrize("io_threads", [1, 4])
def test_gds_toy(tmp_path, io_threads):
    inv, seed = models.model_inventory("toy")
    idx, lay, parts, payloads = write_ckpt(tmp_path, inv, seed)
    res = sllm.load_files(idx, str(tmp_path), {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20, mode="gds"),
                          io_threads=io_threads)
    assert res.report["storage_bytes"] == 13_594_624 and res.report["transferred_bytes"] == 13_594_624
    assert res.report["mode"] == 5
    check(res, inv, payloads, lay, [0])


@pytest.mark.skipif(not GDS, reason="SLLM_ENABLE_GDS=1 not set (needs a host where cuFile opens)")
def test_gds_two_partitions_many_windows(tmp_path):
    """~1.1 GB over two partitions, 64 MiB windows, A = 16 (file lengths not 4 KiB multiples)."""
    inv = models.llama2(1024, 36, 4096, 256, vocab=8192, tp=2)
    inv = [models.TensorSpec(t.name, t.device, t.dtype, t.shape) for t in inv] + \
          [models.TensorSpec("odd@0", 0, "u8", (33,)), models.TensorSpec("odd@1", 1, "f16", ())]
    idx, lay, parts, payloads = write_ckpt(tmp_path, inv, 78, A=16, B=1 << 20)
    res = sllm.load_files(idx, str(tmp_path), {0: 0, 1: 0}, sllm.LoadConfig(chunk_bytes=4 << 20, mode="gds"),
                          io_threads=3)
    check(res, inv, payloads, lay, [0, 1])


@pytest.mark.skipif(not GDS, reason="SLLM_ENABLE_GDS=1 not set (needs a host where cuFile opens)")
def test_gds_corruption_and_errors(tmp_path):
    inv, seed = models.model_inventory("toy")
    idx, lay, parts, payloads = write_ckpt(tmp_path, inv, seed)
    path = tmp_path / "part_0.bin"
    data = bytearray(open(path, "rb").read())
    pos = 7 * (1 << 20) + 999
    data[pos] ^= 0x01
    open(path, "wb").write(bytes(data))
    with pytest.raises(sllm.SllmError) as ex:
        sllm.load_files(idx, str(tmp_path), {0: 0}, sllm.LoadConfig(chunk_bytes=2 << 20, mode="gds"))
    assert ex.value.status == 9 and "block 7" in ex.value.message
    os.remove(path)
    with pytest.raises(sllm.SllmError) as ex:
        sllm.load_files(idx, str(tmp_path), {0: 0}, sllm.LoadConfig(mode="gds"))
    assert ex.value.status == 6
