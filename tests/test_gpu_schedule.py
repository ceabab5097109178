"""GPU parity of the ring kernel's work distributions: dynamic units (tickets)
with the fine tail on every launch (the default) or on unbalanced launches only
(SLLM_FINE_TAIL=1), dynamic units without the fine tail (SLLM_FINE_TAIL=0),
the static schedule (SLLM_STATIC_UNITS=1) and both knobs together.  The knobs are read once
per process, so each combination runs in a child process that

  * checksums a ragged device buffer of ~600 MiB (>= 2 waves of 1 MiB blocks, so the fine
    tail is used; last block 4,112 B) with the standalone K4 and compares every block with
    the oracle's Fletcher-64 table of the same bytes;
  * loads a ~0.53 GB LLaMA-shaped checkpoint in all four modes (CE spans, ZC windows,
    SCATTER_CE staging windows, SCATTER_ZC) and compares every tensor byte with its payload
    and every block checksum with the oracle's layout (oracle/layout.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
import paper_2401_14351_b200 as sllm
from paper_2401_14351_b200 import workloads
from oracle import fletcher as ofl, layout as olayout
from synth import models, payload

# standalone K4 on a ragged ~600 MiB buffer
n = (600 << 20) + 4112
host = np.random.default_rng(5).integers(0, 2**32, n // 4, dtype=np.uint32).view(np.uint8)
src = torch.from_numpy(host).cuda()
out = torch.empty(-(-n // (1 << 20)), dtype=torch.int64, device="cuda")
sllm.block_checksums_device(src.data_ptr(), n, 1 << 20, out.data_ptr(), 0, torch.cuda.current_stream())
torch.cuda.synchronize()
want = ofl.block_checksums(host, 1 << 20)
assert out.cpu().numpy().view(np.uint64).tolist() == list(want), "K4 checksums"

# loads in all four modes
inv, seed = models.llama2(1024, 12, 4096, 1024, vocab=32000), 9
payloads = [payload.payload_bytes(seed, e, t.nbytes) for e, t in enumerate(inv)]
lay, oparts = olayout.convert([(t.name, t.device, t.dtype, t.shape, p) for t, p in zip(inv, payloads)], 4096, 1 << 20)
idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
for mode in ("ce", "zerocopy", "scatter_ce", "scatter_zc"):
    for chunk in (1 << 20, 64 << 20):
        res = sllm.load(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=chunk, mode=mode))
        assert res.report["bad_partition"] == -1, mode
        assert res.block_checksums(0).tolist() == lay.checksums[0], (mode, chunk)
        for e, t in enumerate(inv):
            b = res.tensors[t.name].contiguous().view(torch.uint8).reshape(-1)
            assert np.array_equal(b.cpu().numpy(), payloads[e]), (mode, chunk, t.name)
        del res
print("schedule-child ok")
"""


@pytest.mark.parametrize("env", [{}, {"SLLM_FINE_TAIL": "1"}, {"SLLM_FINE_TAIL": "0"}, {"SLLM_STATIC_UNITS": "1"},
                                 {"SLLM_STATIC_UNITS": "1", "SLLM_FINE_TAIL": "0"}],
                         ids=["dynamic+fine", "dynamic+fine-unbalanced", "dynamic", "static+fine", "static"])
def test_work_distribution_parity(env):
    e = dict(os.environ)
    e.pop("SLLM_FINE_TAIL", None)
    e.pop("SLLM_STATIC_UNITS", None)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=e, cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "schedule-child ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
