"""Cross-process handles: the loading process exports
its partition bases with CUDA IPC; a separate inference process maps them, builds every
tensor as base + offset from the index and finds the oracle's bytes there."""
import os
import pickle
import subprocess
import sys
import textwrap

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

import paper_2401_14351_b200 as sllm  # noqa: E402
from paper_2401_14351_b200 import ipc, workloads  # noqa: E402
from synth import models  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = textwrap.dedent("""
    import pickle, sys
    sys.path.insert(0, {root!r})
    import numpy as np, torch
    from paper_2401_14351_b200 import ipc
    from synth import models, payload
    exp = pickle.load(open({path!r}, "rb"))
    imp = ipc.import_tensors(exp)
    inv, seed = models.model_inventory("toy")
    bad = 0
    for e, t in enumerate(inv):
        got = imp.tensors[t.name].reshape(-1).view(torch.uint8).cpu().numpy()
        bad += not np.array_equal(got, payload.payload_bytes(seed, e, t.nbytes))
    # the importer may also write (shared memory): mark one byte for the parent to see
    imp.bases[0][-1] = 0x7E
    torch.cuda.synchronize()
    imp.close()
    print("child-ok" if bad == 0 else f"child-bad {{bad}}")
""")


def test_ipc_export_import_across_processes(tmp_path):
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20)
    res = sllm.load(idx, bufs, {0: 0}, sllm.LoadConfig(mode="ce"))
    exp = ipc.export(res)
    assert set(exp["regions"]) == {0} and len(exp["regions"][0]) == 88
    path = tmp_path / "exported.pkl"
    pickle.dump(exp, open(path, "wb"))
    code = CHILD.format(root=ROOT, path=str(path))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert "child-ok" in out.stdout, out.stdout + out.stderr
    base = res._keep[3][0]
    assert int(base[-1].item()) == 0x7E       # the child wrote through the mapping


def test_ipc_rejects_host_memory_and_unknown_pointers():
    import ctypes as C
    from paper_2401_14351_b200 import _abi
    r = _abi.IpcRegion()
    host = np.zeros(16, np.uint8)
    with pytest.raises(sllm.SllmError):
        _abi.check(sllm.lib().sllm_ipc_export(C.c_void_p(host.ctypes.data), 16, C.byref(r)))
    with pytest.raises(sllm.SllmError):
        _abi.check(sllm.lib().sllm_ipc_close(C.c_void_p(0x1000)))
