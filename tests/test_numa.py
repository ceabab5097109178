"""NUMA placement of the DRAM tier: page placement read back
through the library (get_mempolicy) against the kernel's own account in /proc/self/numa_maps,
the GPU's node against sysfs, and the caller's CPU affinity untouched by the library's
node-bound worker / touch / converter threads."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2401_14351_b200 as sllm
from paper_2401_14351_b200 import _abi


def _numa_maps_nodes(addr: int):
    """Nodes holding pages of the mapping that contains addr, per /proc/self/numa_maps."""
    for line in open("/proc/self/numa_maps"):
        f = line.split()
        start = int(f[0], 16)
        # numa_maps gives only the start; find the mapping's end in /proc/self/maps
        for m in open("/proc/self/maps"):
            a, b = (int(x, 16) for x in m.split()[0].split("-"))
            if a == start and a <= addr < b:
                return {int(x[1:].split("=")[0]) for x in f if x.startswith("N") and "=" in x}
    return None


def _host_node(addr: int) -> int:
    out = C.c_int32()
    _abi.check(sllm.lib().sllm_host_numa_node(C.c_void_p(addr), C.byref(out)))
    return out.value


def test_page_node_matches_numa_maps():
    if not os.path.exists("/proc/self/numa_maps"):
        pytest.skip("no /proc/self/numa_maps")
    a = np.ones(64 << 20, np.uint8)     # touched: every page is resident
    node = _host_node(a.ctypes.data + (32 << 20))
    nodes = _numa_maps_nodes(a.ctypes.data)
    if node < 0 or not nodes:
        pytest.skip("get_mempolicy / numa_maps unavailable in this container")
    assert node in nodes


def test_bad_arguments():
    out = C.c_int32()
    assert sllm.lib().sllm_host_numa_node(None, C.byref(out)) == _abi.E_INVALID
    assert sllm.lib().sllm_gpu_numa_node(-1, C.byref(out)) == _abi.E_INVALID


@pytest.mark.gpu
def test_pinned_pages_on_the_gpus_node_and_caller_affinity_kept():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    from paper_2401_14351_b200 import workloads
    from synth import models
    g = C.c_int32()
    _abi.check(sllm.lib().sllm_gpu_numa_node(0, C.byref(g)))
    props = torch.cuda.get_device_properties(0)
    path = f"/sys/bus/pci/devices/{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0/numa_node"
    if os.path.exists(path):
        assert g.value == int(open(path).read().strip())
    before = os.sched_getaffinity(0)
    inv, seed = models.model_inventory("toy")
    idx, bufs = workloads.build_pinned(inv, seed, 4096, 1 << 20, gpu_of={0: 0})   # touch + converter threads
    buf = bufs[0]
    nodes = {_host_node(buf.ptr + k) for k in range(0, buf.nbytes, 1 << 20)}
    multi = len([d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")]) > 1
    if multi and g.value >= 0:
        assert nodes == {g.value}                    # mbind'ed to the GPU's node
    else:
        assert len(nodes) >= 1 and -1 not in nodes or nodes == {-1}
    res = sllm.load(idx, bufs, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20))      # node-bound worker
    res.wait()
    assert os.sched_getaffinity(0) == before         # the library never re-binds the caller


def test_worker_rebinds_across_nodes_fake_sysfs(tmp_path):
    """A pooled worker bound to one node for one job is re-bound to another node for the
    next, and unbound for an unknown node (numa.cpp against a fake two-node sysfs tree)."""
    import subprocess
    cpus = sorted(os.sched_getaffinity(0))
    if len(cpus) < 2:
        pytest.skip("needs two allowed CPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for n, c in enumerate(cpus[:2]):
        d = tmp_path / "devices" / "system" / "node" / f"node{n}"
        d.mkdir(parents=True)
        (d / "cpulist").write_text(f"{c}\n")
    exe = str(tmp_path / "numa_bind")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-o", exe, os.path.join(root, "tests", "c", "numa_bind.cpp"),
                        f"-I{root}/include", f"-I{cuda}/include", f"-L{cuda}/lib64", "-lcudart_static",
                        "-lpthread", "-ldl", "-lrt"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    r = subprocess.run([exe, str(cpus[0]), str(cpus[1])], capture_output=True, text=True, timeout=60,
                       env={**os.environ, "SLLM_SYSFS_ROOT": str(tmp_path)})
    assert r.returncode == 0 and "numa bind ok" in r.stdout, r.stdout + r.stderr
