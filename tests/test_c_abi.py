"""The C ABI used from plain C (tests/c/abi_load.c): only include/sllm.h + the CUDA
runtime, no Python and no torch types.  Compiling it is a CPU check that the header is
self-contained C; running it (GPU) loads a two-partition checkpoint in CE and zero-copy
mode and checks every device byte, every tensor handle and the fault report."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c", "abi_load.c")
LIBDIR = os.path.join(ROOT, "paper_2401_14351_b200")
CUDA = "/usr/local/cuda"


def build(tmp_path):
    exe = str(tmp_path / "abi_load")
    cmd = ["gcc", "-std=c99", "-O1", "-Wall", "-Werror", "-o", exe, SRC, f"-I{ROOT}/include", f"-I{CUDA}/include",
           os.path.join(LIBDIR, "libsllm.so"), f"-Wl,-rpath,{LIBDIR}", f"-L{CUDA}/lib64", "-lcudart",
           f"-Wl,-rpath,{CUDA}/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_client_compiles(tmp_path):
    build(tmp_path)


@pytest.mark.gpu
def test_c_client_loads_on_gpu(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    exe = build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c-abi ok" in r.stdout
