"""Builds libsllm.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_2401_14351_b200.build [--force]

Every source under csrc/ is compiled by nvcc (``-gencode arch=compute_100a,code=sm_100a
-lineinfo``), the CUDA runtime is linked statically and NCCL is dlopen'ed at run time,
so the library loads on machines without a GPU or NCCL.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsllm.so")
BUILD = os.path.join(ROOT, "build", "sllm")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _nccl_include() -> str:
    try:
        import nvidia.nccl  # noqa: F401  (header only; the library is dlopen'ed)
        base = os.path.dirname(nvidia.nccl.__file__) if getattr(nvidia.nccl, "__file__", None) \
            else list(nvidia.nccl.__path__)[0]
        inc = os.path.join(base, "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    except Exception:
        pass
    for c in glob.glob(os.path.join(sys.prefix, "lib", "python*", "site-packages", "nvidia", "nccl", "include")):
        return c
    raise RuntimeError("nccl.h not found (nvidia-nccl wheel)")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return glob.glob(os.path.join(CSRC, "*.h*")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "sllm.h")]


# (nvcc splits -Xcompiler values on commas: one sanitizer per flag)
SAN_FLAGS = "-fsanitize=address,-fsanitize=undefined,-fno-omit-frame-pointer,-fno-sanitize-recover=all"


def build(force: bool = False, verbose: bool = False, sanitize: bool = False, variant: str = "",
          defines=()) -> str:
    """sanitize=True: an AddressSanitizer + UBSan build of the host code (kernels unchanged)
    at build/sllm_asan/libsllm_asan.so, for tests/test_sanitizers.py -- never the product.
    variant="name", defines=[...]: an A/B measurement build at build/ab/<name>/libsllm.so
    (loaded with SLLM_LIB_PATH) -- never the product."""
    srcs = sources()
    out = os.path.join(ROOT, "build", "sllm_asan", "libsllm_asan.so") if sanitize else OUT
    bdir = os.path.join(ROOT, "build", "sllm_asan") if sanitize else BUILD
    if variant:
        bdir = os.path.join(ROOT, "build", "ab", variant)
        out = os.path.join(bdir, "libsllm.so")
    newest = max(os.path.getmtime(p) for p in srcs + _headers() + [__file__])
    if not force and os.path.exists(out) and os.path.getmtime(out) >= newest:
        return out
    os.makedirs(bdir, exist_ok=True)
    nvcc = _nvcc()
    host = "-fPIC,-O3,-fvisibility=hidden" if not sanitize else "-fPIC,-O1,-g,-fvisibility=hidden," + SAN_FLAGS
    extra = os.environ.get("SLLM_NVCC_DEFINES", "").split() + list(defines)  # A/B builds only, e.g. "-DSLLM_STAGE_KIB=32"
    common = ["-O3", "-std=c++17", "-lineinfo", *ARCH, *extra, "-Xcompiler", host,
              "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", _nccl_include()]

    def compile_one(src):
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        cmd = [nvcc, *common, "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout + r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = f"{out}.tmp{os.getpid()}"
    cmd = [nvcc, "-shared", *ARCH, "-cudart", "static", "-o", tmp, *objs, "-ldl", "-lpthread", "-lrt",
           "-Xlinker", "--exclude-libs,ALL"] + (["-Xcompiler", SAN_FLAGS] if sanitize else [])
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
