"""The ctypes mirrors of the C ABI's structs (paper_2401_14351_b200/_abi.py) have the same
size and field offsets as the declarations in include/sllm.h: a small C program generated
here prints sizeof / offsetof for every field as the C compiler lays them out, and each is
compared with ctypes' layout.  CPU only (gcc, no CUDA runtime calls)."""
import ctypes as C
import json
import os
import subprocess

import pytest

from paper_2401_14351_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PAIRS = [("sllm_src_tensor", _abi.SrcTensor), ("sllm_index_info", _abi.IndexInfo),
         ("sllm_tensor_info", _abi.TensorInfo), ("sllm_load_config", _abi.LoadConfig),
         ("sllm_load_report", _abi.LoadReport), ("sllm_tensor_handle", _abi.TensorHandle),
         ("sllm_ipc_region", _abi.IpcRegion), ("sllm_cache_stats", _abi.CacheStats)]


def c_layout(tmp_path):
    lines = ["#include <stddef.h>", "#include <stdio.h>", '#include "sllm.h"', "int main(void) {", 'printf("{");']
    for i, (cname, cls) in enumerate(PAIRS):
        sep = "," if i else ""
        lines.append(f'printf("{sep}\\"{cname}\\": {{\\"size\\": %zu", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'printf(", \\"{f}\\": %zu", offsetof({cname}, {f}));')
        lines.append('printf("}");')
    lines += ['printf("}\\n");', "return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = str(tmp_path / "layout")
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
                        "-o", exe, str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return json.loads(subprocess.run([exe], capture_output=True, text=True, check=True).stdout)


@pytest.mark.parametrize("cname,cls", PAIRS, ids=[p[0] for p in PAIRS])
def test_ctypes_matches_c_layout(tmp_path, cname, cls):
    lay = c_layout(tmp_path)[cname]
    assert C.sizeof(cls) == lay["size"], (cname, C.sizeof(cls), lay["size"])
    for f, _ in cls._fields_:
        assert getattr(cls, f).offset == lay[f], (cname, f, getattr(cls, f).offset, lay[f])
