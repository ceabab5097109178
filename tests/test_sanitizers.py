"""Host code under AddressSanitizer + UBSan (SURVEY §5 "ASan/UBSan on host code"): the
library's host sources are rebuilt with -fsanitize=address,undefined (kernels unchanged,
build/sllm_asan/) and driven by tests/c/host_fuzz.c -- random checkpoints through plan /
convert_into / seal / serialize, every index truncation and thousands of byte flips through
the parser, lookups, addresses, conversion errors, files and the pinned-cache policy.
Any sanitizer report (including leaks) fails the test.  No GPU needed."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_host_code_clean_under_asan_ubsan(tmp_path):
    from paper_2401_14351_b200 import build
    lib = build.build(sanitize=True)
    exe = str(tmp_path / "host_fuzz")
    r = subprocess.run(["gcc", "-std=c99", "-O1", "-g", "-fsanitize=address,undefined", "-fno-omit-frame-pointer",
                        "-o", exe, os.path.join(ROOT, "tests", "c", "host_fuzz.c"), f"-I{ROOT}/include", lib,
                        f"-Wl,-rpath,{os.path.dirname(lib)}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    env = {**os.environ, "ASAN_OPTIONS": "detect_leaks=1:abort_on_error=0",
           "UBSAN_OPTIONS": "halt_on_error=1:print_stacktrace=1"}
    env.pop("LD_PRELOAD", None)
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    assert "host fuzz ok" in r.stdout
    assert "runtime error" not in r.stderr and "AddressSanitizer" not in r.stderr, r.stderr[-4000:]
