"""Per-kernel counts of the Blackwell tile-movement / synchronisation instructions in the built
libsllm.so (cuobjdump -sass of its sm_100a cubin).  Runs here, no GPU.

    python tools/sass_excerpt.py > profiles/r02/sass_excerpt.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2401_14351_b200", "libsllm.so")
KEEP = re.compile(r"^(UBLKCP|SYNCS|LDS\.128|SHFL\.BFLY|STG\.E|LDG\.E|ATOMG|REDG|MEMBAR|NANOSLEEP|CS2R)")

HEADER = """# cuobjdump -sass paper_2401_14351_b200/libsllm.so (sm_100a cubin), tools/sass_excerpt.py
# per kernel: count of the Blackwell-native tile-movement / sync instructions
#   UBLKCP.S.G  = cp.async.bulk global->shared (TMA 1-D bulk load; host-mapped or HBM source)
#   UBLKCP.G.S  = cp.async.bulk shared->global (TMA bulk store, engine tma_store)
#   SYNCS.*     = mbarrier init / arrive(.expect_tx) / try_wait.parity (the 12-stage ring)
#   LDS.128     = consumers' 16-byte shared-memory reads; SHFL.BFLY = checksum warp reduction
#   STG.E.NA.128 = 16-byte stores (st.global.L1::no_allocate) into tensors / peer replicas
#   STG.E.128   = the NVLS multicast store (multimem.st.global.v4.f32 on the multicast mapping)
#   ATOMG.E.ADD.64 = ticket draws (dynamic units), split-block combines; ATOMG.E.MIN = failing block;
#   REDG.E.MAX.64 = profile-3 in-kernel span marks
#   CS2R ... SR_GLOBALTIMERLO = %globaltimer (mbarrier watchdog, profile-3 in-kernel spans)
"""


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if cur and m and KEEP.match(m.group(1)):
            kernels[cur][m.group(1)] += 1
    names = subprocess.run(["c++filt"], input="\n".join(kernels), capture_output=True, text=True).stdout.split("\n")
    print(HEADER)
    for (k, c), n in zip(kernels.items(), names):
        if c:
            print(n or k)
            print("    " + str(dict(sorted(c.items()))))


if __name__ == "__main__":
    main()
