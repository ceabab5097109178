"""A/B measurement builds of libsllm.so with compile-time knobs (never the product):

    python tools/build_variant.py stage32 -DSLLM_STAGE_KIB=32
    SLLM_LIB_PATH=build/ab/stage32/libsllm.so python tools/zc_ab.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    from paper_2401_14351_b200 import build
    print(build.build(force=True, variant=sys.argv[1], defines=sys.argv[2:]))
