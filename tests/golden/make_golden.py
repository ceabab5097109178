"""Writes the golden fixtures under tests/golden/ by calling ONLY oracle/ (never the
CUDA path).  Run: python tests/golden/make_golden.py"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import index, layout  # noqa: E402


def spec_s49():
    # SPEC.md S:49 worked example: two tensors on device 0, 10 B and 6 B, align 4096.
    tensors = [("a", 0, "u8", (10,), b"\x01" * 10), ("b", 0, "u8", (6,), b"\x02" * 6)]
    lay, _ = layout.convert(tensors, 4096, 4096, "spec-s49")
    with open(os.path.join(HERE, "spec_s49_index.hex"), "w") as f:
        f.write(index.write(lay).hex() + "\n")


if __name__ == "__main__":
    spec_s49()
