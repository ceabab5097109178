"""The C payload generator equals the NumPy definition (O10) byte for byte."""
import ctypes

import numpy as np

from synth import payload


def test_splitmix64_known_values():
    # splitmix64 reference outputs for seed 0 (state increments by the golden gamma):
    # the first outputs of the canonical SplitMix64 generator seeded with 0.
    assert int(payload.splitmix64(np.uint64(0))) == 0xE220A8397B1DCDAF
    assert int(payload.splitmix64(np.uint64(0x9E3779B97F4A7C15))) == 0x6E789E6AA1B965F4


def test_c_matches_numpy(csynth):
    sizes = [1, 7, 8, 9, 4095, 4 << 20, (4 << 20) + 13, 10_000_003]
    bufs = [np.zeros(s, dtype=np.uint8) for s in sizes]
    es = list(range(len(sizes)))
    csynth.payload_into([b.ctypes.data for b in bufs], sizes, 1234, es, threads=4)
    for b, s, e in zip(bufs, sizes, es):
        assert np.array_equal(b, payload.payload_bytes(1234, e, s))
