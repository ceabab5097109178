import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def csynth():
    from synth import payload
    payload.build_csynth()
    return payload


@pytest.fixture(scope="session", autouse=True)
def _built_libraries():
    """Build libsynth.so (input generator) and libsllm.so (the product) in-tree."""
    from synth import payload
    payload.build_csynth()
    from paper_2401_14351_b200 import build
    build.build()
