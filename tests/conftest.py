import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libdare_b200.so")
    # (re)build the CUDA library and the CPU oracle when sources are newer
    from paper_2605_26325_b200 import build as cuda_build
    from oracle import oracle

    cuda_build.build()
    if os.environ.get("DARE_CHECKED") == "1":
        cuda_build.build(checked=True)
    oracle.build()


@pytest.fixture
def rng() -> np.random.Generator:
    return np.random.default_rng(20240809)


@pytest.fixture(scope="session")
def golden():
    from golden_io import Golden

    return Golden()
