import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer-running CPU check")


@pytest.fixture(scope="session")
def oracle():
    import oracle_ctypes

    oracle_ctypes.build_oracle()
    return oracle_ctypes


@pytest.fixture(scope="session")
def stmg():
    import paper_2502_09159_b200 as m

    m.load_library()
    return m


@pytest.fixture(scope="session")
def ctx(stmg):
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    return stmg.Context(0)
