import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (large N)")


@pytest.fixture(scope="session")
def hx():
    import paper_1911_00093_b200 as mod
    return mod


@pytest.fixture(scope="session")
def orc():
    from oracle import hmx_oracle
    return hmx_oracle
