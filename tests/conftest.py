import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU; run with -m gpu")


@pytest.fixture(scope="session")
def port():
    import oracle_lib
    return oracle_lib.port()


@pytest.fixture(scope="session")
def ref():
    import oracle_lib
    return oracle_lib.ref()
