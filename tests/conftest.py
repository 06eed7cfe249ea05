import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) -- run with -m gpu")


@pytest.fixture(scope="session")
def ctx():
    from paper_2306_17801_b200 import rvk
    c = rvk.Ctx()
    yield c
    c.close()
