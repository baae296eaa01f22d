import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built librkc.so")


@pytest.fixture(scope="session", autouse=True)
def _built_cpu_libs():
    from oracle import oracle
    from paper_2605_24259_b200 import gen
    oracle.build()
    gen.build()
    yield
