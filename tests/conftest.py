import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


_built = False


def _build_oracle():
    global _built
    if not _built:
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
        _built = True


@pytest.fixture(scope="session", autouse=True)
def oracle_built():
    _build_oracle()
