import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the CUDA path through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running")


def _ensure_oracle():
    lib = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
    runner = os.path.join(ROOT, "oracle", "_build", "kat_runner")
    if not (os.path.exists(lib) and os.path.exists(runner)):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-j4"], check=True,
                       stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def oracle():
    _ensure_oracle()
    from oracle_py import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def product_lib():
    from paper_2509_17340_b200 import _abi

    return _abi.load()
