"""Shared fixtures.  `-m gpu` tests need a B200 (run through gpurun); the rest
run on CPU.  The oracle (oracle/) is the parity checker only."""
import gzip
import json
import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


def load_golden(name):
    path = os.path.join(GOLDEN, name)
    if name.endswith(".gz"):
        with gzip.open(path, "rt") as f:
            return json.load(f)
    with open(path) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def engine():
    import paper_2605_28400_b200 as ta
    ta.lib()
    return ta


@pytest.fixture(scope="session")
def gpu_engine():
    import paper_2605_28400_b200 as ta
    if ta.device_count() < 1:
        pytest.fail("no CUDA device visible: -m gpu tests must run on the B200 box")
    return ta
