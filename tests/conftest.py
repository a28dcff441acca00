"""Shared fixtures.  GPU tests are marked @pytest.mark.gpu and are selected only
on a B200 box (`pytest -m gpu`); there they FAIL (not skip) if the native
library or the device is missing -- no silent fallback path exists."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def orc():
    from oracle_py import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_py import REF_SO, Reference
    if not os.path.exists(REF_SO):
        pytest.skip("reference CPU build (oracle/_ref) not present")
    return Reference()


@pytest.fixture(scope="session")
def cct():
    import paper_1504_04343_b200 as cct
    cct.lib()
    return cct


@pytest.fixture(scope="session")
def dev():
    import torch
    assert torch.cuda.is_available(), "GPU test selected but no CUDA device"
    major, minor = torch.cuda.get_device_capability(0)
    assert major == 10, f"expected an sm_100 (B200) device, got sm_{major}{minor}"
    return torch.device("cuda:0")
