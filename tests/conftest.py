import json
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; parity through the C-ABI")
    config.addinivalue_line("markers", "slow: full-size (BASELINE) parity run")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(HERE, "golden", "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def orc():
    from oracle_bind import oracle

    return oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_bind import reference

    r = reference()
    if r is None:
        pytest.skip("oracle/_ref (compiled reference) not built")
    return r


@pytest.fixture(scope="session")
def mb():
    import paper_2008_08654_b200 as mb

    return mb


@pytest.fixture(scope="session")
def cuda(mb):
    """The GPU tests never fall back: a missing device is a hard failure."""
    import torch

    assert torch.cuda.is_available(), "GPU test run without a visible CUDA device"
    assert mb.device_count() >= 1, "no sm_100 device visible to libmersenne_b200.so"
    return torch
