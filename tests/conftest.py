"""Shared fixtures.  `-m gpu` tests need a B200 (sm_100a) and the built
C-ABI library; everything else runs on CPU."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU check")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(os.path.join(GOLDEN, "golden.npz")))


@pytest.fixture(scope="session")
def table_text():
    with open(os.path.join(GOLDEN, "gelu_table_default_v1.txt")) as f:
        return f.read()


@pytest.fixture(scope="session")
def port():
    import oracle
    oracle.build()
    return oracle.Port()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.have_ref():
        pytest.skip("reference library oracle/_ref not built (needs /root/reference)")
    return oracle.Ref()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@pytest.fixture(scope="session")
def tops(cuda):
    """The product ops module, with the CUDA library loaded (fails loudly if
    it was not built: there is no fallback)."""
    from paper_2210_10246_b200 import ops
    from paper_2210_10246_b200._capi import lib
    lib()
    return ops
