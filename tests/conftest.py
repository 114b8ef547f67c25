"""Shared fixtures.  `-m gpu` tests need a B200 and call the engine through the
C-ABI; everything else runs on CPU (oracle vs golden vectors, host logic,
library exports, gloo multi-process sharding)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_cases.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    from oracle.oracle import load_golden
    return load_golden(GOLDEN)


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import COracle
    return COracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import RefOracle
    if not RefOracle.available():
        pytest.skip("oracle/_ref not built (reference tree absent)")
    return RefOracle()


@pytest.fixture(scope="session")
def abq():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_2408_08554_b200 as abq
    return abq


def seeded_codes(seed, rows, cols, bits):
    return np.random.default_rng(seed).integers(0, 1 << bits, size=(rows, cols), dtype=np.uint8)


def family(golden, prefix):
    """indices present for a numbered case family, e.g. 'gemm23'"""
    ids = sorted({int(k.split("/")[1]) for k in golden if k.startswith(prefix + "/")})
    return ids
