"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``; everything
else runs on CPU (`pytest -m "not gpu"`)."""

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden", "reference_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def bf16_round(x):
    """fp32 -> bf16 (round to nearest even) -> fp32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def gaussian_qkv(s, d, seed, bf16=False):
    """tests/conftest.py:10-15 of the reference: seeds s, s+1, s+2."""
    from oracle import port

    q = port.seeded_gaussian(s, d, seed)
    k = port.seeded_gaussian(s, d, seed + 1)
    v = port.seeded_gaussian(s, d, seed + 2)
    if bf16:
        q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    return q, k, v


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN, allow_pickle=False)


@pytest.fixture
def rng():
    return np.random.Generator(np.random.PCG64(12345))


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
