import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def gaussian(n, d, seed):
    """core.gen_synthetic(..., 'gaussian') of the reference (core.py:209-233)."""
    return np.random.default_rng(seed).standard_normal((n, d)).astype(np.float32)


def lowrank(n, d, d_int, noise, seed):
    g = np.random.default_rng(seed)
    a = g.standard_normal((d_int, d)) / np.sqrt(d_int)
    x = g.standard_normal((n, d_int)) @ a + noise * g.standard_normal((n, d))
    return x.astype(np.float32)


def u8_rows(n, d, seed):
    """tests/golden/make_golden.py:u8_rows — BigANN-like u8 rows from a low-rank sample."""
    x = lowrank(n, d, 8, 0.05, seed)
    lo, hi = x.min(), x.max()
    return np.clip(np.rint((x - lo) / (hi - lo) * 255.0), 0, 255).astype(np.uint8)


def split(flat, lens):
    ends = np.cumsum(lens)
    return [flat[e - n:e] for e, n in zip(ends, lens)]


@pytest.fixture(scope="session")
def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
