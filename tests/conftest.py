import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def rel_l2(got, want):
    got, want = np.asarray(got), np.asarray(want)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))


def block_rel(got, want, n):
    """Per-block relative L2 (u_x, u_y, phi): the phi block is ~1e3x smaller
    than the u blocks, so a whole-vector norm would hide it."""
    return [rel_l2(got[k * n:(k + 1) * n], want[k * n:(k + 1) * n]) for k in range(len(got) // n)]


@pytest.fixture(scope="session")
def golden():
    return load_golden


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
