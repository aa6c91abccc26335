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


def sketch(v, n, seed=77, samples=4096):
    """Size-independent summary of a long vector for production-size pins
    (tests/golden/make_golden.py --production): per-block L2 norms, four seeded
    Gaussian projections per block and `samples` seeded entries per block."""
    v = np.asarray(v, dtype=float)
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(n, size=min(samples, n), replace=False))
    out = {"norms": [], "proj": [], "idx": idx, "vals": []}
    for k in range(v.size // n):
        b = v[k * n:(k + 1) * n]
        out["norms"].append(np.linalg.norm(b))
        g = np.random.default_rng(seed + 1 + k)
        out["proj"].append([float(g.standard_normal(n) @ b) for _ in range(4)])
        out["vals"].append(b[idx])
    return {k: np.asarray(x) for k, x in out.items()}


def sketch_rel(got, want):
    """Largest per-block relative deviation between two sketches: norms,
    projections (relative to the block norm) and the sampled entries (relative
    L2 over the sample)."""
    worst = 0.0
    for k in range(len(want["norms"])):
        nk = want["norms"][k]
        worst = max(worst, abs(got["norms"][k] - nk) / nk,
                    float(np.max(np.abs(np.asarray(got["proj"][k]) - want["proj"][k]))) / nk,
                    rel_l2(got["vals"][k], want["vals"][k]))
    return worst


@pytest.fixture(scope="session")
def golden():
    return load_golden


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
