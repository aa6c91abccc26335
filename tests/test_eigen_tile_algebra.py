"""CPU check of the algebra behind the sweep kernels' 7-array Miehe tile (csrc/pff_sweep.cu,
k_refresh_tiled / k_sweep_q2): the eigen-frame form with the strain regime in two sign bits
reproduces the reference's split tangent and coupling (src/_kernels.py:26-123, restated here in
numpy the way csrc/pff_common.cuh restates it) for random strains, directions and degradations,
in every regime.  Host logic only: no GPU, no library call."""

import numpy as np
import pytest

LAM, MU = 121.15e3, 80.77e3


def eig2(a11, a22, a12):
    m, dh = 0.5 * (a11 + a22), 0.5 * (a11 - a22)
    r = np.sqrt(dh * dh + a12 * a12)
    left = dh <= 0.0
    vx = np.where(left, a12, r + dh)
    vy = np.where(left, r - dh, a12)
    nrm = np.sqrt(vx * vx + vy * vy)
    ok = nrm > 0.0
    safe = np.where(ok, nrm, 1.0)
    return m + r, m - r, np.where(ok, vx / safe, 1.0), np.where(ok, vy / safe, 0.0)


def reference_tangent(g, e11, e22, e12, d11, d22, d12):
    """g dsigma+ + dsigma- and sigma+ : de, src/_kernels.py:50-74,102-123."""
    ev1, ev2, c, s = eig2(e11, e22, e12)
    scale = np.maximum(np.sqrt(e11 * e11 + e22 * e22 + 2.0 * e12 * e12), 1.0)
    t0, t1 = d11 * c + d12 * s, d12 * c + d22 * s
    dl1 = c * t0 + s * t1
    dl2 = s * s * d11 - 2.0 * s * c * d12 + c * c * d22
    dl1p, dl2p = np.where(ev1 >= 0.0, dl1, 0.0), np.where(ev2 >= 0.0, dl2, 0.0)
    l1p, l2p = np.maximum(ev1, 0.0), np.maximum(ev2, 0.0)
    gap = ev1 - ev2
    gap_ok = gap > 1e-12 * scale
    alpha = np.where(gap_ok, (c * t1 - s * t0) / np.where(gap_ok, gap, 1.0), 0.0)
    rot = alpha * (l1p - l2p)
    o11 = dl1p * c * c + dl2p * s * s - 2.0 * rot * s * c
    o22 = dl1p * s * s + dl2p * c * c + 2.0 * rot * s * c
    o12 = (dl1p - dl2p) * c * s + rot * (c * c - s * s)
    tre, trde = e11 + e22, d11 + d22
    tt = np.where(tre < 0.0, 0.0, trde)
    dp11, dp22, dp12 = LAM * tt + 2 * MU * o11, LAM * tt + 2 * MU * o22, 2 * MU * o12
    f11, f22, f12 = LAM * trde + 2 * MU * d11, LAM * trde + 2 * MU * d22, 2 * MU * d12
    trp = np.maximum(tre, 0.0)
    sp11 = LAM * trp + 2 * MU * (l1p * c * c + l2p * s * s)
    sp22 = LAM * trp + 2 * MU * (l1p * s * s + l2p * c * c)
    sp12 = 2 * MU * (l1p - l2p) * c * s
    spde = sp11 * d11 + sp22 * d22 + 2.0 * sp12 * d12
    return g * dp11 + (f11 - dp11), g * dp22 + (f22 - dp22), g * dp12 + (f12 - dp12), spde


def encode_tile(g, e11, e22, e12):
    """k_refresh_tiled<true>: +-g, +-gamma, cos / sin of twice the eigen-angle, the two
    eigen-frame coupling coefficients (unit weight, dg = 1)."""
    ev1, ev2, c, s = eig2(e11, e22, e12)
    scale = np.maximum(np.sqrt(e11 * e11 + e22 * e22 + 2.0 * e12 * e12), 1.0)
    gap_ok = (ev1 - ev2) > 1e-12 * scale
    l1p, l2p = np.maximum(ev1, 0.0), np.maximum(ev2, 0.0)
    tre = e11 + e22
    trp = np.maximum(tre, 0.0)
    beta = np.where(gap_ok, (l1p - l2p) / np.where(gap_ok, ev1 - ev2, 1.0), 0.0)
    gam = g * beta + (1.0 - beta)
    htr, h1, h2 = ~(tre < 0.0), ev1 >= 0.0, ev2 >= 0.0
    bb = np.where(htr, h2, h1)
    return (np.where(htr, g, -g), np.where(bb, gam, -gam), c * c - s * s, 2.0 * c * s,
            0.5 * (LAM * trp + 2 * MU * l1p), 0.5 * (LAM * trp + 2 * MU * l2p))


def apply_tile(tile, d11, d22, d12):
    """The q-point physics of k_sweep_q2<MIEHE> (unit weight)."""
    gs, ms, c2, s2, q1h, q2h = tile
    D12 = 2.0 * d12
    pd, qd = d11 + d22, d11 - d22
    u2 = c2 * qd + s2 * D12
    v2 = c2 * D12 - s2 * qd
    e1, e2 = pd + u2, pd - u2
    ha, hb = ~np.signbit(gs), ~np.signbit(ms)
    g, gam = np.abs(gs), np.abs(ms)
    ca, c1, cb = np.where(ha, g, 1.0), np.where(ha | hb, g, 1.0), np.where(ha & hb, g, 1.0)
    at = (0.5 * LAM * ca) * pd
    hs1 = (0.5 * MU * c1) * e1 + at
    hs2 = (0.5 * MU * cb) * e2 + at
    s3 = (MU * gam) * v2
    hp, hd = hs1 + hs2, hs1 - hs2
    t = c2 * hd - s2 * s3
    return hp + t, hp - t, s2 * hd + c2 * s3, q1h * e1 + q2h * e2


def _check(g, e, d, tol=2e-13):
    want = reference_tangent(g, *e, *d)
    got = apply_tile(encode_tile(g, *e), *d)
    dn = np.sqrt(d[0] ** 2 + d[1] ** 2 + 2 * d[2] ** 2)
    en = np.sqrt(e[0] ** 2 + e[1] ** 2 + 2 * e[2] ** 2)
    sc_s = (LAM + 2 * MU) * dn + 1e-300
    sc_c = (LAM + 2 * MU) * en * dn + 1e-300
    for k in range(3):
        assert np.max(np.abs(got[k] - want[k]) / sc_s) <= tol, k
    assert np.max(np.abs(got[3] - want[3]) / sc_c) <= tol


def test_random_states_all_regimes():
    rng = np.random.default_rng(0)
    n = 200_000
    e = rng.uniform(-1e-3, 1e-3, (3, n))
    d = rng.uniform(-1.0, 1.0, (3, n))
    g = rng.uniform(1e-10, 1.0, n)
    ev1, ev2, _, _ = eig2(*e)
    tre = e[0] + e[1]
    # all four regimes of (H_tr, H_1, H_2) are present in the sample
    for cond in ((ev2 >= 0), (ev1 < 0), (ev1 >= 0) & (ev2 < 0) & (tre >= 0),
                 (ev1 >= 0) & (ev2 < 0) & (tre < 0)):
        assert cond.sum() > 1000
    _check(g, e, d)


@pytest.mark.parametrize("e", [(0.0, 0.0, 0.0), (-1e-3, -1e-3, 0.0), (1e-3, 1e-3 * (1 + 1e-6), 0.0),
                               (1e-3, -3e-4, 0.0), (3e-4, -1e-3, 0.0), (1e-5, 0.0, 1e-3),
                               (0.0, -1e-5, 5e-4), (-2e-3, -1e-3, 4e-4), (2e-3, 1e-3, 4e-4)])
def test_single_regime_states(e):
    rng = np.random.default_rng(1)
    n = 1000
    d = rng.uniform(-1.0, 1.0, (3, n))
    g = rng.uniform(1e-10, 1.0, n)
    ee = [np.full(n, x) for x in e]
    _check(g, ee, d)


def test_sign_bits_survive_zero_degradation():
    """g = 0 (kappa = 0, phi~ = 0): the regime still decodes from +-0."""
    rng = np.random.default_rng(2)
    n = 5000
    e = rng.uniform(-1e-3, 1e-3, (3, n))
    d = rng.uniform(-1.0, 1.0, (3, n))
    _check(np.zeros(n), e, d)
