"""CPU oracle for the matrix-free PFF hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker for the B200 product path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import it; the product package
``paper_2005_00331_b200`` never does, and it fails loudly when its CUDA
library is missing instead of falling back to anything here.

It restates the reference (fracturekit 0.1.0; ``src/`` below means
``/root/reference/pkg/src/fracturekit/``) in numpy + a small C library
(``pff_oracle.c``, built by the Makefile next to this file):

* shape data                    src/tensor_basis.py:19-81
* Q_p numbering, injection      src/mesh_hierarchy.py:156-189, 316-338
* linearisation state + cache   src/pff_operator.py:64-196
* Jacobian family, diagonals    src/pff_operator.py:244-327
* residual                      src/pff_operator.py:218-241
* state restriction             src/pff_operator.py:380-400
* prolongation / transfers      src/multigrid.py:44-120
* Lanczos range estimate        src/multigrid.py:123-162
* Chebyshev smoother            src/multigrid.py:170-198
* GMG V-cycle                   src/multigrid.py:201-344
* restarted MGS-GMRES           src/krylov.py:37-119
* lumped mass, active set       src/active_set_solver.py:60-82

Parity pin: every function here is checked against golden vectors produced
by running the reference itself (``tests/golden/make_golden.py``,
fixtures in ``tests/golden/*.npz``; test ``tests/test_oracle_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse as sp

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libpff_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle (``make`` in this directory)."""
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "pff_oracle.c"))
    ):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        i, d = ctypes.c_int, ctypes.c_double
        L.or_cache.argtypes = [i, i, dp, dp, dp, dp, dp, dp, dp, d, d, d, d, d, i,
                               dp, dp, dp, dp, dp, dp, dp, i]
        L.or_jacobian.argtypes = [i, i, dp, dp, dp, dp, dp, dp, dp, dp, dp, dp, dp, dp,
                                  d, d, d, d, i, i, i, i, dp, dp, dp, i]
        L.or_diagonal.argtypes = [i, i, dp, dp, dp, dp, dp, dp, dp, dp, d, d, d, d, i,
                                  dp, dp, dp, i]
        L.or_residual.argtypes = [i, i, dp, dp, dp, dp, dp, dp, dp, d, d, d, d, d, i,
                                  dp, dp, dp, i]
        L.or_mass_rowsum.argtypes = [i, i, dp, dp, dp, dp, i]
        L.or_max_threads.restype = i
        for name in ("or_cache", "or_jacobian", "or_diagonal", "or_residual", "or_mass_rowsum"):
            getattr(L, name).restype = i
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def max_threads() -> int:
    return int(lib().or_max_threads())


# ------------------------------------------------------------ shape data
# src/tensor_basis.py:19-81: Gauss-Legendre q = p+1 points on [0,1],
# equidistant support points, Lagrange values/derivatives via the inverse
# Vandermonde matrix.

def gauss_legendre_01(q: int):
    x, wt = np.polynomial.legendre.leggauss(q)
    return 0.5 * (x + 1.0), 0.5 * wt


def support_points_01(p: int) -> np.ndarray:
    return np.linspace(0.0, 1.0, p + 1)


def lagrange_matrices(support: np.ndarray, points: np.ndarray):
    n = support.size
    coeff = np.linalg.inv(np.vander(support, n, increasing=True))
    pw = np.vander(points, n, increasing=True)
    dpw = np.zeros_like(pw)
    dpw[:, 1:] = pw[:, :-1] * np.arange(1, n)
    return pw @ coeff, dpw @ coeff


@dataclass(frozen=True)
class Shape:
    p: int
    points: np.ndarray
    w: np.ndarray
    support: np.ndarray
    N: np.ndarray
    D: np.ndarray

    @property
    def q(self) -> int:
        return self.points.size


def shape(p: int) -> Shape:
    pts, w = gauss_legendre_01(p + 1)
    sup = support_points_01(p)
    N, D = lagrange_matrices(sup, pts)
    return Shape(p, pts, w, sup, np.ascontiguousarray(N), np.ascontiguousarray(D))


# ------------------------------------------------------------------- mesh
# src/mesh_hierarchy.py:156-189 closed form: grid node (i, j) -> j*n1 + i,
# upper slit copies n_grid + i for cells with cy >= N/2 on row j = i_mid,
# i < i_mid (no slit at level 0).

@dataclass(frozen=True)
class Level:
    p: int
    level: int

    @property
    def nside(self) -> int:
        return 2 ** self.level

    @property
    def n1(self) -> int:
        return self.p * self.nside + 1

    @property
    def n_grid(self) -> int:
        return self.n1 * self.n1

    @property
    def i_mid(self) -> int:
        return self.p * self.nside // 2

    @property
    def n_dup(self) -> int:
        return self.i_mid if self.level >= 1 else 0

    @property
    def n(self) -> int:
        return self.n_grid + self.n_dup

    @property
    def h(self) -> float:
        return 1.0 / self.nside

    @property
    def n_cells(self) -> int:
        return self.nside * self.nside

    def conn(self) -> np.ndarray:
        p, ns, n1 = self.p, self.nside, self.n1
        cy, cx = np.divmod(np.arange(ns * ns), ns)
        b, a = np.divmod(np.arange((p + 1) ** 2), p + 1)
        j = cy[:, None] * p + b[None, :]
        i = cx[:, None] * p + a[None, :]
        gid = j * n1 + i
        if self.level >= 1:
            up = (cy[:, None] >= ns // 2) & (j == self.i_mid) & (i < self.i_mid)
            gid = np.where(up, self.n_grid + i, gid)
        return gid.astype(np.int64)

    def coords(self) -> np.ndarray:
        xs = np.arange(self.n1) / (self.n1 - 1)
        gx, gy = np.meshgrid(xs, xs, indexing="xy")
        c = np.column_stack([gx.ravel(), gy.ravel()])
        if self.n_dup:
            c = np.vstack([c, np.column_stack([xs[: self.n_dup], np.full(self.n_dup, 0.5)])])
        return c

    def boundary_nodes(self, tag: str) -> np.ndarray:
        g = np.arange(self.n_grid)
        gi, gj = g % self.n1, g // self.n1
        sel = {"bottom": gj == 0, "top": gj == self.n1 - 1,
               "left": gi == 0, "right": gi == self.n1 - 1}[tag]
        ids = np.flatnonzero(sel)
        if tag == "left" and self.n_dup:
            ids = np.sort(np.append(ids, self.n_grid))
        return ids.astype(np.int64)


def injection(p: int, fine_level: int) -> np.ndarray:
    """src/mesh_hierarchy.py:316-338."""
    f, c = Level(p, fine_level), Level(p, fine_level - 1)
    idx = np.arange(c.n1) * 2
    jj, ii = np.meshgrid(idx, idx, indexing="ij")
    inj = (jj * f.n1 + ii).ravel()
    if c.n_dup:
        inj = np.append(inj, f.n_grid + 2 * np.arange(c.n_dup))
    return inj.astype(np.int64)


# ----------------------------------------------------------------- state

@dataclass(frozen=True)
class Material:
    """src/material_model.py:20-44 (kN / mm units of the reference)."""
    lame_lambda: float = 121.15
    mu: float = 80.77
    g_c: float = 2.7e-3
    kappa: float = 1e-10
    eps: float = 4e-3


class State:
    """Linearisation point on one level (src/pff_operator.py:64-196)."""

    def __init__(self, p: int, level: int, params: Material, split: str = "miehe"):
        if split not in ("none", "miehe"):
            raise ValueError("split must be 'none' or 'miehe'")
        self.lv = Level(p, level)
        self.p, self.level, self.params, self.split = p, level, params, split
        self.shape = shape(p)
        n = self.lv.n
        self.U = np.zeros(3 * n)
        self.U[2 * n:] = 1.0
        self.phi_tilde = np.ones(n)
        self.phi_old = np.ones(n)
        self.active = np.zeros(n, dtype=bool)
        self.dirichlet = np.zeros(n, dtype=bool)
        self.cache = None

    @property
    def n(self) -> int:
        return self.lv.n

    def constrained_mask(self) -> np.ndarray:
        return np.concatenate([self.dirichlet, self.dirichlet, self.active])

    def refresh_cache(self, nthreads: int = 1):
        lv, s, pr = self.lv, self.shape, self.params
        m = lv.n_cells * s.q * s.q
        c = {k: np.empty(m) for k in ("e11", "e22", "e12", "gt", "dg", "esp", "pc")}
        n = lv.n
        ux, uy, ph = (np.ascontiguousarray(self.U[k * n:(k + 1) * n]) for k in range(3))
        pt = np.ascontiguousarray(self.phi_tilde)
        rc = lib().or_cache(self.p, self.level, _p(s.N), _p(s.D), _p(s.w), _p(ux), _p(uy),
                            _p(ph), _p(pt), pr.lame_lambda, pr.mu, pr.g_c, pr.eps, pr.kappa,
                            int(self.split == "miehe"), _p(c["e11"]), _p(c["e22"]),
                            _p(c["e12"]), _p(c["gt"]), _p(c["dg"]), _p(c["esp"]),
                            _p(c["pc"]), nthreads)
        assert rc == 0
        self.cache = c


def _run_jacobian(st: State, dux, duy, dph, do_uu, do_pp, do_coup, nthreads=1):
    """src/pff_operator.py:244-259."""
    c, s, pr, n = st.cache, st.shape, st.params, st.n
    out = np.zeros(3 * n)
    ox, oy, op = out[:n], out[n:2 * n], out[2 * n:]
    dux, duy, dph = (np.ascontiguousarray(v, dtype=np.float64) for v in (dux, duy, dph))
    rc = lib().or_jacobian(st.p, st.level, _p(s.N), _p(s.D), _p(s.w), _p(dux), _p(duy),
                           _p(dph), _p(c["e11"]), _p(c["e22"]), _p(c["e12"]), _p(c["gt"]),
                           _p(c["dg"]), _p(c["pc"]), pr.lame_lambda, pr.mu, pr.g_c, pr.eps,
                           int(st.split == "miehe"), int(do_uu), int(do_pp), int(do_coup),
                           _p(ox), _p(oy), _p(op), nthreads)
    assert rc == 0
    return out


def apply_jacobian(st: State, dU, nthreads=1):
    """src/pff_operator.py:262-270."""
    dU = np.asarray(dU, dtype=float)
    n = st.n
    mask = st.constrained_mask()
    z = np.where(mask, 0.0, dU)
    out = _run_jacobian(st, z[:n], z[n:2 * n], z[2 * n:], True, True, True, nthreads)
    out[mask] = dU[mask]
    return out


def apply_block_uu(st: State, du, nthreads=1):
    """src/pff_operator.py:273-282."""
    n = st.n
    du = np.asarray(du, dtype=float)
    zx = np.where(st.dirichlet, 0.0, du[:n])
    zy = np.where(st.dirichlet, 0.0, du[n:])
    out = _run_jacobian(st, zx, zy, np.zeros(n), True, False, False, nthreads)[:2 * n]
    out[:n][st.dirichlet] = du[:n][st.dirichlet]
    out[n:][st.dirichlet] = du[n:][st.dirichlet]
    return out


def apply_block_phiphi(st: State, dphi, nthreads=1):
    """src/pff_operator.py:285-291."""
    dphi = np.asarray(dphi, dtype=float)
    z = np.where(st.active, 0.0, dphi)
    zn = np.zeros(st.n)
    out = _run_jacobian(st, zn, zn, z, False, True, False, nthreads)[2 * st.n:]
    out[st.active] = dphi[st.active]
    return out


def apply_phi_row(st: State, dU, nthreads=1):
    """src/pff_operator.py:294-302."""
    dU = np.asarray(dU, dtype=float)
    n = st.n
    mask = st.constrained_mask()
    z = np.where(mask, 0.0, dU)
    out = _run_jacobian(st, z[:n], z[n:2 * n], z[2 * n:], False, True, True, nthreads)[2 * n:]
    out[st.active] = dU[2 * n:][st.active]
    return out


def block_diagonal(st: State, block: str, nthreads=1):
    """src/pff_operator.py:305-327."""
    c, s, pr, n = st.cache, st.shape, st.params, st.n
    dx, dy, dp = np.zeros(n), np.zeros(n), np.zeros(n)
    rc = lib().or_diagonal(st.p, st.level, _p(s.N), _p(s.D), _p(s.w), _p(c["e11"]),
                           _p(c["e22"]), _p(c["e12"]), _p(c["gt"]), _p(c["pc"]),
                           pr.lame_lambda, pr.mu, pr.g_c, pr.eps, int(st.split == "miehe"),
                           _p(dx), _p(dy), _p(dp), nthreads)
    assert rc == 0
    if block == "uu":
        dx[st.dirichlet] = 1.0
        dy[st.dirichlet] = 1.0
        return np.concatenate([dx, dy])
    if block == "phiphi":
        dp[st.active] = 1.0
        return dp
    raise ValueError("block must be 'uu' or 'phiphi'")


def residual(st: State, mask_dirichlet=True, mask_active=False, nthreads=1):
    """src/pff_operator.py:218-241."""
    s, pr, n = st.shape, st.params, st.n
    out = np.zeros(3 * n)
    ux, uy, ph = (np.ascontiguousarray(st.U[k * n:(k + 1) * n]) for k in range(3))
    pt = np.ascontiguousarray(st.phi_tilde)
    rc = lib().or_residual(st.p, st.level, _p(s.N), _p(s.D), _p(s.w), _p(ux), _p(uy),
                           _p(ph), _p(pt), pr.lame_lambda, pr.mu, pr.g_c, pr.eps, pr.kappa,
                           int(st.split == "miehe"), _p(out[:n]), _p(out[n:2 * n]),
                           _p(out[2 * n:]), nthreads)
    assert rc == 0
    if mask_dirichlet:
        out[:n][st.dirichlet] = 0.0
        out[n:2 * n][st.dirichlet] = 0.0
    if mask_active:
        out[2 * n:][st.active] = 0.0
    return out


def lumped_mass(p: int, level: int, nthreads=1):
    """src/active_set_solver.py:60-69 -> _kernels.py:828-843."""
    s = shape(p)
    out = np.zeros(Level(p, level).n)
    rc = lib().or_mass_rowsum(p, level, _p(s.N), _p(s.D), _p(s.w), _p(out), nthreads)
    assert rc == 0
    return out


def restrict_state(st: State, target: int) -> State:
    """src/pff_operator.py:380-400 (composed injection)."""
    if not 0 <= target <= st.level:
        raise ValueError("target level out of range")
    if target == st.level:
        return st
    inj = None
    for fine in range(st.level, target, -1):
        step = injection(st.p, fine)
        inj = step if inj is None else inj[step]
    n = st.n
    c = State(st.p, target, st.params, st.split)
    c.U = np.concatenate([st.U[:n][inj], st.U[n:2 * n][inj], st.U[2 * n:][inj]])
    c.phi_tilde = st.phi_tilde[inj].copy()
    c.phi_old = st.phi_old[inj].copy()
    c.active = st.active[inj].copy()
    c.dirichlet = st.dirichlet[inj].copy()
    return c


# -------------------------------------------------------------- transfers

def build_prolongation(p: int, fine_level: int) -> sp.csr_matrix:
    """src/multigrid.py:44-94: each fine row is owned by the first fine cell
    (ascending cell index) that references it; weights are the coarse Lagrange
    basis evaluated through that cell's parent; |w| <= 1e-14 dropped."""
    if fine_level < 1:
        raise ValueError("fine level must be >= 1")
    f, c = Level(p, fine_level), Level(p, fine_level - 1)
    n1 = p + 1
    sup = support_points_01(p)
    embed = [lagrange_matrices(sup, (ch + sup) / 2.0)[0] for ch in (0, 1)]
    cf, cc = f.conn(), c.conn()
    flat = cf.ravel()
    fdofs, first = np.unique(flat, return_index=True)
    cell, k = np.divmod(first, n1 * n1)
    b, a = np.divmod(k, n1)
    fy, fx = np.divmod(cell, f.nside)
    ccell = (fy // 2) * c.nside + fx // 2
    E = np.stack(embed)                                   # (2, n1, n1)
    ey = E[fy % 2, b]                                     # (nrows, n1) over coarse my
    ex = E[fx % 2, a]                                     # (nrows, n1) over coarse mx
    W = (ey[:, :, None] * ex[:, None, :]).reshape(len(fdofs), n1 * n1)
    C = cc[ccell]
    keep = np.abs(W) > 1e-14
    counts = keep.sum(axis=1)
    indptr = np.zeros(f.n + 1, dtype=np.int64)
    indptr[fdofs + 1] = counts
    np.cumsum(indptr, out=indptr)
    return sp.csr_matrix((W[keep], C[keep], indptr), shape=(f.n, c.n))


class Transfer:
    """src/multigrid.py:97-120."""

    def __init__(self, p: int, fine_level: int):
        self.P = build_prolongation(p, fine_level)
        self.R = self.P.T.tocsr()
        self.nf, self.nc = self.P.shape

    def prolongate(self, x):
        nc, nf = self.nc, self.nf
        return np.concatenate([self.P @ x[k * nc:(k + 1) * nc] for k in range(3)])

    def restrict(self, y):
        nc, nf = self.nc, self.nf
        return np.concatenate([self.R @ y[k * nf:(k + 1) * nf] for k in range(3)])


# ---------------------------------------------------------------- solvers

def estimate_lambda_range(apply_fn, diag, max_iterations=30, seed=0, rtol=1e-4):
    """src/multigrid.py:123-162: Lanczos on D^-1/2 A D^-1/2."""
    n = diag.size
    dh = 1.0 / np.sqrt(diag)
    v = np.random.default_rng(seed).standard_normal(n)
    v /= np.linalg.norm(v)
    v_prev = np.zeros(n)
    beta = 0.0
    al, be = [], []
    lo = hi = 1.0
    prev = None
    for _ in range(min(max_iterations, n)):
        w = dh * apply_fn(dh * v)
        w -= beta * v_prev
        alpha = float(v @ w)
        w -= alpha * v
        al.append(alpha)
        ritz = scipy.linalg.eigvalsh_tridiagonal(al, be) if be else np.array([alpha])
        lo, hi = float(ritz[0]), float(ritz[-1])
        beta = float(np.linalg.norm(w))
        if beta < 1e-12 * max(1.0, abs(hi)):
            break
        if prev is not None and abs(hi - prev) <= rtol * abs(hi):
            break
        prev = hi
        be.append(beta)
        v_prev = v
        v = w / beta
    return lo, hi


def chebyshev_apply(apply_fn, diag, rhs, a, b, sweeps):
    """src/multigrid.py:170-198."""
    if not (0.0 < a < b):
        raise ValueError(f"invalid Chebyshev interval [{a}, {b}]")
    if sweeps < 1:
        raise ValueError("sweeps must be >= 1")
    theta, delta = 0.5 * (b + a), 0.5 * (b - a)
    sigma1 = theta / delta
    inv_diag = 1.0 / diag
    d = inv_diag * rhs / theta
    z = d.copy()
    if sweeps == 1:
        return z
    r = rhs - apply_fn(d)
    rho_old = 1.0 / sigma1
    for k in range(1, sweeps):
        rho = 1.0 / (2.0 * sigma1 - rho_old)
        d = (rho * rho_old) * d + (2.0 * rho / delta) * (inv_diag * r)
        z += d
        rho_old = rho
        if k < sweeps - 1:
            r -= apply_fn(d)
    return z


@dataclass
class ChebCfg:
    """src/multigrid.py:27-41."""
    sweeps: int = 5
    coarse_sweeps: int = 32
    c: float = 0.24
    C: float = 1.2
    lambda_min_floor: float = 1e-3
    lanczos_iterations: int = 30
    seed: int = 20240915


class Gmg:
    """src/multigrid.py:201-344."""

    def __init__(self, p: int, max_level: int, coarse_level: int = 2, cheb: ChebCfg | None = None,
                 nthreads: int = 1):
        self.p, self.coarse_level, self.cheb = p, coarse_level, cheb or ChebCfg()
        self.nt = nthreads
        self.transfers = {l: Transfer(p, l) for l in range(coarse_level + 1, max_level + 1)}
        self.states, self.diags, self.ranges, self.cons = {}, {}, {}, {}
        self.finest = None

    def setup(self, st: State, reuse_eigen=False, ranges=None):
        self.finest = st.level
        if st.cache is None:
            st.refresh_cache(self.nt)
        self.states[st.level] = st
        for l in range(st.level - 1, self.coarse_level - 1, -1):
            s = restrict_state(st, l)
            s.refresh_cache(self.nt)
            self.states[l] = s
        for l in range(self.coarse_level, st.level + 1):
            s = self.states[l]
            self.cons[l] = s.constrained_mask()
            self.diags[l] = {"uu": block_diagonal(s, "uu", self.nt),
                             "phiphi": block_diagonal(s, "phiphi", self.nt)}
            if ranges is not None:
                self.ranges[l] = ranges[l]
            elif not reuse_eigen or l not in self.ranges:
                self.ranges[l] = self._estimate(l)

    def _estimate(self, l):
        s, cfg, out = self.states[l], self.cheb, {}
        for block, fn in (("uu", lambda v: apply_block_uu(s, v, self.nt)),
                          ("phiphi", lambda v: apply_block_phiphi(s, v, self.nt))):
            lo, hi = estimate_lambda_range(fn, self.diags[l][block],
                                           max_iterations=cfg.lanczos_iterations,
                                           seed=cfg.seed + 101 * l + (0 if block == "uu" else 1))
            hi = max(hi, 1e-30)
            lo = max(lo, cfg.lambda_min_floor * hi)
            out[block] = (lo, hi)
        return out

    def apply(self, r):
        return self._vcycle(self.finest, np.asarray(r, dtype=float))

    __call__ = apply

    def _smooth(self, l, z, r):
        s, n = self.states[l], self.states[l].n
        res = r - apply_jacobian(s, z, self.nt)
        hi = self.ranges[l]["uu"][1]
        z[:2 * n] += chebyshev_apply(lambda v: apply_block_uu(s, v, self.nt), self.diags[l]["uu"],
                                     res[:2 * n], self.cheb.c * hi, self.cheb.C * hi,
                                     self.cheb.sweeps)
        res_phi = r[2 * n:] - apply_phi_row(s, z, self.nt)
        hi = self.ranges[l]["phiphi"][1]
        z[2 * n:] += chebyshev_apply(lambda v: apply_block_phiphi(s, v, self.nt),
                                     self.diags[l]["phiphi"], res_phi, self.cheb.c * hi,
                                     self.cheb.C * hi, self.cheb.sweeps)

    def _coarse(self, l, r):
        s, n = self.states[l], self.states[l].n
        z = np.zeros(3 * n)
        lo, hi = self.ranges[l]["uu"]
        z[:2 * n] = chebyshev_apply(lambda v: apply_block_uu(s, v, self.nt), self.diags[l]["uu"],
                                    r[:2 * n], lo, self.cheb.C * hi, self.cheb.coarse_sweeps)
        res_phi = r[2 * n:] - apply_phi_row(s, z, self.nt)
        lo, hi = self.ranges[l]["phiphi"]
        z[2 * n:] = chebyshev_apply(lambda v: apply_block_phiphi(s, v, self.nt),
                                    self.diags[l]["phiphi"], res_phi, lo, self.cheb.C * hi,
                                    self.cheb.coarse_sweeps)
        cons = self.cons[l]
        z[cons] = r[cons]
        return z

    def _vcycle(self, l, r):
        if l == self.coarse_level:
            return self._coarse(l, r)
        cons = self.cons[l]
        z = np.where(cons, r, 0.0)
        self._smooth(l, z, r)
        res = r - apply_jacobian(self.states[l], z, self.nt)
        rc = self.transfers[l].restrict(res)
        rc[self.cons[l - 1]] = 0.0
        zc = self._vcycle(l - 1, rc)
        dz = self.transfers[l].prolongate(zc)
        dz[cons] = 0.0
        z += dz
        self._smooth(l, z, r)
        return z


@dataclass
class GmresOut:
    solution: np.ndarray
    iterations: int
    history: list = field(default_factory=list)
    converged: bool = False
    wall_seconds: float = 0.0


def gmres(apply_op, rhs, tol=1e-6, max_iterations=1000, restart=100, floor=1e-30,
          preconditioner=None, x0=None) -> GmresOut:
    """src/krylov.py:37-119: right-preconditioned restarted GMRES, MGS,
    Givens rotations, true residual at every restart."""
    t0 = time.perf_counter()
    rhs = np.asarray(rhs, dtype=float)
    n = rhs.size
    x = np.zeros(n) if x0 is None else np.asarray(x0, dtype=float).copy()
    bn = float(np.linalg.norm(rhs))
    target = max(tol * bn, floor)
    r = rhs - apply_op(x) if x0 is not None else rhs.copy()
    rn = float(np.linalg.norm(r))
    hist = [rn]
    total = 0
    if rn <= target:
        return GmresOut(x, 0, hist, True, time.perf_counter() - t0)
    M = preconditioner or (lambda v: v)
    while total < max_iterations:
        m = min(restart, max_iterations - total)
        V = np.empty((m + 1, n))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        V[0] = r / rn
        g[0] = rn
        used = 0
        for j in range(m):
            w = np.array(apply_op(M(V[j])), dtype=float, copy=True)
            for i in range(j + 1):
                H[i, j] = float(V[i] @ w)
                w -= H[i, j] * V[i]
            hn = float(np.linalg.norm(w))
            H[j + 1, j] = hn
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = float(np.hypot(H[j, j], H[j + 1, j]))
            if den == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            used = j + 1
            hist.append(abs(g[j + 1]))
            if abs(g[j + 1]) <= target:
                break
            if hn <= 1e-14 * max(1.0, rn):
                break
            V[j + 1] = w / hn
        y = np.zeros(used)
        for i in range(used - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:used] @ y[i + 1:]) / H[i, i]
        x = x + M(V[:used].T @ y)
        r = rhs - apply_op(x)
        rn = float(np.linalg.norm(r))
        hist[-1] = rn
        if rn <= target:
            return GmresOut(x, total, hist, True, time.perf_counter() - t0)
    return GmresOut(x, total, hist, False, time.perf_counter() - t0)


def determine_active_set(newton_rhs, U, phi_old, m_diag, c):
    """src/active_set_solver.py:72-82."""
    n = m_diag.size
    return newton_rhs[2 * n:] / m_diag + c * (U[2 * n:] - phi_old) > 0.0


# ------------------------------------------------------- synthetic inputs
# BASELINE.json configs; rng = default_rng(seed),
# draw order u0 (2n) -> phi0 (n) -> x (3n); phi_tilde = phi_old = phi0;
# active = phi0 < 0.05; Dirichlet = top + bottom; eps = 2h.

def baseline_material(level: int) -> Material:
    return Material(lame_lambda=121.15e3, mu=80.77e3, g_c=2.7, kappa=1e-10, eps=2.0 / 2 ** level)


def baseline_state(p: int, level: int, split: str, seed: int = 0, notch: bool = False):
    """Returns (state, x) for the BASELINE configs (x ~ U[-1,1], 3n)."""
    st = State(p, level, baseline_material(level), split)
    lv, n = st.lv, st.n
    rng = np.random.default_rng(seed)
    u0 = rng.uniform(-1e-3, 1e-3, 2 * n)
    if notch:
        phi0 = notch_phase(lv, st.params.eps)
    else:
        phi0 = rng.uniform(0.0, 1.0, n)
    x = rng.uniform(-1.0, 1.0, 3 * n)
    st.U = np.concatenate([u0, phi0])
    st.phi_tilde = phi0.copy()
    st.phi_old = phi0.copy()
    st.active = phi0 < 0.05
    st.dirichlet = np.zeros(n, dtype=bool)
    st.dirichlet[np.concatenate([lv.boundary_nodes("top"), lv.boundary_nodes("bottom")])] = True
    return st, x


def notch_phase(lv: Level, eps: float) -> np.ndarray:
    """phi0 = 1 - exp(-d/eps), d = distance to the slit {y=0.5, 0<=x<=0.5}."""
    c = lv.coords()
    x, y = c[:, 0], c[:, 1]
    dx = np.maximum(x - 0.5, 0.0)
    d = np.sqrt(dx * dx + (y - 0.5) ** 2)
    return 1.0 - np.exp(-d / eps)


# ------------------------------------------------------- active-set loop
# src/simulation_driver.py:116-148 (boundary data) and
# src/active_set_solver.py:31-163 (PDAS loop)

def boundary_program(scenario: str, t: float, du: float = 1e-5) -> dict:
    """src/simulation_driver.py:116-131."""
    if t < 0:
        raise ValueError("time must be nonnegative")
    if scenario == "tension":
        return {("top", 0): 0.0, ("top", 1): t * du, ("bottom", 0): 0.0, ("bottom", 1): 0.0}
    if scenario == "shear":
        return {("top", 0): t * du, ("top", 1): 0.0, ("bottom", 0): 0.0, ("bottom", 1): 0.0}
    raise ValueError(f"unknown scenario {scenario!r}")


def apply_boundary_values(st: State, values: dict) -> None:
    """src/simulation_driver.py:134-145."""
    n = st.n
    nodes_all = []
    for (tag, comp), val in values.items():
        nodes = st.lv.boundary_nodes(tag)
        st.U[comp * n + nodes] = val
        nodes_all.append(nodes)
    st.dirichlet = np.zeros(n, dtype=bool)
    st.dirichlet[np.unique(np.concatenate(nodes_all))] = True
    st.cache = None


class SolverFailure(RuntimeError):
    pass


@dataclass
class ActiveSetReport:
    as_iterations: int = 0
    gmres_iterations: list = field(default_factory=list)
    active_counts: list = field(default_factory=list)
    residual_norms: list = field(default_factory=list)
    r0_norm: float = 0.0
    converged: bool = False


def active_set_solve_step(st: State, gmg: Gmg, m_diag, c=100.0, tol=1e-8, max_iterations=50,
                          lin_tol=1e-6, lin_max=1000, restart=100, nthreads=1) -> ActiveSetReport:
    """src/active_set_solver.py:101-163 (ActiveSetSolver.solve_step)."""
    rep = ActiveSetReport()
    n = st.n
    prev = None
    for k in range(max_iterations):
        rhs = -residual(st, nthreads=nthreads)
        active = determine_active_set(rhs, st.U, st.phi_old, m_diag, c)
        moved = active & (st.U[2 * n:] != st.phi_old)
        if np.any(moved):
            st.U[2 * n:][moved] = st.phi_old[moved]
            rhs = -residual(st, nthreads=nthreads)
        st.active = active
        st.cache = None
        rhs[2 * n:][active] = 0.0
        r_norm = float(np.linalg.norm(rhs))
        if k == 0:
            rep.r0_norm = max(r_norm, 1e-300)
        rep.active_counts.append(int(active.sum()))
        rep.residual_norms.append(r_norm)
        if prev is not None and np.array_equal(active, prev) and r_norm <= tol * rep.r0_norm:
            rep.converged = True
            break
        st.refresh_cache(nthreads)
        reuse = prev is not None and np.array_equal(active, prev)
        gmg.setup(st, reuse_eigen=reuse)
        A = lambda v: apply_jacobian(st, v, nthreads)  # noqa: E731
        res = gmres(A, rhs, tol=lin_tol, max_iterations=lin_max, restart=restart,
                    preconditioner=gmg.apply)
        if not res.converged:
            res = gmres(A, rhs, tol=lin_tol, max_iterations=2 * lin_max, restart=restart,
                        preconditioner=gmg.apply, x0=res.solution)
            if not res.converged:
                raise SolverFailure(f"linear solve stagnated at active-set iteration {k}")
        st.U = st.U + res.solution
        st.cache = None
        rep.gmres_iterations.append(res.iterations)
        rep.as_iterations = k + 1
        prev = active
    else:
        raise SolverFailure(f"active-set loop did not converge within {max_iterations} iterations")
    return rep
