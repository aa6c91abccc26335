"""Geometric multigrid V-cycle on the B200 (drop-in for src/multigrid.py).

Same algebra as the reference (src/multigrid.py:201-344): block
Chebyshev-Jacobi smoothing (u block, then phi block), Q_p embedding
transfers, a Chebyshev "solve" on the coarse level, Lanczos range
estimates with the reference's seeds.  Every vector operation of the cycle
is a libpff_b200 kernel on device-resident per-level buffers, and the whole
cycle is captured once per setup into a CUDA graph, so one ``apply`` is one
graph launch instead of a few hundred kernel launches.
"""

from __future__ import annotations

import ctypes
import logging
import os
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from functools import cached_property

import numpy as np
import scipy.linalg
import scipy.sparse as sp
import torch

from . import _lib
from . import operator as op
from ._lib import call, ptr, stream_handle
from .basis import MaterialParams, lagrange_matrices, shape_data, support_points_01
from .mesh import MeshHierarchy

logger = logging.getLogger(__name__)

FUSE_CHEB = True   # Chebyshev steps fused into the block applications (pff_apply_cheb)
# coarse solve as precomputed dense linear maps (pff_coarse_dense) on coarse
# levels of at most COARSE_DENSE_NMAX scalar nodes (Q2 level 2: 85)
# pff_cheb_init folded into the residual producers (pff_apply_emit, pff_smooth_init)
FUSE_INIT = os.environ.get("PFF_FUSE_INIT", "1") != "0"
EMIT_PHIROW = os.environ.get("PFF_EMIT_PHIROW", "1") != "0"
# the later smoothings' u-block residual as the UU application on (z_u, r_u): its phi
# rows are never read and G has no u-phi block, so the u rows are bitwise those of the
# FULL residual at 4 tile arrays and 2 fields instead of 7 and 3 (Newton solve at
# 1024^2: 97.5 -> 95.2 ms of device time)
POST_UU = os.environ.get("PFF_POST_UU", "1") != "0"
# first smoothing: pff_smooth_init adds the u block's Chebyshev start to z itself and the
# fused steps touch z only every second step ((z + d_k) + d_k+1 in one update,
# PFF_CHEB_NOACC / PFF_CHEB_FIRST: bitwise the step-by-step sums, one read and write
# of z fewer per skipped step)
DEFER_ACC = os.environ.get("PFF_DEFER_ACC", "1") != "0"
# that residual emitting the u block's d0 (pff_apply_emit): as the FULL application it
# measured slower (+4.5 ms per solve) than the separate pff_cheb_init pass it replaces;
# as the UU application it is faster (95.2 -> 94.0 ms) -- on with POST_UU
EMIT_FULL = os.environ.get("PFF_EMIT_FULL", "1" if POST_UU else "0") != "0"
DENSE_COARSE = os.environ.get("PFF_DENSE_COARSE", "1") != "0"
COARSE_DENSE_NMAX = 256
# the whole V-cycle from the level above the coarse one as one dense map
# (pff_dense_matvec) when that level has at most DENSE_LEVEL_NMAX scalar nodes
# (Q2 level 3: 297)
DENSE_LEVEL = os.environ.get("PFF_DENSE_LEVEL", "1") != "0"
DENSE_LEVEL_NMAX = 400
NATIVE_LANCZOS = True   # setup's batched Lanczos driven by pff_lanczos_ranges (C++)
_EAGER_DONE: set = set()


@dataclass
class ChebyshevConfig:
    """Smoothing/solve ranges and sweep counts (src/multigrid.py:27-41)."""

    sweeps: int = 5
    coarse_sweeps: int = 32
    c: float = 0.24
    C: float = 1.2
    lambda_min_floor: float = 1e-3
    lanczos_iterations: int = 30
    seed: int = 20240915

    def __post_init__(self):
        if not (0.0 < self.c <= 1.0 <= self.C):
            raise ValueError("need 0 < c <= 1 <= C")


# --------------------------------------------------------------- helpers

def _dev():
    _lib.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _empty(n):
    return torch.empty(n, dtype=torch.float64, device=_dev())


def _dot(x: torch.Tensor, y: torch.Tensor, scratch: torch.Tensor, out: torch.Tensor) -> float:
    call("pff_dot", x.numel(), ptr(x), ptr(y), ptr(scratch), ptr(out), stream_handle())
    return float(out[0].item())


class _Scratch:
    def __init__(self):
        self.partials = _empty(_lib.load().pff_reduce_scratch_len())
        self.out = _empty(4)

    def dot(self, x, y) -> float:
        return _dot(x, y, self.partials, self.out)

    def norm(self, x) -> float:
        return float(np.sqrt(self.dot(x, x)))


def _axpby(a, x, b, y):
    call("pff_axpby", y.numel(), float(a), ptr(x), float(b), ptr(y), stream_handle())
    return y


class _HostCallable:
    """Wrap a user callable so it sees the array type the user passed in."""

    def __init__(self, fn, numpy_mode: bool):
        self.fn, self.numpy_mode = fn, numpy_mode

    def __call__(self, t: torch.Tensor) -> torch.Tensor:
        if self.numpy_mode:
            res = self.fn(t.cpu().numpy())
        else:
            res = self.fn(t)
        out, _ = op.as_device(res, t.numel())
        if out.data_ptr() == t.data_ptr():
            out = out.clone()   # the reference's callables always return new arrays
        return out


def _level_handle(hierarchy: MeshHierarchy, level: int):
    h = ctypes.c_void_p()
    s = shape_data(hierarchy.degree)
    mat = _lib.material(MaterialParams())
    E = s.embedding()
    call("pff_level_create", ctypes.byref(h), hierarchy.degree, level, 0, ctypes.byref(mat),
         s.values.ctypes.data, s.derivatives.ctypes.data, s.quad_weights.ctypes.data,
         E.ctypes.data)
    return h


# ------------------------------------------------------------- transfers

def build_prolongation(hierarchy: MeshHierarchy, fine_level: int) -> sp.csr_matrix:
    """The assembled scalar embedding (src/multigrid.py:44-94), for callers
    that want the matrix; the V-cycle itself uses the structured kernels."""
    if fine_level < 1:
        raise ValueError("fine level must be >= 1")
    dmf, dmc = hierarchy.dof_map(fine_level), hierarchy.dof_map(fine_level - 1)
    p = hierarchy.degree
    n1 = p + 1
    sup = support_points_01(p)
    E = np.stack([lagrange_matrices(sup, (ch + sup) / 2.0)[0] for ch in (0, 1)])
    flat = dmf.conn.ravel()
    fdofs, first = np.unique(flat, return_index=True)
    cell, k = np.divmod(first, n1 * n1)
    b, a = np.divmod(k, n1)
    nsf = 2 ** fine_level
    fy, fx = np.divmod(cell, nsf)
    ccell = (fy // 2) * (nsf // 2) + fx // 2
    W = (E[fy % 2, b][:, :, None] * E[fx % 2, a][:, None, :]).reshape(len(fdofs), n1 * n1)
    C = dmc.conn[ccell]
    keep = np.abs(W) > 1e-14
    indptr = np.zeros(dmf.n_scalar + 1, dtype=np.int64)
    indptr[fdofs + 1] = keep.sum(axis=1)
    np.cumsum(indptr, out=indptr)
    return sp.csr_matrix((W[keep], C[keep], indptr), shape=(dmf.n_scalar, dmc.n_scalar))


class TransferOperator:
    """Componentwise prolongation/restriction between adjacent levels
    (src/multigrid.py:97-120), as structured device kernels."""

    def __init__(self, hierarchy: MeshHierarchy, fine_level: int):
        if fine_level < 1:
            raise ValueError("fine level must be >= 1")
        self.hierarchy = hierarchy
        self.fine_level = fine_level
        self.n_fine = hierarchy.dof_map(fine_level).n_scalar
        self.n_coarse = hierarchy.dof_map(fine_level - 1).n_scalar
        self._h = None

    def _handles(self):
        if self._h is None:
            self._h = (_level_handle(self.hierarchy, self.fine_level),
                       _level_handle(self.hierarchy, self.fine_level - 1))
        return self._h

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib._lib is not None:
                for h in self._h:
                    _lib._lib.pff_level_destroy(h)
        except Exception:
            pass

    @cached_property
    def P(self) -> sp.csr_matrix:
        return build_prolongation(self.hierarchy, self.fine_level)

    @cached_property
    def R(self) -> sp.csr_matrix:
        return self.P.T.tocsr()

    def prolongate(self, coarse):
        x, was_np = op.as_device(coarse, 3 * self.n_coarse)
        out = _empty(3 * self.n_fine)
        hf, hc = self._handles()
        call("pff_prolongate", hf, hc, ptr(x), ptr(out), 0, stream_handle())
        return op.back(out, was_np)

    def restrict(self, fine):
        y, was_np = op.as_device(fine, 3 * self.n_fine)
        out = _empty(3 * self.n_coarse)
        hf, hc = self._handles()
        call("pff_restrict", hf, hc, ptr(y), ptr(out), 0, stream_handle())
        return op.back(out, was_np)


# ------------------------------------------------------ Lanczos / Chebyshev

def estimate_lambda_range(apply_fn, diag, max_iterations: int = 30, seed: int = 0,
                          rtol: float = 1e-4):
    """Lanczos Ritz estimates of the extremal eigenvalues of diag^-1 A
    (src/multigrid.py:123-162), device vectors, host tridiagonal solve."""
    numpy_mode = not isinstance(diag, torch.Tensor)
    d, _ = op.as_device(diag)
    n = d.numel()
    fn = apply_fn if getattr(apply_fn, "_pff_device", False) else _HostCallable(apply_fn, numpy_mode)
    sc = _Scratch()
    dhalf = 1.0 / torch.sqrt(d)
    v_h = np.random.default_rng(seed).standard_normal(n)
    v_h /= np.linalg.norm(v_h)
    v = torch.from_numpy(v_h).to(d.device)
    v_prev = torch.zeros_like(v)
    tmp = torch.empty_like(v)
    beta = 0.0
    alphas, betas = [], []
    lam_min = lam_max = 1.0
    prev_max = None
    s = stream_handle()
    for _ in range(min(max_iterations, n)):
        call("pff_mul", n, ptr(dhalf), ptr(v), ptr(tmp), s)
        w = fn(tmp)
        call("pff_mul", n, ptr(dhalf), ptr(w), ptr(w), s)
        _axpby(-beta, v_prev, 1.0, w)
        alpha = sc.dot(v, w)
        _axpby(-alpha, v, 1.0, w)
        alphas.append(alpha)
        ritz = scipy.linalg.eigvalsh_tridiagonal(alphas, betas) if betas else np.array([alpha])
        lam_min, lam_max = float(ritz[0]), float(ritz[-1])
        beta = sc.norm(w)
        if beta < 1e-12 * max(1.0, abs(lam_max)):
            break
        if prev_max is not None and abs(lam_max - prev_max) <= rtol * abs(lam_max):
            break
        prev_max = lam_max
        betas.append(beta)
        v_prev, v = v, w
        call("pff_div", n, ptr(v), None, beta, ptr(v), s)
    return lam_min, lam_max


def estimate_lambda_max(apply_fn, diag, max_iterations: int = 30, seed: int = 0) -> float:
    return estimate_lambda_range(apply_fn, diag, max_iterations, seed)[1]


def chebyshev_apply(apply_fn, diag, rhs, a: float, b: float, sweeps: int):
    """Fixed-sweep Chebyshev iteration for A z = rhs on [a, b]
    (src/multigrid.py:170-198)."""
    if not (0.0 < a < b):
        raise ValueError(f"invalid Chebyshev interval [{a}, {b}]")
    if sweeps < 1:
        raise ValueError("sweeps must be >= 1")
    numpy_mode = not isinstance(rhs, torch.Tensor)
    rh, was_np = op.as_device(rhs)
    dg, _ = op.as_device(diag, rh.numel())
    n = rh.numel()
    fn = apply_fn if getattr(apply_fn, "_pff_device", False) else _HostCallable(apply_fn, numpy_mode)
    theta, delta = 0.5 * (b + a), 0.5 * (b - a)
    sigma1 = theta / delta
    invd = 1.0 / dg
    d, z = torch.empty_like(rh), torch.empty_like(rh)
    s = stream_handle()
    call("pff_cheb_init", n, ptr(invd), ptr(rh), theta, ptr(d), ptr(z), 0, s)
    if sweeps == 1:
        return op.back(z, was_np)
    r = rh.clone()
    _axpby(-1.0, fn(d), 1.0, r)
    rho_old = 1.0 / sigma1
    for k in range(1, sweeps):
        rho = 1.0 / (2.0 * sigma1 - rho_old)
        call("pff_cheb_step", n, ptr(invd), ptr(r), rho * rho_old, 2.0 * rho / delta, ptr(d),
             ptr(z), s)
        rho_old = rho
        if k < sweeps - 1:
            _axpby(-1.0, fn(d), 1.0, r)
    return op.back(z, was_np)


# --------------------------------------------------------------- V-cycle

class _BlockApply:
    """Device block operator of one level, flagged as tensor-native.  Results
    alternate between two buffers (callers keep at most the previous one)."""
    _pff_device = True

    def __init__(self, state, mode, n):
        self.state, self.mode, self.n = state, mode, n
        self._buf = None
        self._k = 0

    def __call__(self, v):
        if self._buf is None:
            self._buf = (_empty(self.n), _empty(self.n), _empty(self.n))
        self._k = (self._k + 1) % 3
        out = self._buf[self._k]
        self.state.apply_into(self.mode, v, out)
        return out


# Lanczos start vectors: numpy's default_rng(seed).standard_normal(n), exactly
# the reference's draw (src/multigrid.py:133-135), so ranges match it.  They
# depend only on (seed, n): generated once on a worker thread (numpy releases
# the GIL) that overlaps the GPU setup work, and cached across setups.
_START = {}
_START_LOCK = threading.Lock()
_POOL = None


def _start_vector_host(seed: int, n: int) -> np.ndarray:
    v = np.random.default_rng(seed).standard_normal(n)
    v /= np.linalg.norm(v)
    return v


def prefetch_start_vectors(keys):
    global _POOL
    with _START_LOCK:
        if _POOL is None:
            _POOL = ThreadPoolExecutor(max_workers=1, thread_name_prefix="pff-lanczos-rng")
        for key in keys:
            if key not in _START:
                _START[key] = _POOL.submit(_start_vector_host, *key)
                while len(_START) > 64:            # bounded cache
                    _START.pop(next(iter(_START)))


def start_vector(seed: int, n: int) -> np.ndarray:
    prefetch_start_vectors([(seed, n)])
    return _START[(seed, n)].result()


_START_DEV: dict = {}


def start_vector_device(seed: int, n: int, device) -> torch.Tensor:
    """The seeded start vector (numpy's generator, as the reference) kept on
    the device across setups; callers get their own copy."""
    key = (seed, n, str(device))
    t = _START_DEV.get(key)
    if t is None:
        t = torch.from_numpy(start_vector(seed, n)).pin_memory().to(device, non_blocking=True)
        _START_DEV[key] = t
        while len(_START_DEV) > 64:
            _START_DEV.pop(next(iter(_START_DEV)))
    return t.clone()


class _LanczosRun:
    """One estimate_lambda_range run split at its two reductions."""

    def __init__(self, level, block, fn, diag, seed, max_it):
        self.level, self.block, self.fn = level, block, fn
        self.n = diag.numel()
        self.dhalf = 1.0 / torch.sqrt(diag)
        self.v = start_vector_device(seed, self.n, diag.device)
        self.v_prev = torch.zeros_like(self.v)
        self.tmp = torch.empty_like(self.v)
        self.w = None
        self.beta = 0.0
        self.alphas, self.betas = [], []
        self.lo = self.hi = 1.0
        self.prev = None
        self.left = min(max_it, self.n)
        self.done = self.left <= 0

    def step_a(self):
        st = stream_handle()
        call("pff_mul", self.n, ptr(self.dhalf), ptr(self.v), ptr(self.tmp), st)
        self.w = self.fn(self.tmp)
        call("pff_mul", self.n, ptr(self.dhalf), ptr(self.w), ptr(self.w), st)
        _axpby(-self.beta, self.v_prev, 1.0, self.w)

    def step_b(self, alpha, ritz=True):
        _axpby(-alpha, self.v, 1.0, self.w)
        self.alphas.append(alpha)
        if ritz:
            r = (scipy.linalg.eigvalsh_tridiagonal(self.alphas, self.betas) if self.betas
                 else np.array([alpha]))
            self.lo, self.hi = float(r[0]), float(r[-1])


    def step_c(self, beta):
        self.beta = beta
        self.left -= 1
        if beta < 1e-12 * max(1.0, abs(self.hi)):
            self.done = True
            return
        if self.prev is not None and abs(self.hi - self.prev) <= 1e-4 * abs(self.hi):
            self.done = True
            return
        self.prev = self.hi
        self.betas.append(beta)
        self.v_prev, self.v = self.v, self.w
        call("pff_div", self.n, ptr(self.v), None, beta, ptr(self.v), stream_handle())
        if self.left <= 0:
            self.done = True


def _ritz_batched(runs):
    """Extreme Ritz values of several Lanczos tridiagonals at once (runs in
    lockstep have equal sizes): one batched dense eigvalsh per size instead of
    one tridiagonal solve per run."""
    by_k: dict = {}
    for r in runs:
        by_k.setdefault(len(r.alphas), []).append(r)
    for k, group in by_k.items():
        T = np.zeros((len(group), k, k))
        idx = np.arange(k)
        for g, r in enumerate(group):
            T[g, idx, idx] = r.alphas
            if k > 1:
                T[g, idx[1:], idx[:-1]] = r.betas
                T[g, idx[:-1], idx[1:]] = r.betas
        ev = np.linalg.eigvalsh(T)
        for g, r in enumerate(group):
            r.lo, r.hi = float(ev[g, 0]), float(ev[g, -1])


def _recip(x: torch.Tensor, mode: int) -> torch.Tensor:
    """1/x (mode 0) or 1/sqrt(x) (mode 1) by pff_recip."""
    y = torch.empty_like(x)
    call("pff_recip", x.numel(), ptr(x), ptr(y), mode, stream_handle())
    return y


class _LevelWork:
    def __init__(self, n):
        self.r = _empty(3 * n)      # level right-hand side (restricted residual)
        self.z = _empty(3 * n)      # level correction
        self.res = _empty(3 * n)
        self.resphi = _empty(n)
        self.d = _empty(2 * n)
        self.d2 = _empty(2 * n)     # ping-pong partner of d (fused Chebyshev steps)
        self.cr = _empty(2 * n)


class _ConsView(dict):
    """gmg.cons[l] as in the reference (host masks), computed on demand."""

    def __init__(self, gmg):
        super().__init__()
        self._gmg = gmg

    def __missing__(self, l):
        return self._gmg.states[l].constrained_mask()

    def __contains__(self, l):
        return l in self._gmg.states


_CAPTURE_STREAMS: dict = {}


def _capture_stream() -> torch.cuda.Stream:
    dev = torch.cuda.current_device()
    if dev not in _CAPTURE_STREAMS:
        _CAPTURE_STREAMS[dev] = torch.cuda.Stream(device=dev)
    return _CAPTURE_STREAMS[dev]


class GmgPreconditioner:
    """V-cycle over restricted linearisation states; a fixed linear operator
    (src/multigrid.py:201-344)."""

    def __init__(self, hierarchy: MeshHierarchy, coarse_level: int = 2,
                 cheb: ChebyshevConfig | None = None, use_graph: bool = True):
        if coarse_level < 2:
            raise ValueError("coarse level must be >= 2")
        if coarse_level > hierarchy.max_level:
            raise ValueError("hierarchy shallower than the coarse level")
        self.hierarchy = hierarchy
        self.coarse_level = coarse_level
        self.cheb = cheb or ChebyshevConfig()
        self.transfers = {l: TransferOperator(hierarchy, l)
                          for l in range(coarse_level + 1, hierarchy.max_level + 1)}
        self.states: dict[int, op.LinearizationState] = {}
        self.diags: dict[int, dict] = {}
        self.ranges: dict[int, dict] = {}
        self.cons = _ConsView(self)
        self.finest: int | None = None
        self.use_graph = use_graph
        self._inv: dict[int, tuple] = {}
        self._work: dict[int, _LevelWork] = {}
        self._dense = None
        self._dense_l = None
        self._graph = None
        self._scratch = None

    # -- setup -----------------------------------------------------------------
    def setup(self, state: op.LinearizationState, reuse_eigen: bool = False, ranges=None):
        self.finest = state.level
        if state.level < self.coarse_level:
            raise ValueError("state level below the coarse level")
        if ranges is None:   # overlap the start-vector draws with the GPU setup below
            keys = []
            for l in range(state.level, self.coarse_level - 1, -1):
                if not reuse_eigen or l not in self.ranges:
                    n = self.hierarchy.dof_map(l).n_scalar
                    keys += [(self.cheb.seed + 101 * l, 2 * n), (self.cheb.seed + 101 * l + 1, n)]
            prefetch_start_vectors(keys)
        if state._cache_version != state.version:
            state.refresh_cache()
        self.states = {state.level: state}
        cur = state
        for l in range(state.level - 1, self.coarse_level - 1, -1):
            cur = op.restrict_state_to_level(cur, l)
            cur.refresh_cache()
            self.states[l] = cur
        for l in range(self.coarse_level, state.level + 1):
            s = self.states[l]
            duu, dpp = op.block_diagonals(s, invert=False)
            self.diags[l] = {"uu": duu, "phiphi": dpp}
            self._inv[l] = (_recip(duu, 0), _recip(dpp, 0))
            if l not in self._work or self._work[l].resphi.numel() != s.n_scalar:
                self._work[l] = _LevelWork(s.n_scalar)
        todo = []
        for l in range(self.coarse_level, state.level + 1):
            if ranges is not None:
                self.ranges[l] = ranges[l]
            elif not reuse_eigen or l not in self.ranges:
                todo.append(l)
        if todo:
            self.ranges.update(self._estimate_ranges_batched(todo))
        self._build_dense_coarse()
        self._build_dense_level()
        self._graph = None
        if logger.isEnabledFor(logging.DEBUG):
            logger.debug("gmg setup: levels %d..%d, ranges %s", self.coarse_level, state.level,
                         {l: (r["uu"][1], r["phiphi"][1]) for l, r in self.ranges.items()})

    # -- dense maps of the coarse end of the cycle (own kernels: pff_dense.cu) ----
    @staticmethod
    def _gemm(C, A, B, alpha=1.0, beta=0.0):
        """C = alpha A B + beta C on row-major (sub-)matrix views."""
        call("pff_dgemm", C.shape[0], C.shape[1], A.shape[1], float(alpha), ptr(A), A.stride(0),
             ptr(B), B.stride(0), float(beta), ptr(C), C.stride(0), stream_handle())
        return C

    @staticmethod
    def _axpby(Y, a, X, b, s=None):
        """Y = a Y + b diag(s) X."""
        call("pff_dmat_axpby", Y.shape[0], Y.shape[1], float(a), ptr(Y), Y.stride(0), float(b),
             ptr(s), ptr(X), X.stride(0), stream_handle())
        return Y

    @staticmethod
    def _diagm(Y, s=None):
        call("pff_dmat_diag", Y.shape[0], ptr(s), ptr(Y), Y.stride(0), stream_handle())
        return Y

    def _dense_jacobian(self, s):
        """Masked dense Jacobian of a (small) level: pff_cell_matrices scattered
        by pff_dense_jacobian (identity constrained rows and columns)."""
        n = s.n_scalar
        nl = 3 * s.dof_map.n_local
        gk = torch.empty((s.mesh.n_cells, nl, nl), dtype=torch.float64, device=_dev())
        st = stream_handle()
        call("pff_cell_matrices", s.bind(), ptr(gk), st)
        G = torch.empty((3 * n, 3 * n), dtype=torch.float64, device=_dev())
        call("pff_dense_jacobian", s.bind(), ptr(gk), ptr(G), st)
        return G

    def _cheb_poly(self, A, invd, a, b, sweeps):
        """The Jacobi-Chebyshev pass (src/multigrid.py:170-198) as a matrix
        polynomial: the reference recurrence run on the identity."""
        nb = A.shape[0]
        theta, delta = 0.5 * (b + a), 0.5 * (b - a)
        sigma1 = theta / delta
        d = self._diagm(torch.empty((nb, nb), dtype=torch.float64, device=A.device), invd)
        self._axpby(d, 0.0, d, 1.0 / theta)
        acc = self._axpby(torch.empty_like(d), 0.0, d, 1.0)
        cr = self._diagm(torch.empty_like(d))
        rho_old = 1.0 / sigma1
        for _ in range(1, sweeps):
            rho = 1.0 / (2.0 * sigma1 - rho_old)
            self._gemm(cr, A, d, -1.0, 1.0)                            # cr -= G d
            self._axpby(d, rho * rho_old, cr, 2.0 * rho / delta, invd)   # d = c1 d + c2 D^-1 cr
            self._axpby(acc, 1.0, d, 1.0)                               # z += d
            rho_old = rho
        return acc

    def _build_dense_coarse(self):
        """Coarse solve (src/multigrid.py:311-328) as fixed linear maps: the
        coarse_sweeps-step Jacobi-Chebyshev pass on a block is the matrix
        polynomial obtained by running the reference recurrence (cheb_init, then
        cr -= G d, d = c1 d + c2 D^-1 cr, z += d) on the identity.  The blocks come
        from the masked dense Jacobian of the coarse level (identity constrained
        rows/columns, as pff_apply's modes)."""
        self._dense = None
        l = self.coarse_level
        s = self.states[l]
        n = s.n_scalar
        if not DENSE_COARSE or n > COARSE_DENSE_NMAX:
            return
        G = self._dense_jacobian(s)
        inv_u, inv_p = self._inv[l]
        cfg = self.cheb
        lo, hi = self.ranges[l]["uu"]
        Cu = self._cheb_poly(G[:2 * n, :2 * n], inv_u, lo, cfg.C * hi, cfg.coarse_sweeps)
        lo, hi = self.ranges[l]["phiphi"]
        Cp = self._cheb_poly(G[2 * n:, 2 * n:], inv_p, lo, cfg.C * hi, cfg.coarse_sweeps)
        Gpu = self._axpby(torch.empty((n, 2 * n), dtype=torch.float64, device=G.device), 0.0,
                          G[2 * n:, :2 * n], 1.0)
        cmask = torch.from_numpy(s.constrained_mask().astype(np.uint8)).to(G.device)
        self._dense = (n, Cu, Gpu, Cp, cmask)

    def _transfer_dense(self, L, dev):
        """Dense scalar prolongation P (n x nc) of level L and its transpose,
        from the structured CSR (host), cached per hierarchy."""
        key = ("dense_P", L)
        cache = self.__dict__.setdefault("_dense_P_cache", {})
        if key not in cache:
            P = self.transfers[L].P.toarray()
            cache[key] = (torch.from_numpy(P).to(dev), torch.from_numpy(np.ascontiguousarray(P.T)).to(dev))
        return cache[key]

    def _build_dense_level(self):
        """The V-cycle from level L = coarse_level + 1 down (src/multigrid.py:330-344:
        pre-smoothing, residual, restriction with zeroed constrained rows, the coarse
        solve, masked prolongation, post-smoothing) is linear in r for a fixed setup:
        compose its dense map M_L once from the masked Jacobian, the Chebyshev
        polynomials of both blocks, the transfer matrix and the dense coarse maps,
        then every V-cycle applies z = M_L r in one launch."""
        self._dense_l = None
        L = self.coarse_level + 1
        if (not DENSE_LEVEL or self._dense is None or self.finest is None or self.finest < L
                or L not in self.states):
            return
        s = self.states[L]
        n = s.n_scalar
        if n > DENSE_LEVEL_NMAX:
            return
        dev = self._dense[1].device
        G = self._dense_jacobian(s)
        inv_u, inv_p = self._inv[L]
        cfg = self.cheb
        N = 3 * n
        hu = self.ranges[L]["uu"][1]
        hp = self.ranges[L]["phiphi"][1]
        Cu = self._cheb_poly(G[:2 * n, :2 * n], inv_u, cfg.c * hu, cfg.C * hu, cfg.sweeps)
        Cp = self._cheb_poly(G[2 * n:, 2 * n:], inv_p, cfg.c * hp, cfg.C * hp, cfg.sweeps)
        cons_np = s.constrained_mask()
        cons = torch.from_numpy(cons_np.astype(np.float64)).to(dev)
        ncons = torch.from_numpy((~cons_np).astype(np.float64)).to(dev)
        f64 = dict(dtype=torch.float64, device=dev)
        T = torch.empty((N, N), **f64)

        def smooth(R, Z):   # _smooth: u block on r - G z, then the phi row with the new z_u
            Tu = self._axpby(T[:2 * n], 0.0, R[:2 * n], 1.0)
            self._gemm(Tu, G[:2 * n], Z, -1.0, 1.0)
            self._gemm(Z[:2 * n], Cu, Tu, 1.0, 1.0)
            Tp = self._axpby(T[2 * n:], 0.0, R[2 * n:], 1.0)
            self._gemm(Tp, G[2 * n:], Z, -1.0, 1.0)
            self._gemm(Z[2 * n:], Cp, Tp, 1.0, 1.0)

        # the coarse level: transfer (scalar P per component) and the dense solve
        nc, Cu2, Gpu2, Cp2, cmask2 = self._dense
        P1, P1T = self._transfer_dense(L, dev)                    # (n, nc), (nc, n)
        cons2_np = self.states[self.coarse_level].constrained_mask()
        c2 = torch.from_numpy(cons2_np.astype(np.float64)).to(dev)
        nc2 = torch.from_numpy((~cons2_np).astype(np.float64)).to(dev)
        R = self._diagm(torch.empty((N, N), **f64))
        Z = self._diagm(torch.empty((N, N), **f64), cons)          # z = select(r)
        smooth(R, Z)                                               # first smoothing
        res = self._axpby(torch.empty((N, N), **f64), 0.0, R, 1.0)
        self._gemm(res, G, Z, -1.0, 1.0)                           # res = r - G z
        Rc = torch.empty((3 * nc, N), **f64)
        for k in range(3):
            self._gemm(Rc[k * nc:(k + 1) * nc], P1T, res[k * n:(k + 1) * n])
        self._axpby(Rc, 0.0, Rc, 1.0, nc2)                         # zero constrained coarse rows
        Zc = torch.empty((3 * nc, N), **f64)
        self._gemm(Zc[:2 * nc], Cu2, Rc[:2 * nc])
        Tc = self._axpby(torch.empty((nc, N), **f64), 0.0, Rc[2 * nc:], 1.0)
        self._gemm(Tc, Gpu2, Zc[:2 * nc], -1.0, 1.0)
        self._gemm(Zc[2 * nc:], Cp2, Tc)
        self._axpby(Zc, 0.0, Zc, 1.0, nc2)                         # constrained: zc = rc
        self._axpby(Zc, 1.0, Rc, 1.0, c2)
        Pz = torch.empty((N, N), **f64)
        for k in range(3):
            self._gemm(Pz[k * n:(k + 1) * n], P1, Zc[k * nc:(k + 1) * nc])
        self._axpby(Z, 1.0, Pz, 1.0, ncons)                        # masked prolongation
        smooth(R, Z)                                               # second smoothing
        self._dense_l = (L, N, Z)

    def _estimate_ranges(self, level: int):
        s = self.states[level]
        n = s.n_scalar
        cfg = self.cheb
        out = {}
        for block, mode, nb in (("uu", _lib.MODE_UU, 2 * n), ("phiphi", _lib.MODE_PHIPHI, n)):
            lo, hi = estimate_lambda_range(
                _BlockApply(s, mode, nb), self.diags[level][block],
                max_iterations=cfg.lanczos_iterations,
                seed=cfg.seed + 101 * level + (0 if block == "uu" else 1))
            hi = max(hi, 1e-30)
            lo = max(lo, cfg.lambda_min_floor * hi)
            out[block] = (lo, hi)
        return out

    def _estimate_ranges_batched(self, levels):
        """estimate_lambda_range for every (level, block) at once: the runs are
        independent, so each round launches the work of all active runs and
        synchronises once per reduction instead of once per run (identical
        per-run algebra: src/multigrid.py:123-162, 259-275)."""
        if NATIVE_LANCZOS:
            return self._estimate_ranges_native(levels)
        cfg = self.cheb
        runs = []
        for l in levels:
            s = self.states[l]
            n = s.n_scalar
            for blk, mode, nb in (("uu", _lib.MODE_UU, 2 * n), ("phiphi", _lib.MODE_PHIPHI, n)):
                runs.append(_LanczosRun(l, blk, _BlockApply(s, mode, nb), self.diags[l][blk],
                                        cfg.seed + 101 * l + (0 if blk == "uu" else 1),
                                        cfg.lanczos_iterations))
        R = len(runs)
        dev = runs[0].v.device
        partials = torch.empty(R * _lib.load().pff_reduce_scratch_len(), dtype=torch.float64,
                               device=dev)
        out = torch.empty(R, dtype=torch.float64, device=dev)
        plen = _lib.load().pff_reduce_scratch_len()
        st = stream_handle()
        while True:
            act = [i for i, r in enumerate(runs) if not r.done]
            if not act:
                break
            for i in act:
                runs[i].step_a()
                r = runs[i]
                call("pff_dot", r.n, ptr(r.v), ptr(r.w), ptr(partials[i * plen:]), ptr(out[i:]), st)
            alphas = out.cpu().numpy()
            for i in act:
                runs[i].step_b(float(alphas[i]), ritz=False)
                r = runs[i]
                call("pff_dot", r.n, ptr(r.w), ptr(r.w), ptr(partials[i * plen:]), ptr(out[i:]), st)
            _ritz_batched([runs[i] for i in act])
            norms2 = out.cpu().numpy()
            for i in act:
                runs[i].step_c(float(np.sqrt(norms2[i])))
        res = {}
        for r in runs:
            hi = max(r.hi, 1e-30)
            lo = max(r.lo, cfg.lambda_min_floor * hi)
            res.setdefault(r.level, {})[r.block] = (lo, hi)
        return res

    def _estimate_ranges_native(self, levels):
        """Same runs as the Python path, the loop inside libpff_b200."""
        cfg = self.cheb
        descs = []
        for l in levels:
            s = self.states[l]
            s._check_cache()
            n = s.n_scalar
            for blk, mode, nb in (("uu", _lib.MODE_UU, 2 * n), ("phiphi", _lib.MODE_PHIPHI, n)):
                diag = self.diags[l][blk]
                work = torch.empty(4 * nb, dtype=torch.float64, device=diag.device)
                work[:nb].copy_(start_vector_device(cfg.seed + 101 * l + (0 if blk == "uu" else 1),
                                                    nb, diag.device))
                descs.append((l, blk, s.bind(), mode, nb, _recip(diag, 1), work))
        R = len(descs)
        dev = descs[0][6].device
        plen = _lib.load().pff_reduce_scratch_len()
        partials = torch.empty(R * plen, dtype=torch.float64, device=dev)
        dots = torch.empty(2 * R, dtype=torch.float64, device=dev)   # alpha, beta^2 per run
        lo_hi = np.zeros(2 * R)
        arr = lambda ctype, vals: (ctype * R)(*vals)  # noqa: E731
        call("pff_lanczos_ranges", R, arr(ctypes.c_void_p, [d[2].value for d in descs]),
             arr(ctypes.c_int, [d[3] for d in descs]), arr(ctypes.c_int64, [d[4] for d in descs]),
             arr(ctypes.c_void_p, [d[5].data_ptr() for d in descs]),
             arr(ctypes.c_void_p, [d[6].data_ptr() for d in descs]), cfg.lanczos_iterations,
             lo_hi.ctypes.data, ptr(partials), ptr(dots), stream_handle())
        res = {}
        for r, d in enumerate(descs):
            hi = max(float(lo_hi[2 * r + 1]), 1e-30)
            lo = max(float(lo_hi[2 * r]), cfg.lambda_min_floor * hi)
            res.setdefault(d[0], {})[d[1]] = (lo, hi)
        return res

    # -- linear operator ---------------------------------------------------------
    def apply(self, r):
        """One V-cycle approximating G z = r from the finest level."""
        if self.finest is None:
            raise RuntimeError("setup() must run before apply()")
        x, was_np = op.as_device(r, 3 * self.states[self.finest].n_scalar)
        top = self._work[self.finest]
        top.r.copy_(x)
        self.run_cycle()
        return op.back(top.z.clone(), was_np)

    __call__ = apply
    _pff_device = True

    def run_cycle(self):
        """V-cycle from work[finest].r into work[finest].z (graph replay)."""
        top = self._work[self.finest]
        if not self.use_graph:
            self._vcycle(self.finest, top.r, top.z)
            return
        if self._graph is None:
            self._capture()
        self._graph.replay()

    def io_buffers(self):
        top = self._work[self.finest]
        return top.r, top.z

    def _capture(self):
        top = self._work[self.finest]
        # one eager pass before the first capture of this hierarchy shape in the
        # process: validates every launch and does the kernels' one-time setup
        # (shared-memory attributes, occupancy queries) outside capture
        key = (self.hierarchy.degree, self.finest, self.coarse_level,
               self.states[self.finest].split)
        dbg = os.environ.get("PFF_CAPTURE_DEBUG")
        t0 = time.perf_counter()
        eager = key not in _EAGER_DONE
        if eager:
            self._vcycle(self.finest, top.r, top.z)
            _EAGER_DONE.add(key)
        else:
            # later captures: only flush pending host->device syncs of the level
            # states (a host read of a state marks its mirror possibly modified)
            for s in self.states.values():
                s.bind()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        # capture_begin/end on a side stream directly: torch.cuda.graph's context
        # manager also empties the device and pinned-host allocator caches on entry
        # (5-45 ms here, and the freed blocks are re-allocated right after)
        g = torch.cuda.CUDAGraph()
        cs = _capture_stream()
        main = torch.cuda.current_stream()
        cs.wait_stream(main)
        tc = time.perf_counter()
        with torch.cuda.stream(cs):
            g.capture_begin(capture_error_mode="thread_local")
            try:
                self._vcycle(self.finest, top.r, top.z)
            finally:
                tr = time.perf_counter()
                g.capture_end()
        main.wait_stream(cs)
        self._graph = g
        if dbg:
            torch.cuda.synchronize()
            logger.warning("capture: %s %.1f ms, begin %.1f ms, record %.1f ms, end+instantiate %.1f ms",
                           "eager pass" if eager else "bind", (t1 - t0) * 1e3, (tc - t1) * 1e3,
                           (tr - tc) * 1e3, (time.perf_counter() - tr) * 1e3)

    # -- device V-cycle (src/multigrid.py:295-344) ---------------------------------
    def _cheb(self, l, mode, rhs, a, b, sweeps, out, assign, pre_d=False, d0_in_acc=False):
        s = self.states[l]
        W = self._work[l]
        nb = rhs.numel()
        inv = self._inv[l][0 if mode == _lib.MODE_UU else 1]
        d, cr = W.d[:nb], W.cr[:nb]
        # the smoothing increments accumulate straight into `out` (z += sum of the
        # Chebyshev updates; assign: z = sum) -- no separate accumulator pass
        acc = out
        theta, delta = 0.5 * (b + a), 0.5 * (b - a)
        sigma1 = theta / delta
        st = stream_handle()
        if pre_d:
            # the residual's producer already wrote d = D^-1 rhs / theta (pff_apply_emit,
            # pff_smooth_init); the first fused step adds it to acc ((acc + d) + d')
            assert sweeps > 1 and FUSE_CHEB and not assign
            h = s.bind()
            d_in, d_out = d, W.d2[:nb]
            src = rhs
            rho_old = 1.0 / sigma1
            skipped = False   # the previous step left acc alone
            for k in range(1, sweeps):
                rho = 1.0 / (2.0 * sigma1 - rho_old)
                if d0_in_acc:
                    # acc already holds d0: steps pair up from the end -- a step with an odd
                    # number of steps after it skips acc, the next adds both
                    if (sweeps - 1 - k) % 2 == 1:
                        fl, skipped = _lib.CHEB_NOACC, True
                    else:
                        fl, skipped = (_lib.CHEB_FIRST if skipped else 0), False
                else:
                    fl = _lib.CHEB_FIRST if k == 1 else 0
                fl |= _lib.CHEB_LAST if k == sweeps - 1 else 0
                call("pff_apply_cheb_ex", h, mode, ptr(d_in), ptr(d_out), ptr(src), ptr(cr),
                     ptr(inv), ptr(acc), rho * rho_old, 2.0 * rho / delta, fl, st)
                rho_old = rho
                src = cr
                d_in, d_out = d_out, d_in
            return
        call("pff_cheb_init", nb, ptr(inv), ptr(rhs), theta, ptr(d), ptr(acc), 0 if assign else 1,
             st)
        if sweeps > 1 and FUSE_CHEB:
            # each step: cr = (rhs | cr) - G d, d' = c1 d + c2 D^-1 cr, acc += d' in ONE
            # pass over the level (d ping-pongs between two buffers)
            h = s.bind()
            d_in, d_out = d, W.d2[:nb]
            src = rhs
            rho_old = 1.0 / sigma1
            for k in range(1, sweeps):
                rho = 1.0 / (2.0 * sigma1 - rho_old)
                call("pff_apply_cheb_ex", h, mode, ptr(d_in), ptr(d_out), ptr(src), ptr(cr),
                     ptr(inv), ptr(acc), rho * rho_old, 2.0 * rho / delta,
                     _lib.CHEB_LAST if k == sweeps - 1 else 0, st)
                rho_old = rho
                src = cr
                d_in, d_out = d_out, d_in
        elif sweeps > 1:
            s.apply_into(mode, d, cr, rhs)
            rho_old = 1.0 / sigma1
            for k in range(1, sweeps):
                rho = 1.0 / (2.0 * sigma1 - rho_old)
                call("pff_cheb_step", nb, ptr(inv), ptr(cr), rho * rho_old, 2.0 * rho / delta,
                     ptr(d), ptr(acc), st)
                rho_old = rho
                if k < sweeps - 1:
                    s.apply_into(mode, d, cr, cr)

    def _fused_init(self):
        return FUSE_CHEB and FUSE_INIT and self.cheb.sweeps > 1

    def _smooth(self, l, z, r, first=False):
        s = self.states[l]
        n = s.n_scalar
        W = self._work[l]
        if self._fused_init():
            # pff_cheb_init folded into the residual producers: d0 of the u block by
            # pff_smooth_init (first smoothing, z = 0 on entry) or the FULL residual,
            # d0 of the phi block by the phi-row residual (bitwise the same cycle)
            c, C = self.cheb.c, self.cheb.C
            hu = self.ranges[l]["uu"][1]
            hp = self.ranges[l]["phiphi"][1]
            th_u = 0.5 * (C * hu + c * hu)
            th_p = 0.5 * (C * hp + c * hp)
            inv_u, inv_p = self._inv[l]
            st = stream_handle()
            h = s.bind()
            defer = first and DEFER_ACC
            if first:
                call("pff_smooth_init_ex", h, ptr(r), ptr(z), ptr(W.res), ptr(inv_u), ptr(W.d), th_u,
                     _lib.SMOOTH_ADD_D0 if defer else 0, st)
            elif EMIT_FULL:
                call("pff_apply_emit", h, _lib.MODE_UU if POST_UU else _lib.MODE_FULL, ptr(z),
                     ptr(W.res), ptr(r), ptr(inv_u), ptr(W.d), th_u, st)
            elif POST_UU:
                s.apply_into(_lib.MODE_UU, z[:2 * n], W.res[:2 * n], r[:2 * n])
            else:
                s.apply_into(_lib.MODE_FULL, z, W.res, r)
            self._cheb(l, _lib.MODE_UU, W.res[:2 * n], c * hu, C * hu, self.cheb.sweeps, z[:2 * n],
                       False, pre_d=first or EMIT_FULL, d0_in_acc=defer)
            if EMIT_PHIROW:
                call("pff_apply_emit", h, _lib.MODE_PHIROW, ptr(z), ptr(W.resphi), ptr(r[2 * n:]),
                     ptr(inv_p), ptr(W.d), th_p, st)
            else:
                s.apply_into(_lib.MODE_PHIROW, z, W.resphi, r[2 * n:])
            self._cheb(l, _lib.MODE_PHIPHI, W.resphi, c * hp, C * hp, self.cheb.sweeps, z[2 * n:],
                       False, pre_d=EMIT_PHIROW)
            return
        if first:
            # z = SELECT(r): r - G z is r with the constrained rows zeroed, exactly
            # (identity rows/columns), so no operator application is needed
            call("pff_cons", s.bind(), _lib.LAYOUT_FULL, _lib.CONS_EXCLUDE, ptr(r), ptr(W.res),
                 stream_handle())
        elif POST_UU:
            s.apply_into(_lib.MODE_UU, z[:2 * n], W.res[:2 * n], r[:2 * n])
        else:
            s.apply_into(_lib.MODE_FULL, z, W.res, r)
        hi = self.ranges[l]["uu"][1]
        self._cheb(l, _lib.MODE_UU, W.res[:2 * n], self.cheb.c * hi, self.cheb.C * hi,
                   self.cheb.sweeps, z[:2 * n], False)
        s.apply_into(_lib.MODE_PHIROW, z, W.resphi, r[2 * n:])
        hi = self.ranges[l]["phiphi"][1]
        self._cheb(l, _lib.MODE_PHIPHI, W.resphi, self.cheb.c * hi, self.cheb.C * hi,
                   self.cheb.sweeps, z[2 * n:], False)

    def _coarse(self, l, r, z):
        s = self.states[l]
        n = s.n_scalar
        W = self._work[l]
        lo, hi = self.ranges[l]["uu"]
        self._cheb(l, _lib.MODE_UU, r[:2 * n], lo, self.cheb.C * hi, self.cheb.coarse_sweeps,
                   z[:2 * n], True)
        z[2 * n:].zero_()
        s.apply_into(_lib.MODE_PHIROW, z, W.resphi, r[2 * n:])
        lo, hi = self.ranges[l]["phiphi"]
        self._cheb(l, _lib.MODE_PHIPHI, W.resphi, lo, self.cheb.C * hi, self.cheb.coarse_sweeps,
                   z[2 * n:], True)
        call("pff_cons", s.bind(), _lib.LAYOUT_FULL, _lib.CONS_COPY, ptr(r), ptr(z),
             stream_handle())

    def _vcycle(self, l, r, z):
        if self._dense_l is not None and l == self._dense_l[0]:
            _, nn, M = self._dense_l
            call("pff_dense_matvec", nn, nn, ptr(M), ptr(r), ptr(z), stream_handle())
            return
        if l == self.coarse_level:
            if self._dense is not None:
                n, Cu, Gpu, Cp, cmask = self._dense
                call("pff_coarse_dense", n, ptr(Cu), ptr(Gpu), ptr(Cp), ptr(cmask), ptr(r), ptr(z),
                     stream_handle())
            else:
                self._coarse(l, r, z)
            return
        s, sc = self.states[l], self.states[l - 1]
        W, Wc = self._work[l], self._work[l - 1]
        st = stream_handle()
        if not self._fused_init():   # pff_smooth_init writes z = SELECT(r) itself
            call("pff_cons", s.bind(), _lib.LAYOUT_FULL, _lib.CONS_SELECT, ptr(r), ptr(z), st)
        self._smooth(l, z, r, first=True)
        s.apply_into(_lib.MODE_FULL, z, W.res, r)
        call("pff_restrict", s.bind(), sc.bind(), ptr(W.res), ptr(Wc.r), 1, st)
        self._vcycle(l - 1, Wc.r, Wc.z)
        call("pff_prolongate", s.bind(), sc.bind(), ptr(Wc.z), ptr(z), 1, st)
        self._smooth(l, z, r)
