"""Multi-GPU Newton-step solve: GMRES + GMG over cell-row slabs.

* Finest level: slab-partitioned (``parallel.SlabState``): operator family with
  NCCL ghost-row exchange, both block diagonals, Lanczos ranges (dots
  all-reduced, start vectors drawn globally with the reference's seeds, so the
  ranges equal the single-GPU ones up to rounding), Chebyshev smoothing.
* Restriction: every rank restricts its owned fine rows into a whole-mesh
  coarse vector; one all-reduce sums the partials (= the exact P^T).
* Coarser levels (ell-1 ... coarse_level): agglomerated -- every rank runs the
  single-GPU V-cycle of ``multigrid.GmgPreconditioner`` redundantly on the
  whole coarse mesh (1/4 of the fine work per level), then prolongates into
  its own fine rows.  Same algebra as src/multigrid.py:330-344.
* GMRES: right-preconditioned, restarted, reference Givens/back-substitution
  (src/krylov.py:37-119) with CGS2 orthogonalisation: two batched multi-dots
  (``pff_mdot``) and all-reduces per iteration instead of j+1 sequential MGS
  reductions (same iteration counts as MGS).

Ghost rows and non-owned slit copies of every Krylov / smoother vector are kept
at zero outside the operator's own exchange, so local dots are owned dots.
"""

from __future__ import annotations

import time

import numpy as np
import scipy.linalg
import torch
import torch.distributed as dist

from . import _lib
from ._lib import call, ptr, stream_handle
from .krylov import GmresResult, KrylovConfig
from .mesh import MeshHierarchy
from .multigrid import ChebyshevConfig, GmgPreconditioner
from .operator import LinearizationState
from .parallel import SlabPartition, SlabState

_NCOMP = {_lib.MODE_FULL: 3, _lib.MODE_UU: 2, _lib.MODE_PHIPHI: 1, _lib.MODE_PHIROW: 3}


class _Comm:
    def __init__(self, world: int, group=None):
        self.world, self.group = world, group

    def sum_(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            dist.all_reduce(t, group=self.group)
        return t


class DistributedGmg:
    """V-cycle with the finest level in slabs and agglomerated coarse levels."""

    def __init__(self, hierarchy: MeshHierarchy, level: int, rank: int, world: int,
                 coarse_level: int = 2, cheb: ChebyshevConfig | None = None, group=None,
                 device=None):
        if level - 1 < coarse_level:
            raise ValueError("need at least one level between the slab level and the coarse level")
        self.h, self.level, self.rank = hierarchy, level, rank
        self.part = SlabPartition(hierarchy.degree, level, world)
        self.comm = _Comm(world, group)
        self.group = group
        self.cheb = cheb or ChebyshevConfig()
        self.coarse_level = coarse_level
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self._scratch = torch.empty(_lib.load().pff_reduce_scratch_len(), dtype=torch.float64,
                                    device=self.device)
        self._dout = torch.empty(4, dtype=torch.float64, device=self.device)

    # -- vectors ----------------------------------------------------------------
    def _owned(self, ncomp: int) -> torch.Tensor:
        own = self.part.owned_mask(self.rank)
        return torch.from_numpy(np.tile(own, ncomp)).to(self.device)

    def dot(self, x: torch.Tensor, y: torch.Tensor) -> float:
        call("pff_dot", x.numel(), ptr(x), ptr(y), ptr(self._scratch), ptr(self._dout),
             stream_handle())
        return float(self.comm.sum_(self._dout[:1].clone()).item())

    def _axpby(self, a, x, b, y):
        call("pff_axpby", y.numel(), float(a), ptr(x), float(b), ptr(y), stream_handle())

    # -- setup -------------------------------------------------------------------
    def setup(self, params, split, U, phi_tilde, phi_old, active, dirichlet):
        """Global host arrays of the finest linearisation point (every rank)."""
        part, rank = self.part, self.rank
        self.fine = SlabState(part, rank, params, split, U, phi_tilde, active, dirichlet,
                              device=self.device, group=self.group)
        self.fine.refresh_cache()
        ln = self.fine.ln
        duu = torch.empty(2 * ln, dtype=torch.float64, device=self.device)
        dpp = torch.empty(ln, dtype=torch.float64, device=self.device)
        call("pff_diagonal", self.fine.handle(), ptr(duu), ptr(dpp), 0, stream_handle())
        own1, own2 = self._owned(1), self._owned(2)
        zero = torch.zeros((), dtype=torch.float64, device=self.device)
        self.diag = {"uu": torch.where(own2, duu, zero), "phiphi": torch.where(own1, dpp, zero)}
        self.inv = {k: torch.where(self._owned(2 if k == "uu" else 1), 1.0 / torch.where(
            d == 0, torch.ones_like(d), d), zero) for k, d in self.diag.items()}
        self.ranges = {"uu": self._lanczos(_lib.MODE_UU, "uu", 0),
                       "phiphi": self._lanczos(_lib.MODE_PHIPHI, "phiphi", 1)}
        # agglomerated coarse hierarchy: the whole level ell-1 on every rank
        inj = self.h.injection(self.level)
        n = part.n
        coarse = LinearizationState(self.h, self.level - 1, params, split=split)
        coarse.set_solution(np.concatenate([np.asarray(U)[k * n:(k + 1) * n][inj] for k in range(3)]))
        coarse.set_phi_tilde(np.asarray(phi_tilde)[inj])
        coarse.set_phi_old(np.asarray(phi_old)[inj])
        coarse.set_active(np.asarray(active)[inj])
        coarse._dir.set(torch.from_numpy(np.asarray(dirichlet)[inj]).to(self.device))
        coarse.refresh_cache()
        self.coarse_state = coarse
        self.cgmg = GmgPreconditioner(self.h, coarse_level=self.coarse_level, cheb=self.cheb)
        self.cgmg.setup(coarse)
        # work vectors (ghost rows stay zero)
        z = lambda k: torch.zeros(k * ln, dtype=torch.float64, device=self.device)  # noqa: E731
        self.w = dict(res=z(3), resphi=z(1), d=z(2), acc=z(2), cr=z(2), z=z(3))
        self.rc = torch.zeros(3 * coarse.n_scalar, dtype=torch.float64, device=self.device)

    def _lanczos(self, mode, block, blk_index):
        """estimate_lambda_range (src/multigrid.py:123-162) on the slab."""
        cfg, part = self.cheb, self.part
        diag = self.diag[block]
        ncomp = _NCOMP[mode] if mode != _lib.MODE_PHIROW else 1
        own = self._owned(ncomp)
        zero = torch.zeros((), dtype=torch.float64, device=self.device)
        dhalf = torch.where(own, 1.0 / torch.sqrt(torch.where(diag > 0, diag, torch.ones_like(diag))), zero)
        nglob = ncomp * part.n
        seed = cfg.seed + 101 * self.level + blk_index
        v_h = np.random.default_rng(seed).standard_normal(nglob)
        v_h /= np.linalg.norm(v_h)
        v = torch.from_numpy(part.scatter(v_h, self.rank, ncomp)).to(self.device) * own
        v_prev = torch.zeros_like(v)
        tmp = torch.zeros_like(v)
        w = torch.zeros_like(v)
        beta = 0.0
        alphas, betas = [], []
        lo = hi = 1.0
        prev = None
        for _ in range(min(cfg.lanczos_iterations, nglob)):
            torch.mul(dhalf, v, out=tmp)
            self.fine.apply_into(mode, tmp, w)
            self.fine.halo.zero_ghosts(tmp, ncomp)
            w.mul_(dhalf)
            self._axpby(-beta, v_prev, 1.0, w)
            alpha = self.dot(v, w)
            self._axpby(-alpha, v, 1.0, w)
            alphas.append(alpha)
            ritz = scipy.linalg.eigvalsh_tridiagonal(alphas, betas) if betas else np.array([alpha])
            lo, hi = float(ritz[0]), float(ritz[-1])
            beta = float(np.sqrt(self.dot(w, w)))
            if beta < 1e-12 * max(1.0, abs(hi)):
                break
            if prev is not None and abs(hi - prev) <= 1e-4 * abs(hi):
                break
            prev = hi
            betas.append(beta)
            v_prev, v = v, w.clone()
            v.div_(beta)
        hi = max(hi, 1e-30)
        lo = max(lo, cfg.lambda_min_floor * hi)
        return lo, hi

    # -- V-cycle -------------------------------------------------------------------
    def _cheb(self, mode, rhs, a, b, sweeps, out):
        block = "uu" if mode == _lib.MODE_UU else "phiphi"
        inv = self.inv[block]
        nb = rhs.numel()
        d, cr, acc = self.w["d"][:nb], self.w["cr"][:nb], self.w["acc"][:nb]
        theta, delta = 0.5 * (b + a), 0.5 * (b - a)
        sigma1 = theta / delta
        st = stream_handle()
        call("pff_cheb_init", nb, ptr(inv), ptr(rhs), theta, ptr(d), ptr(acc), 0, st)
        if sweeps > 1:
            self.fine.apply_into(mode, d, cr, rhs)
            rho_old = 1.0 / sigma1
            for k in range(1, sweeps):
                rho = 1.0 / (2.0 * sigma1 - rho_old)
                call("pff_cheb_step", nb, ptr(inv), ptr(cr), rho * rho_old, 2.0 * rho / delta,
                     ptr(d), ptr(acc), st)
                rho_old = rho
                if k < sweeps - 1:
                    self.fine.apply_into(mode, d, cr, cr)
        self._axpby(1.0, acc, 1.0, out)

    def _smooth(self, z, r, first=False):
        ln, W, c = self.fine.ln, self.w, self.cheb
        if first:   # z = SELECT(r): the residual is r with constrained rows zeroed
            call("pff_cons", self.fine.handle(), _lib.LAYOUT_FULL, _lib.CONS_EXCLUDE, ptr(r),
                 ptr(W["res"]), stream_handle())
        else:
            self.fine.apply_into(_lib.MODE_FULL, z, W["res"], r)
        hi = self.ranges["uu"][1]
        self._cheb(_lib.MODE_UU, W["res"][:2 * ln], c.c * hi, c.C * hi, c.sweeps, z[:2 * ln])
        self.fine.apply_into(_lib.MODE_PHIROW, z, W["resphi"], r[2 * ln:])
        hi = self.ranges["phiphi"][1]
        self._cheb(_lib.MODE_PHIPHI, W["resphi"], c.c * hi, c.C * hi, c.sweeps, z[2 * ln:])

    def apply_into(self, r: torch.Tensor, z: torch.Tensor):
        """z = V-cycle(r) on local slab vectors (src/multigrid.py:330-344)."""
        st = stream_handle()
        fh = self.fine.handle()
        call("pff_cons", fh, _lib.LAYOUT_FULL, _lib.CONS_SELECT, ptr(r), ptr(z), st)
        self._smooth(z, r, first=True)
        res = self.w["res"]
        self.fine.apply_into(_lib.MODE_FULL, z, res, r)
        ch = self.coarse_state.bind()
        call("pff_restrict", fh, ch, ptr(res), ptr(self.rc), 0, st)
        self.comm.sum_(self.rc)
        call("pff_cons", ch, _lib.LAYOUT_FULL, _lib.CONS_ZERO, None, ptr(self.rc), st)
        r_top, z_top = self.cgmg.io_buffers()
        r_top.copy_(self.rc)
        self.cgmg.run_cycle()
        call("pff_prolongate", fh, ch, ptr(z_top), ptr(z), 1, st)
        self._smooth(z, r)
        self.fine.halo.zero_ghosts(z, 3)
        return z

    def __call__(self, r):
        z = torch.zeros_like(r)
        return self.apply_into(r, z)


def distributed_gmres(gmg: DistributedGmg, rhs: torch.Tensor, config: KrylovConfig,
                      x0: torch.Tensor | None = None) -> GmresResult:
    """Right-preconditioned restarted GMRES on local slab vectors (src/krylov.py
    algebra; CGS2 orthogonalisation with two all-reduced multi-dots)."""
    t_start = time.perf_counter()
    fine = gmg.fine
    dev = rhs.device
    n = rhs.numel()
    b = rhs.clone()
    fine.halo.zero_ghosts(b, 3)
    st = stream_handle()
    x = torch.zeros_like(b) if x0 is None else x0.clone()
    b_norm = float(np.sqrt(gmg.dot(b, b)))
    target = max(config.relative_tolerance * b_norm, config.absolute_floor)
    r = b.clone()
    if x0 is not None:
        fine.apply_into(_lib.MODE_FULL, x, r, b)
    r_norm = float(np.sqrt(gmg.dot(r, r)))
    history = [r_norm]
    total = 0
    if r_norm <= target:
        return GmresResult(x, 0, history, True, time.perf_counter() - t_start)
    m_max = config.restart
    V = torch.zeros((m_max + 1, n), dtype=torch.float64, device=dev)
    parts = torch.empty((m_max + 1) * _lib.load().pff_reduce_scratch_len(), dtype=torch.float64,
                        device=dev)
    hbuf = torch.empty(m_max + 2, dtype=torch.float64, device=dev)
    zbuf = torch.zeros_like(b)
    upd = torch.zeros_like(b)
    while total < config.max_iterations:
        m = min(config.restart, config.max_iterations - total)
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        V.zero_()
        call("pff_div", n, ptr(r), None, r_norm, ptr(V[0]), st)
        g[0] = r_norm
        used = 0
        for j in range(m):
            z = gmg.apply_into(V[j], zbuf)
            w = V[j + 1]
            fine.apply_into(_lib.MODE_FULL, z, w)
            hcol = np.zeros(j + 2)
            for _ in range(2):   # CGS2
                call("pff_mdot", n, j + 1, ptr(V), n, ptr(w), ptr(parts), ptr(hbuf), st)
                h = gmg.comm.sum_(hbuf[: j + 1].clone())
                neg = -h
                call("pff_combine", n, j + 1, ptr(V), n, ptr(neg), ptr(w), 1, st)
                hcol[: j + 1] += h.cpu().numpy()
            h_next = float(np.sqrt(gmg.dot(w, w)))
            hcol[j + 1] = h_next
            H[: j + 2, j] = hcol
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
            history.append(abs(g[j + 1]))
            if abs(g[j + 1]) <= target:
                break
            if h_next <= 1e-14 * max(1.0, r_norm):
                break
            call("pff_div", n, ptr(w), None, h_next, ptr(w), st)
        y = np.zeros(used)
        for i in range(used - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1: used] @ y[i + 1:]) / H[i, i]
        ydev = torch.from_numpy(y).to(dev)
        call("pff_combine", n, used, ptr(V), n, ptr(ydev), ptr(upd), 0, st)
        corr = gmg.apply_into(upd, zbuf)
        call("pff_axpby", n, 1.0, ptr(corr), 1.0, ptr(x), st)
        r.copy_(b)
        fine.apply_into(_lib.MODE_FULL, x, r, b)
        fine.halo.zero_ghosts(x, 3)
        r_norm = float(np.sqrt(gmg.dot(r, r)))
        history[-1] = r_norm
        if r_norm <= target:
            return GmresResult(x, total, history, True, time.perf_counter() - t_start)
    return GmresResult(x, total, history, False, time.perf_counter() - t_start)
