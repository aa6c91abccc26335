"""Multi-GPU Newton-step solve: GMRES + GMG over cell-row slabs.

* Slab levels (the finest and every coarser level with >= 16 cell rows per
  rank): ``parallel.SlabState`` operator family with NCCL ghost-row exchange,
  both block diagonals, Lanczos ranges (dots all-reduced, start vectors drawn
  globally with the reference's seeds, so the ranges equal the single-GPU ones
  up to rounding), Chebyshev smoothing.
* Slab -> slab transfers: the restriction writes the coarse window and one
  reverse ghost-row message per neighbour completes the exact P^T; the
  prolongation reads the coarse window after a ghost-row exchange.
* Below the last slab level: agglomerated -- the restriction sums whole-mesh
  partial vectors with one all-reduce and every rank runs the single-GPU
  V-cycle of ``multigrid.GmgPreconditioner`` on that small level, then
  prolongates into its own rows.  Same algebra as src/multigrid.py:330-344.
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
FUSE_CHEB = True   # slab levels run the fused Chebyshev steps (pff_apply_cheb_ex)


class _Comm:
    def __init__(self, world: int, group=None):
        self.world, self.group = world, group

    def sum_(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            dist.all_reduce(t, group=self.group)
        return t


class _SlabLevel:
    """One slab level of the distributed V-cycle: window state, inverse block
    diagonals (zero off the owned rows), Chebyshev ranges and work vectors."""

    def __init__(self, part: SlabPartition, state: SlabState):
        self.part, self.st = part, state
        self.level = part.level


class DistributedGmg:
    """V-cycle over cell-row slabs on every level with at least ``min_rows``
    cell rows per rank (and >= 64^2 cells: the slab kernel is the Q2 sweep),
    agglomerated below that.

    Slab levels: operator family with ghost-row exchange, both block diagonals,
    Lanczos ranges with the reference's seeded global start vectors (so the
    ranges equal the single-GPU ones up to rounding), Chebyshev smoothing.
    Slab -> slab transfers are local: the restriction writes the coarse
    window (its top ghost row gets this rank's partial sums, which one reverse
    ghost-row message adds into the next rank's bottom owned row), the
    prolongation reads the coarse window after a ghost-row exchange.  Below
    the last slab level the restriction sums whole-mesh partial vectors with
    one all-reduce and every rank runs the single-GPU CUDA-graph V-cycle of
    ``GmgPreconditioner`` on that (small) level.  Same algebra as
    src/multigrid.py:330-344; the paper's distributed setting assigns each
    rank its part of every level.
    """

    def __init__(self, hierarchy: MeshHierarchy, level: int, rank: int, world: int,
                 coarse_level: int = 2, cheb: ChebyshevConfig | None = None, group=None,
                 device=None, min_rows: int = 16, max_slab_levels: int | None = None):
        if level - 1 < coarse_level:
            raise ValueError("need at least one level between the slab level and the coarse level")
        self.h, self.level, self.rank, self.world = hierarchy, level, rank, world
        self.comm = _Comm(world, group)
        self.group = group
        self.cheb = cheb or ChebyshevConfig()
        self.coarse_level = coarse_level
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self._scratch = torch.empty(_lib.load().pff_reduce_scratch_len(), dtype=torch.float64,
                                    device=self.device)
        self._dout = torch.empty(4, dtype=torch.float64, device=self.device)
        # slab levels: the finest always; coarser ones while each rank keeps
        # >= min_rows cell rows, the mesh stays on the sweep kernel (>= 64^2)
        # and a level remains below for the agglomerated V-cycle
        levels = [level]
        while True:
            l = levels[-1] - 1
            if max_slab_levels is not None and len(levels) >= max_slab_levels:
                break
            if l - 1 < coarse_level or 2 ** l < 64 or 2 ** l // world < max(min_rows, 2):
                break
            levels.append(l)
        self.slab_levels = levels
        self.agg_level = levels[-1] - 1
        self.part = SlabPartition(hierarchy.degree, level, world)

    @property
    def fine(self) -> SlabState:
        return self.lv[0].st

    # -- vectors ----------------------------------------------------------------
    def _owned(self, part: SlabPartition, ncomp: int) -> torch.Tensor:
        own = part.owned_mask(self.rank)
        return torch.from_numpy(np.tile(own, ncomp)).to(self.device)

    def dot(self, x: torch.Tensor, y: torch.Tensor) -> float:
        call("pff_dot", x.numel(), ptr(x), ptr(y), ptr(self._scratch), ptr(self._dout),
             stream_handle())
        return float(self.comm.sum_(self._dout[:1].clone()).item())

    def _axpby(self, a, x, b, y):
        call("pff_axpby", y.numel(), float(a), ptr(x), float(b), ptr(y), stream_handle())

    # -- setup -------------------------------------------------------------------
    def setup(self, params, split, U, phi_tilde, phi_old, active, dirichlet):
        """Global host arrays of the finest linearisation point (every rank);
        the coarser states are injected level by level (src/pff_operator.py:380-400)."""
        rank, h = self.rank, self.h
        U, pt, po = np.asarray(U), np.asarray(phi_tilde), np.asarray(phi_old)
        act, dirn = np.asarray(active), np.asarray(dirichlet)
        self.lv = []
        for k, l in enumerate(self.slab_levels + [self.agg_level]):
            if k > 0:   # inject the global state one level down
                inj = h.injection(l + 1)
                n = h.dof_map(l + 1).n_scalar
                U = np.concatenate([U[c * n:(c + 1) * n][inj] for c in range(3)])
                pt, po, act, dirn = pt[inj], po[inj], act[inj], dirn[inj]
            if l == self.agg_level:
                break
            part = SlabPartition(h.degree, l, self.world)
            st = SlabState(part, rank, params, split, U, pt, act, dirn, device=self.device,
                           group=self.group)
            st.refresh_cache()
            L = _SlabLevel(part, st)
            ln = st.ln
            duu = torch.empty(2 * ln, dtype=torch.float64, device=self.device)
            dpp = torch.empty(ln, dtype=torch.float64, device=self.device)
            call("pff_diagonal", st.handle(), ptr(duu), ptr(dpp), 0, stream_handle())
            own1, own2 = self._owned(part, 1), self._owned(part, 2)
            zero = torch.zeros((), dtype=torch.float64, device=self.device)
            L.diag = {"uu": torch.where(own2, duu, zero), "phiphi": torch.where(own1, dpp, zero)}
            L.inv = {k2: torch.where(self._owned(part, 2 if k2 == "uu" else 1), 1.0 / torch.where(
                d == 0, torch.ones_like(d), d), zero) for k2, d in L.diag.items()}
            z = lambda m: torch.zeros(m * ln, dtype=torch.float64, device=self.device)  # noqa: E731
            L.w = dict(res=z(3), resphi=z(1), d=z(2), d2=z(2), acc=z(2), cr=z(2), r=z(3), z=z(3))
            self.lv.append(L)
            L.ranges = {"uu": self._lanczos(L, _lib.MODE_UU, "uu", 0),
                        "phiphi": self._lanczos(L, _lib.MODE_PHIPHI, "phiphi", 1)}
        # agglomerated hierarchy below the last slab level: the whole mesh on every rank
        coarse = LinearizationState(h, self.agg_level, params, split=split)
        coarse.set_solution(U)
        coarse.set_phi_tilde(pt)
        coarse.set_phi_old(po)
        coarse.set_active(act)
        coarse._dir.set(torch.from_numpy(dirn).to(self.device))
        coarse.refresh_cache()
        self.coarse_state = coarse
        self.cgmg = GmgPreconditioner(h, coarse_level=self.coarse_level, cheb=self.cheb)
        self.cgmg.setup(coarse)
        self.rc = torch.zeros(3 * coarse.n_scalar, dtype=torch.float64, device=self.device)
        self.ranges = self.lv[0].ranges
        self.diag, self.inv, self.w = self.lv[0].diag, self.lv[0].inv, self.lv[0].w

    def _lanczos(self, L: _SlabLevel, mode, block, blk_index):
        """estimate_lambda_range (src/multigrid.py:123-162) on the slab."""
        cfg, part = self.cheb, L.part
        diag = L.diag[block]
        ncomp = _NCOMP[mode] if mode != _lib.MODE_PHIROW else 1
        own = self._owned(part, ncomp)
        zero = torch.zeros((), dtype=torch.float64, device=self.device)
        dhalf = torch.where(own, 1.0 / torch.sqrt(torch.where(diag > 0, diag, torch.ones_like(diag))), zero)
        nglob = ncomp * part.n
        seed = cfg.seed + 101 * L.level + blk_index
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
            L.st.apply_into(mode, tmp, w)
            L.st.halo.zero_ghosts(tmp, ncomp)
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
    def _cheb(self, L: _SlabLevel, mode, rhs, a, b, sweeps, out):
        block = "uu" if mode == _lib.MODE_UU else "phiphi"
        inv = L.inv[block]
        nb = rhs.numel()
        d, cr, acc = L.w["d"][:nb], L.w["cr"][:nb], L.w["acc"][:nb]
        theta, delta = 0.5 * (b + a), 0.5 * (b - a)
        sigma1 = theta / delta
        st = stream_handle()
        call("pff_cheb_init", nb, ptr(inv), ptr(rhs), theta, ptr(d), ptr(acc), 0, st)
        if sweeps > 1 and FUSE_CHEB:
            # each step in ONE sweep over the slab after the direction's ghost-row
            # exchange: cr = (rhs | cr) - G d, d' = c1 d + c2 D^-1 cr, acc += d'
            # (pff_apply_cheb_ex: the single-GPU cycle's fused form, bitwise the
            # unfused steps); d ping-pongs between two buffers
            ncomp = _NCOMP[mode]
            d_in, d_out = d, L.w["d2"][:nb]
            src = rhs
            rho_old = 1.0 / sigma1
            h = L.st.handle()
            for k in range(1, sweeps):
                rho = 1.0 / (2.0 * sigma1 - rho_old)
                L.st.halo.exchange(d_in, ncomp)
                call("pff_apply_cheb_ex", h, mode, ptr(d_in), ptr(d_out), ptr(src), ptr(cr),
                     ptr(inv), ptr(acc), rho * rho_old, 2.0 * rho / delta,
                     _lib.CHEB_LAST if k == sweeps - 1 else 0, st)
                rho_old = rho
                src = cr
                d_in, d_out = d_out, d_in
        elif sweeps > 1:
            L.st.apply_into(mode, d, cr, rhs)
            rho_old = 1.0 / sigma1
            for k in range(1, sweeps):
                rho = 1.0 / (2.0 * sigma1 - rho_old)
                call("pff_cheb_step", nb, ptr(inv), ptr(cr), rho * rho_old, 2.0 * rho / delta,
                     ptr(d), ptr(acc), st)
                rho_old = rho
                if k < sweeps - 1:
                    L.st.apply_into(mode, d, cr, cr)
        self._axpby(1.0, acc, 1.0, out)

    def _smooth(self, L: _SlabLevel, z, r, first=False):
        ln, W, c = L.st.ln, L.w, self.cheb
        if first:   # z = SELECT(r): the residual is r with constrained rows zeroed
            call("pff_cons", L.st.handle(), _lib.LAYOUT_FULL, _lib.CONS_EXCLUDE, ptr(r),
                 ptr(W["res"]), stream_handle())
        else:   # the u rows of r - G z alone (no u-phi block): 2 components exchanged, not 3
            L.st.apply_into(_lib.MODE_UU, z[:2 * ln], W["res"][:2 * ln], r[:2 * ln])
        hi = L.ranges["uu"][1]
        self._cheb(L, _lib.MODE_UU, W["res"][:2 * ln], c.c * hi, c.C * hi, c.sweeps, z[:2 * ln])
        L.st.apply_into(_lib.MODE_PHIROW, z, W["resphi"], r[2 * ln:])
        hi = L.ranges["phiphi"][1]
        self._cheb(L, _lib.MODE_PHIPHI, W["resphi"], c.c * hi, c.C * hi, c.sweeps, z[2 * ln:])

    def _vcycle(self, k: int, r: torch.Tensor, z: torch.Tensor):
        L = self.lv[k]
        st = stream_handle()
        fh = L.st.handle()
        call("pff_cons", fh, _lib.LAYOUT_FULL, _lib.CONS_SELECT, ptr(r), ptr(z), st)
        self._smooth(L, z, r, first=True)
        res = L.w["res"]
        L.st.apply_into(_lib.MODE_FULL, z, res, r)
        if k + 1 < len(self.lv):   # slab -> slab
            C = self.lv[k + 1]
            ch = C.st.handle()
            rc, zc = C.w["r"], C.w["z"]
            call("pff_restrict", fh, ch, ptr(res), ptr(rc), 0, st)
            C.st.halo.reverse_add(rc, 3)
            call("pff_cons", ch, _lib.LAYOUT_FULL, _lib.CONS_ZERO, None, ptr(rc), st)
            self._vcycle(k + 1, rc, zc)
            C.st.halo.exchange(zc, 3)   # the coarse ghost rows the prolongation reads
            call("pff_prolongate", fh, ch, ptr(zc), ptr(z), 1, st)
        else:   # slab -> agglomerated whole mesh
            ch = self.coarse_state.bind()
            call("pff_restrict", fh, ch, ptr(res), ptr(self.rc), 0, st)
            self.comm.sum_(self.rc)
            call("pff_cons", ch, _lib.LAYOUT_FULL, _lib.CONS_ZERO, None, ptr(self.rc), st)
            r_top, z_top = self.cgmg.io_buffers()
            r_top.copy_(self.rc)
            self.cgmg.run_cycle()
            call("pff_prolongate", fh, ch, ptr(z_top), ptr(z), 1, st)
        self._smooth(L, z, r)
        L.st.halo.zero_ghosts(z, 3)
        return z

    def apply_into(self, r: torch.Tensor, z: torch.Tensor):
        """z = V-cycle(r) on local slab vectors of the finest level
        (src/multigrid.py:330-344)."""
        return self._vcycle(0, r, z)

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
            # CGS2: both passes' coefficients and the new norm stay on the device
            # until ONE host read per iteration (all-reduces are stream-ordered)
            hsum = torch.zeros(j + 2, dtype=torch.float64, device=dev)
            for _ in range(2):
                call("pff_mdot", n, j + 1, ptr(V), n, ptr(w), ptr(parts), ptr(hbuf), st)
                h = gmg.comm.sum_(hbuf[: j + 1].clone())
                neg = -h
                call("pff_combine", n, j + 1, ptr(V), n, ptr(neg), ptr(w), 1, st)
                hsum[: j + 1] += h
            call("pff_dot", n, ptr(w), ptr(w), ptr(gmg._scratch), ptr(gmg._dout), st)
            hsum[j + 1] = gmg._dout[0]
            gmg.comm.sum_(hsum[j + 1:])
            hcol = hsum.cpu().numpy()
            h_next = float(np.sqrt(hcol[j + 1]))
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
