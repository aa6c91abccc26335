"""Run-to-run determinism of every device path (the reference is serial and
deterministic; its tests compare CSV output bitwise across runs).  The
generic kernels and the restriction use colour passes instead of atomics, the
sweep kernel writes every entry once, reductions use a fixed grid."""

import numpy as np
import pytest
import torch

from conftest import load_golden
import paper_2005_00331_b200 as P
from paper_2005_00331_b200 import _lib

pytestmark = pytest.mark.gpu


def state(p, level, split):
    d = load_golden(f"op_p{p}_l3_{split}") if (p != 2 and level == 3) else None
    h = P.build_hierarchy(max(level, 2), p)
    st = P.LinearizationState(h, level, P.MaterialParams(lame_lambda=121.15e3, mu=80.77e3,
                                                         g_c=2.7, kappa=1e-10,
                                                         eps=2.0 / 2 ** level), split=split)
    n = st.n_scalar
    rng = np.random.default_rng(3)
    phi0 = rng.uniform(0, 1, n)
    st.set_solution(np.concatenate([rng.uniform(-1e-3, 1e-3, 2 * n), phi0]))
    st.set_phi_tilde(phi0)
    st.set_phi_old(phi0)
    st.set_active(phi0 < 0.05)
    dm = h.dof_map(level)
    st.set_dirichlet_nodes(np.concatenate([dm.boundary_nodes["top"], dm.boundary_nodes["bottom"]]))
    st.refresh_cache()
    return h, st, rng.uniform(-1, 1, 3 * n), d


@pytest.mark.parametrize("p,level", [(1, 4), (2, 5), (3, 3), (4, 3), (2, 7)])
@pytest.mark.parametrize("split", ["none", "miehe"])
def test_operator_family_bitwise_repeatable(p, level, split):
    h, st, x, _ = state(p, level, split)
    n = st.n_scalar
    xd = torch.from_numpy(x).cuda()
    runs = []
    for _ in range(3):
        out = [P.apply_jacobian(st, xd), P.apply_block_uu(st, xd[:2 * n]),
               P.apply_block_phiphi(st, xd[2 * n:]), P.apply_phi_row(st, xd),
               *P.block_diagonals(st), P.residual(st, as_numpy=False)]
        runs.append([o.clone() for o in out])
    for r in runs[1:]:
        for a, b in zip(runs[0], r):
            assert torch.equal(a, b)


@pytest.mark.parametrize("p", [1, 2, 4])
def test_restriction_bitwise_repeatable(p):
    h = P.build_hierarchy(5, p)
    tr = P.TransferOperator(h, 5)
    y = np.random.default_rng(p).uniform(-1, 1, 3 * h.dof_map(5).n_scalar)
    a = tr.restrict(y)
    for _ in range(3):
        assert np.array_equal(tr.restrict(y), a)
    # and it is the transpose of the prolongation
    Pm = P.build_prolongation(h, 5)
    n, nc = h.dof_map(5).n_scalar, h.dof_map(4).n_scalar
    want = np.concatenate([Pm.T @ y[k * n:(k + 1) * n] for k in range(3)])
    assert np.abs(a - want).max() <= 1e-13 * np.abs(want).max()


def test_gmres_vcycle_bitwise_repeatable():
    h, st, x, _ = state(2, 6, "miehe")
    gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    gmg.setup(st)
    rhs = x.copy()
    rhs[st.constrained_mask()] = 0.0
    sols = []
    for _ in range(2):
        res = P.gmres_solve(P.JacobianOperator(st), torch.from_numpy(rhs).cuda(),
                            P.KrylovConfig(relative_tolerance=1e-8, restart=50),
                            preconditioner=gmg.apply)
        sols.append((res.iterations, res.solution.clone()))
    assert sols[0][0] == sols[1][0] and torch.equal(sols[0][1], sols[1][1])


@pytest.mark.parametrize("level,split", [(7, "miehe"), (7, "none"), (5, "miehe")])
def test_fused_chebyshev_vcycle_bitwise_equal(level, split):
    """pff_apply_cheb (Chebyshev steps fused into the block applications) gives
    the same bits as pff_apply + pff_cheb_step."""
    from paper_2005_00331_b200 import multigrid as MG
    h, st, x, _ = state(2, level, split)
    outs = []
    for fuse in (False, True):
        MG.FUSE_CHEB = fuse
        try:
            gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3),
                                      use_graph=False)
            gmg.setup(st)
            outs.append(gmg.apply(torch.from_numpy(x).cuda()).clone())
        finally:
            MG.FUSE_CHEB = True
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("level,split", [(7, "miehe"), (6, "none")])
def test_native_lanczos_matches_python_loop(level, split):
    """pff_lanczos_ranges (C++ loop, Sturm bisection) gives the ranges of the
    Python lockstep loop (scipy/numpy tridiagonal eigenvalues)."""
    from paper_2005_00331_b200 import multigrid as MG
    h, st, x, _ = state(2, level, split)
    out = []
    for native in (False, True):
        MG.NATIVE_LANCZOS = native
        try:
            gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
            gmg.setup(st)
            out.append(gmg.ranges)
        finally:
            MG.NATIVE_LANCZOS = True
    for l, blocks in out[0].items():
        for blk, (lo, hi) in blocks.items():
            lo2, hi2 = out[1][l][blk]
            assert hi2 == pytest.approx(hi, rel=1e-12) and lo2 == pytest.approx(lo, rel=1e-11), (l, blk)
