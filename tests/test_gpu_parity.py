"""Parity of the CUDA path (libpff_b200.so through the drop-in API) against
the reference's golden vectors and the CPU oracle.  GPU only.

Bar (BASELINE.json north star): fp64 operator and V-cycle outputs within
1e-12 relative L2 PER BLOCK (u_x, u_y, phi), GMRES iterations within +-1.
"""

import glob
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN, block_rel, load_golden, rel_l2
import paper_2005_00331_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-12


def product_state(d, split):
    p, level = int(d["meta"][0]), int(d["meta"][1])
    h = P.build_hierarchy(max(level, 2), p)
    st = P.LinearizationState(h, level, O.baseline_material(level), split=split)
    st.set_solution(d["U"])
    st.set_phi_tilde(d["phi_tilde"])
    st.set_phi_old(d["phi_old"])
    st.set_active(d["active"])
    st.set_dirichlet_nodes(np.flatnonzero(d["dirichlet"]))
    st.refresh_cache()
    return st


def oracle_state(d, split):
    p, level = int(d["meta"][0]), int(d["meta"][1])
    st = O.State(p, level, O.baseline_material(level), split)
    st.U, st.phi_tilde, st.phi_old = d["U"].copy(), d["phi_tilde"].copy(), d["phi_old"].copy()
    st.active, st.dirichlet = d["active"].copy(), d["dirichlet"].copy()
    st.refresh_cache()
    return st


OP_CASES = sorted(os.path.basename(f)[:-4] for f in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if os.path.basename(f).startswith(("pr1_", "op_")))


@pytest.mark.parametrize("name", OP_CASES)
def test_operator_family_vs_golden(name):
    d = load_golden(name)
    split = "miehe" if int(d["meta"][3]) else "none"
    st = product_state(d, split)
    n = st.n_scalar
    x = d["x"]
    assert max(block_rel(P.apply_jacobian(st, x), d["jac"], n)) <= TOL
    assert max(block_rel(P.apply_block_uu(st, x[:2 * n]), d["uu"], n)) <= TOL
    assert rel_l2(P.apply_block_phiphi(st, x[2 * n:]), d["pp"]) <= TOL
    assert rel_l2(P.apply_phi_row(st, x), d["prow"]) <= TOL
    assert max(block_rel(P.block_diagonal(st, "uu"), d["diag_uu"], n)) <= TOL
    assert rel_l2(P.block_diagonal(st, "phiphi"), d["diag_pp"]) <= TOL
    r = P.residual(st)
    for k, v in enumerate(block_rel(r, d["residual"], n)):
        assert v <= TOL or np.abs(d["residual"][k * n:(k + 1) * n]).max() == 0.0
    assert max(block_rel(P.residual(st, mask_dirichlet=False), d["residual_raw"], n)) <= TOL


@pytest.mark.parametrize("split", ["none", "miehe"])
def test_cache_vs_golden(split):
    d = load_golden(f"pr1_{split}")
    st = product_state(d, split)
    c = st.cache()
    for k in ("e11", "e22", "e12", "gt", "dg", "pc"):
        got = c[k].contiguous().cpu().numpy().ravel()
        assert rel_l2(got, d["cache_" + k]) <= TOL, k


def test_identity_rows_and_columns():
    d = load_golden("pr1_miehe")
    st = product_state(d, "miehe")
    n3 = 3 * st.n_scalar
    mask = st.constrained_mask()
    cdofs = np.flatnonzero(mask)
    rng = np.random.default_rng(13)
    v = rng.standard_normal(n3)
    out = P.apply_jacobian(st, v)
    assert np.array_equal(out[cdofs], v[cdofs])
    for i in cdofs[:4]:
        e = np.zeros(n3)
        e[i] = 1.0
        col = P.apply_jacobian(st, e)
        assert col[i] == 1.0
        col[i] = 0.0
        assert np.all(col == 0.0)
    assert np.all(P.apply_jacobian(st, np.zeros(n3)) == 0.0)


def test_stale_cache_raises():
    d = load_golden("pr1_none")
    st = product_state(d, "none")
    st.set_solution(st.U * 1.01)
    with pytest.raises(P.StaleCacheError):
        P.apply_jacobian(st, np.zeros(3 * st.n_scalar))


def test_fused_residual_form():
    d = load_golden("pr1_miehe")
    st = product_state(d, "miehe")
    n = st.n_scalar
    x = torch.from_numpy(d["x"]).cuda()
    r = torch.from_numpy(np.random.default_rng(3).standard_normal(3 * n)).cuda()
    out = torch.empty_like(r)
    st.apply_into(0, x, out, r)
    want = d["x"] * 0 + r.cpu().numpy() - d["jac"]
    assert max(block_rel(out.cpu().numpy(), want, n)) <= TOL
    r2 = r.clone()
    st.apply_into(0, x, r2, r2)   # dst aliases rhs
    assert max(block_rel(r2.cpu().numpy(), out.cpu().numpy(), n)) <= 1e-15


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_transfers_vs_golden(p):
    d = load_golden(f"transfer_p{p}_l4")
    tr = P.TransferOperator(P.build_hierarchy(4, p), 4)
    assert rel_l2(tr.prolongate(d["xc"]), d["Px"]) <= 1e-14
    assert rel_l2(tr.restrict(d["yf"]), d["Ry"]) <= 1e-14


def test_transfer_level1():
    d = load_golden("transfer_p2_l1")
    tr = P.TransferOperator(P.build_hierarchy(2, 2), 1)
    assert rel_l2(tr.prolongate(d["xc"]), d["Px"]) <= 1e-14
    assert rel_l2(tr.restrict(d["yf"]), d["Ry"]) <= 1e-14


def test_restrict_state_vs_golden():
    d = load_golden("restrict_p2_l5_l2")
    st = product_state(dict(d, meta=np.array([2, 5, 0, 1])), "miehe")
    c = P.restrict_state_to_level(st, 2)
    assert np.array_equal(c.U, d["cU"])
    assert np.array_equal(c.phi_tilde, d["cphi_tilde"])
    assert np.array_equal(c.active, d["cactive"])
    assert np.array_equal(c.dirichlet_nodes, d["cdirichlet"])


SOLVE_CASES = sorted(os.path.basename(f)[:-4] for f in glob.glob(os.path.join(GOLDEN, "solve_*.npz")))


@pytest.mark.parametrize("name", SOLVE_CASES)
def test_solver_stack_vs_golden(name):
    d = load_golden(name)
    p, level, seed, miehe, notch, sweeps = (int(v) for v in d["meta"])
    split = "miehe" if miehe else "none"
    st = product_state(dict(d, meta=np.array([p, level, seed, miehe])), split)
    n = st.n_scalar
    gmg = P.GmgPreconditioner(st.hierarchy, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=sweeps))
    gmg.setup(st)
    for l in range(2, level + 1):
        got = gmg.ranges[l]
        assert np.allclose([got["uu"][0], got["uu"][1], got["phiphi"][0], got["phiphi"][1]],
                           d[f"range_{l}"], rtol=1e-10, atol=0), l
    z = gmg.apply(d["x"])
    assert max(block_rel(z, d["vcycle"], n)) <= TOL
    # same cycle without the CUDA graph
    gmg.use_graph = False
    assert max(block_rel(gmg.apply(d["x"]), z, n)) <= 1e-14
    gmg.use_graph = True
    # the matrix-free coarse solve (the reference's Chebyshev passes) agrees
    # with the dense-map coarse solve (pff_coarse_dense) and with the golden
    from paper_2005_00331_b200 import multigrid as MG
    assert gmg._dense is not None
    MG.DENSE_COARSE = False
    try:
        gmg2 = P.GmgPreconditioner(st.hierarchy, coarse_level=2,
                                   cheb=P.ChebyshevConfig(sweeps=sweeps))
        gmg2.setup(st)
        assert gmg2._dense is None
        z2 = gmg2.apply(d["x"])
    finally:
        MG.DENSE_COARSE = True
    assert max(block_rel(z2, d["vcycle"], n)) <= TOL
    assert max(block_rel(z2, z, n)) <= 1e-13
    hi = gmg.ranges[level]["uu"][1]
    cheb = P.chebyshev_apply(lambda v: P.apply_block_uu(st, v), gmg.diags[level]["uu"].cpu().numpy(),
                             d["x"][:2 * n], 0.24 * hi, 1.2 * hi, 5)
    assert max(block_rel(cheb, d["cheb_uu"], n)) <= TOL
    lz = P.estimate_lambda_range(lambda v: P.apply_block_uu(st, v),
                                 gmg.diags[level]["uu"].cpu().numpy(), seed=7)
    assert np.allclose(lz, d["lanczos_uu"], rtol=1e-10, atol=0)
    rhs = d["x"].copy()
    rhs[st.constrained_mask()] = 0.0
    res = P.gmres_solve(P.JacobianOperator(st), rhs,
                        P.KrylovConfig(relative_tolerance=1e-8, restart=50),
                        preconditioner=gmg.apply)
    assert res.converged == bool(d["gmres_conv"][0])
    assert abs(res.iterations - int(d["gmres_iters"][0])) <= 1
    assert max(block_rel(res.solution, d["gmres_x"], n)) <= 1e-8
    # reference-style closures give the same answer
    res2 = P.gmres_solve(lambda v: P.apply_jacobian(st, v), rhs,
                         P.KrylovConfig(relative_tolerance=1e-8, restart=50),
                         preconditioner=gmg.apply)
    assert res2.iterations == res.iterations


@pytest.mark.parametrize("split", ["none", "miehe"])
@pytest.mark.parametrize("p,level", [(2, 10), (4, 9)])
def test_full_size_vs_oracle(split, p, level):
    """BASELINE configs[1] / configs[2] at full size against the C oracle."""
    ost, x = O.baseline_state(p, level, split, seed=0)
    ost.refresh_cache(nthreads=O.max_threads())
    want = O.apply_jacobian(ost, x, nthreads=O.max_threads())
    h = P.build_hierarchy(level, p)
    st = P.LinearizationState(h, level, ost.params, split=split)
    st.set_solution(ost.U)
    st.set_phi_tilde(ost.phi_tilde)
    st.set_phi_old(ost.phi_old)
    st.set_active(ost.active)
    st.set_dirichlet_nodes(np.flatnonzero(ost.dirichlet))
    st.refresh_cache()
    got = P.apply_jacobian(st, x)
    n = st.n_scalar
    assert max(block_rel(got, want, n)) <= TOL
    # linearity on device at full size (size-independent property)
    xd = torch.from_numpy(x).cuda()
    y1 = P.apply_jacobian(st, xd)
    y2 = P.apply_jacobian(st, 2.0 * xd)
    assert rel_l2((y2 - 2.0 * y1).cpu().numpy() + 2.0 * y1.cpu().numpy(),
                  2.0 * y1.cpu().numpy()) <= 1e-14


def test_gmres_small_dense_numpy_callables():
    """The reference's own Krylov tests drive gmres with numpy callables."""
    rng = np.random.default_rng(1)
    A = rng.standard_normal((5, 5)) + 5 * np.eye(5)
    b = rng.standard_normal(5)
    res = P.gmres_solve(lambda v: A @ v, b, P.KrylovConfig(relative_tolerance=1e-12))
    assert res.converged and res.iterations <= 5
    assert np.linalg.norm(A @ res.solution - b) <= 1e-10 * np.linalg.norm(b)
    d = np.arange(1.0, 11.0)
    res = P.gmres_solve(lambda v: d * v, np.ones(10), P.KrylovConfig(),
                        preconditioner=lambda v: v / d)
    assert res.converged and res.iterations == 1
    res = P.gmres_solve(lambda v: v, rng.standard_normal(20), P.KrylovConfig())
    assert res.converged and res.iterations == 1


def test_lanczos_and_chebyshev_numpy_callables():
    n = 50
    dd = np.arange(1.0, n + 1)
    got = P.estimate_lambda_max(lambda v: dd * v, np.ones(n), seed=2)
    assert abs(got - n) <= 0.05 * n
    lo, hi = P.estimate_lambda_range(lambda v: 3.0 * v, np.ones(8), seed=4)
    assert hi == pytest.approx(3.0, abs=1e-9) and lo == pytest.approx(3.0, abs=1e-9)
    rhs = np.random.default_rng(0).standard_normal(25)
    z = P.chebyshev_apply(lambda v: v, np.ones(25), rhs, 1.0, 1.2, 32)
    assert np.linalg.norm(z - rhs) <= 1e-13 * np.linalg.norm(rhs)


@pytest.fixture
def generic_apply():
    from paper_2005_00331_b200 import _lib
    def run(flag):
        _lib.set_option(_lib.OPT_GENERIC_APPLY, int(flag))
    yield run
    _lib.set_option(_lib.OPT_GENERIC_APPLY, 0)
    _lib.set_option(_lib.OPT_SWEEP_ROWS, 0)


@pytest.mark.parametrize("split", ["none", "miehe"])
@pytest.mark.parametrize("level,rows", [(1, 0), (5, 3), (6, 1), (6, 31), (7, 5), (7, 64),
                                        (8, 64), (8, 7), (9, 0), (9, 256)])
def test_sweep_matches_generic_all_modes(generic_apply, split, level, rows):
    """The write-once Q2 kernel against the per-cell atomic kernel, every mode,
    plain and fused, over chunkings that put chunk edges on and off the slit."""
    from paper_2005_00331_b200 import _lib
    ost, x = O.baseline_state(2, level, split, seed=level)
    h = P.build_hierarchy(max(level, 2), 2)
    st = P.LinearizationState(h, level, ost.params, split=split)
    st.set_solution(ost.U)
    st.set_phi_tilde(ost.phi_tilde)
    st.set_phi_old(ost.phi_old)
    act = ost.active.copy()
    act[np.random.default_rng(level).choice(st.n_scalar, 7, replace=False)] = True
    dn = ost.dirichlet.copy()
    dn[h.dof_map(level).slit_upper[:2]] = True
    st.set_active(act)
    st.set_dirichlet_nodes(np.flatnonzero(dn))
    st.refresh_cache()
    n = st.n_scalar
    xd = torch.from_numpy(x).cuda()
    rhs = torch.from_numpy(np.random.default_rng(1).standard_normal(3 * n)).cuda()
    _lib.set_option(_lib.OPT_SWEEP_ROWS, rows)
    cases = [(0, xd, 3 * n), (1, xd[:2 * n], 2 * n), (2, xd[2 * n:], n), (3, xd, n)]
    for mode, src, nout in cases:
        outs = []
        for flag in (1, 0):
            generic_apply(flag)
            y = torch.empty(nout, dtype=torch.float64, device="cuda")
            st.apply_into(mode, src, y)
            yf = torch.empty(nout, dtype=torch.float64, device="cuda")
            st.apply_into(mode, src, yf, rhs[:nout])
            outs.append((y.cpu().numpy(), yf.cpu().numpy()))
        (g, gf), (s, sf) = outs
        k = nout // n
        assert max(block_rel(s, g, n)) <= 1e-13, (mode, block_rel(s, g, n))
        assert max(block_rel(sf, gf, n)) <= 1e-13, mode
    generic_apply(0)
    if level >= 6:   # the write-once sweep kernel runs from 64x64 cells up: deterministic
        y1 = P.apply_jacobian(st, xd)
        y2 = P.apply_jacobian(st, xd)
        assert torch.equal(y1, y2)


REGIMES = {
    # affine displacement fields u = (a x + b y, c x + d y): one strain regime on every q-point
    "zero": (0.0, 0.0, 0.0, 0.0),                   # e = 0: degenerate gap, tr e = 0
    "near_biaxial_tension": (1e-3, 0.0, 0.0, 1e-3 * (1 + 1e-6)),    # gap 1e-9: resolved
    "biaxial_compression": (-1e-3, 0.0, 0.0, -1e-3),  # ev1 = ev2 < 0: sigma+ = 0 in any frame
    "uniaxial_tension": (1e-3, 0.0, 0.0, -3e-4),    # mixed signs, tr e > 0
    "uniaxial_compression": (3e-4, 0.0, 0.0, -1e-3),  # mixed signs, tr e < 0
    "shear_tr_pos": (1e-5, 1e-3, 1e-3, 0.0),        # ev ~ +-|e12|, tr e > 0
    "shear_tr_neg": (0.0, 1e-3, 0.0, -1e-5),        # simple shear, tr e < 0
    "tension_tension": (1e-3, 2e-4, -1e-4, 4e-4),   # both eigenvalues > 0, distinct
    "compression_compression": (-1e-3, 2e-4, -1e-4, -4e-4),
}


@pytest.mark.parametrize("regime", sorted(REGIMES))
def test_sweep_miehe_regimes_vs_oracle(regime):
    """The Q2 sweep kernel's eigen-frame Miehe tile (regime in the sign bits of g and gamma)
    against the C oracle on states that hold ONE strain regime everywhere, including the
    zero state and equal compressive eigenvalues (src/_kernels.py:50-74,102-123).  Not
    here: states where the reference's own branches are decided by round-off -- tr e = 0
    up to rounding (pure shear: `tre < 0` flips) or ev1 = ev2 > 0 up to rounding (the
    eigen-frame of _dpos2s is noise and its off-diagonal term is dropped below the gap
    threshold, so the result depends on that frame); the oracle and any device kernel
    (the round-1 symmetric-tangent form included) differ there by O(1)."""
    level = 6
    ost, x = O.baseline_state(2, level, "miehe", seed=3)
    a, b, c, d = REGIMES[regime]
    xy = ost.lv.coords()
    n = ost.n
    ost.U[:n] = a * xy[:, 0] + b * xy[:, 1]
    ost.U[n:2 * n] = c * xy[:, 0] + d * xy[:, 1]
    ost.refresh_cache(nthreads=O.max_threads())
    h = P.build_hierarchy(level, 2)
    st = P.LinearizationState(h, level, ost.params, split="miehe")
    st.set_solution(ost.U)
    st.set_phi_tilde(ost.phi_tilde)
    st.set_phi_old(ost.phi_old)
    st.set_active(ost.active)
    st.set_dirichlet_nodes(np.flatnonzero(ost.dirichlet))
    st.refresh_cache()
    assert st.uses_sweep_kernel()
    nt = O.max_threads()
    assert max(block_rel(P.apply_jacobian(st, x), O.apply_jacobian(ost, x, nthreads=nt), n)) <= TOL
    assert max(block_rel(P.apply_block_uu(st, x[:2 * n]),
                         O.apply_block_uu(ost, x[:2 * n], nthreads=nt), n)) <= TOL
    assert rel_l2(P.apply_phi_row(st, x), O.apply_phi_row(ost, x, nthreads=nt)) <= TOL


@pytest.mark.parametrize("split", ["miehe", "none"])
@pytest.mark.parametrize("level,rows", [(6, 0), (7, 5), (8, 0), (9, 64)])
def test_sweep_column_ring_matches_row_stages_bitwise(split, level, rows):
    """Both stagings of the tangent block (the single-buffered Gauss-column ring and the two
    whole-row stages) run the same arithmetic: every mode, plain, fused and the fused
    Chebyshev step, bit for bit."""
    from paper_2005_00331_b200 import _lib
    ost, x = O.baseline_state(2, level, split, seed=level + 1)
    h = P.build_hierarchy(level, 2)
    st = P.LinearizationState(h, level, ost.params, split=split)
    st.set_solution(ost.U); st.set_phi_tilde(ost.phi_tilde); st.set_phi_old(ost.phi_old)
    st.set_active(ost.active)
    st.set_dirichlet_nodes(np.flatnonzero(ost.dirichlet))
    st.refresh_cache()
    assert st.uses_sweep_kernel()
    n = st.n_scalar
    xd = torch.from_numpy(x).cuda()
    g = torch.Generator(device="cuda").manual_seed(level)
    rhs = torch.rand(3 * n, dtype=torch.float64, device="cuda", generator=g)
    invd = torch.rand(2 * n, dtype=torch.float64, device="cuda", generator=g) + 0.5
    acc0 = torch.rand(2 * n, dtype=torch.float64, device="cuda", generator=g)
    outs = []
    try:
        _lib.set_option(_lib.OPT_SWEEP_ROWS, rows)
        for ring in (0, 1):
            _lib.set_option(_lib.OPT_SWEEP_COLRING, ring)
            res = []
            for mode, src, nout in ((0, xd, 3 * n), (1, xd[:2 * n], 2 * n), (2, xd[2 * n:], n),
                                    (3, xd, n)):
                y = torch.empty(nout, dtype=torch.float64, device="cuda")
                st.apply_into(mode, src, y)
                yf = torch.empty(nout, dtype=torch.float64, device="cuda")
                st.apply_into(mode, src, yf, rhs[:nout])
                res += [y, yf]
            # one fused Chebyshev step on the u block (cr, d', acc)
            cr = torch.empty(2 * n, dtype=torch.float64, device="cuda")
            dn = torch.empty(2 * n, dtype=torch.float64, device="cuda")
            acc = acc0.clone()
            _lib.call("pff_apply_cheb_ex", st.bind(), _lib.MODE_UU, _lib.ptr(xd[:2 * n].contiguous()),
                      _lib.ptr(dn), _lib.ptr(rhs[:2 * n].contiguous()), _lib.ptr(cr), _lib.ptr(invd),
                      _lib.ptr(acc), 0.3, 0.7, _lib.CHEB_FIRST, _lib.stream_handle())
            res += [cr, dn, acc]
            outs.append([t.clone() for t in res])
    finally:
        _lib.set_option(_lib.OPT_SWEEP_COLRING, -1)
        _lib.set_option(_lib.OPT_SWEEP_ROWS, 0)
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("split", ["miehe", "none"])
@pytest.mark.parametrize("level", [6, 9])
def test_pipelined_host_path_matches_device_path(split, level):
    """apply_* with a pinned host tensor runs the chunked H2D/compute/D2H
    pipeline (pff_apply_host); results must equal the device path exactly."""
    ost, x = O.baseline_state(2, level, split, seed=11)
    h = P.build_hierarchy(level, 2)
    st = P.LinearizationState(h, level, ost.params, split=split)
    st.set_solution(ost.U); st.set_phi_tilde(ost.phi_tilde); st.set_active(ost.active)
    st.set_dirichlet_nodes(np.flatnonzero(ost.dirichlet))
    st.refresh_cache()
    n = st.n_scalar
    xh = torch.from_numpy(x).pin_memory()
    xd = xh.cuda()
    for fn, sl in ((P.apply_jacobian, slice(0, 3 * n)), (P.apply_block_uu, slice(0, 2 * n)),
                   (P.apply_block_phiphi, slice(2 * n, 3 * n)), (P.apply_phi_row, slice(0, 3 * n))):
        got = fn(st, xh[sl].contiguous().pin_memory())
        assert not got.is_cuda
        want = fn(st, xd[sl].contiguous())
        assert torch.equal(got, want.cpu())

@pytest.mark.parametrize("nchunks", [1, 2, 7, 64])
def test_apply_host_chunkings(nchunks):
    """pff_apply_host with equal chunkings (one chunk, two, odd, the maximum
    64 on a 64-row level: one cell row each) equals the device path per mode."""
    from paper_2005_00331_b200 import operator as OP
    from paper_2005_00331_b200 import _lib
    ost, x = O.baseline_state(2, 6, "miehe", seed=12)
    h = P.build_hierarchy(6, 2)
    st = P.LinearizationState(h, 6, ost.params, split="miehe")
    st.set_solution(ost.U); st.set_phi_tilde(ost.phi_tilde); st.set_active(ost.active)
    st.set_dirichlet_nodes(np.flatnonzero(ost.dirichlet))
    st.refresh_cache()
    n = st.n_scalar
    xd = torch.from_numpy(x).cuda()
    for mode, sl, nout in ((_lib.MODE_FULL, slice(0, 3 * n), 3 * n), (_lib.MODE_UU, slice(0, 2 * n), 2 * n),
                           (_lib.MODE_PHIPHI, slice(2 * n, 3 * n), n), (_lib.MODE_PHIROW, slice(0, 3 * n), n)):
        got = OP._pipelined(st, mode, xd[sl].cpu().contiguous().pin_memory(), nchunks)
        want = torch.empty(nout, dtype=torch.float64, device="cuda")
        st.apply_into(mode, xd[sl].contiguous(), want)
        assert torch.equal(got, want.cpu()), mode


def test_apply_host_pageable_buffers():
    """pff_apply_host on pageable (numpy) host buffers: the copies are staged by
    the driver instead of overlapped, the result is the same bit for bit."""
    import ctypes
    from paper_2005_00331_b200 import _lib
    ost, x = O.baseline_state(2, 6, "none", seed=13)
    h = P.build_hierarchy(6, 2)
    st = P.LinearizationState(h, 6, ost.params, split="none")
    st.set_solution(ost.U); st.set_phi_tilde(ost.phi_tilde); st.set_active(ost.active)
    st.set_dirichlet_nodes(np.flatnonzero(ost.dirichlet))
    st.refresh_cache()
    n = st.n_scalar
    xh = np.ascontiguousarray(x, dtype=np.float64)
    yh = np.zeros(3 * n)
    xd = torch.empty(3 * n, dtype=torch.float64, device="cuda")
    yd = torch.empty(3 * n, dtype=torch.float64, device="cuda")
    L = _lib.load()
    s = torch.cuda.current_stream()
    assert L.pff_apply_host(st.bind(), _lib.MODE_FULL, xh.ctypes.data_as(ctypes.c_void_p),
                            yh.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(xd.data_ptr()),
                            ctypes.c_void_p(yd.data_ptr()), 5, ctypes.c_void_p(s.cuda_stream)) == 0
    s.synchronize()
    want = torch.empty(3 * n, dtype=torch.float64, device="cuda")
    st.apply_into(_lib.MODE_FULL, torch.from_numpy(xh).cuda(), want)
    assert np.array_equal(yh, want.cpu().numpy())


@pytest.mark.gpu
@pytest.mark.parametrize("split", ["miehe", "none"])
def test_vcycle_fused_chebyshev_start_bitwise(split):
    """pff_smooth_init / pff_apply_emit / pff_apply_cheb_first (the Chebyshev
    start folded into the residual producers) give the V-cycle of the separate
    pff_cons + pff_cheb_init passes bit for bit, on sweep (>= 64^2) and generic
    levels."""
    import bench
    from paper_2005_00331_b200 import multigrid as MG
    level = 7
    h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, level, split, seed=1, notch=True)
    st = P.LinearizationState(h, level, params, split=split)
    st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
    st.set_dirichlet_nodes(dirn)
    st.refresh_cache()
    out = []
    saved = (MG.FUSE_INIT, MG.EMIT_FULL, MG.POST_UU, MG.DEFER_ACC)
    try:
        # (.., post_uu): the later smoothings' u-block residual as the UU application
        # instead of the FULL one (its phi rows are never read); (.., defer): the first
        # smoothing's z updated every second fused step (PFF_CHEB_NOACC)
        for fuse, emit, post_uu, defer in ((False, False, False, False), (False, False, True, False),
                                           (True, False, False, False), (True, False, True, True),
                                           (True, True, False, True), (True, True, True, False),
                                           (True, True, True, True)):
            MG.FUSE_INIT, MG.EMIT_FULL, MG.POST_UU, MG.DEFER_ACC = fuse, emit, post_uu, defer
            g = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
            g.setup(st)
            out.append(g.apply(x))
    finally:
        MG.FUSE_INIT, MG.EMIT_FULL, MG.POST_UU, MG.DEFER_ACC = saved
    for o in out[1:]:
        assert np.array_equal(out[0], o)


@pytest.mark.parametrize("sweeps", [2, 4, 5])
def test_vcycle_deferred_acc_other_sweep_counts(sweeps):
    """The NOACC / FIRST pairing of the fused Chebyshev steps for sweep counts other than
    the default 3 (odd and even numbers of fused steps), bitwise against the step-by-step z."""
    import bench
    from paper_2005_00331_b200 import multigrid as MG
    level = 6
    h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, level, "miehe", seed=2, notch=True)
    st = P.LinearizationState(h, level, params, split="miehe")
    st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
    st.set_dirichlet_nodes(dirn)
    st.refresh_cache()
    out = []
    saved = MG.DEFER_ACC
    try:
        for defer in (False, True):
            MG.DEFER_ACC = defer
            g = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=sweeps))
            g.setup(st)
            out.append(g.apply(x))
    finally:
        MG.DEFER_ACC = saved
    assert np.array_equal(out[0], out[1])


def test_dense_matvec_matches_torch():
    """pff_dense_matvec (the precomputed small-level V-cycle map) against a
    plain torch fp64 matvec."""
    from paper_2005_00331_b200._lib import call, ptr, stream_handle
    g = torch.Generator(device="cuda").manual_seed(3)
    for rows, cols in ((891, 891), (37, 1000), (1, 5)):
        M = torch.rand(rows, cols, dtype=torch.float64, device="cuda", generator=g) - 0.5
        x = torch.rand(cols, dtype=torch.float64, device="cuda", generator=g) - 0.5
        y = torch.empty(rows, dtype=torch.float64, device="cuda")
        call("pff_dense_matvec", rows, cols, ptr(M), ptr(x), ptr(y), stream_handle())
        ref = M @ x
        assert rel_l2(y.cpu().numpy(), ref.cpu().numpy()) <= 1e-14


def test_dense_setup_kernels_match_torch():
    """The GMG setup's own dense kernels (pff_dense.cu) against plain torch fp64:
    GEMM on sub-matrix views with alpha/beta, the row-scaled axpby, diag, recip."""
    from paper_2005_00331_b200._lib import call, ptr, stream_handle
    g = torch.Generator(device="cuda").manual_seed(4)
    rnd = lambda *sh: torch.rand(*sh, dtype=torch.float64, device="cuda", generator=g) - 0.5  # noqa: E731
    st = stream_handle()
    for m, n, k in ((891, 891, 891), (85, 891, 297), (1, 3, 2), (170, 170, 170), (65, 63, 17)):
        A, B = rnd(m + 3, k + 5), rnd(k, n + 2)
        C0 = rnd(m, n)
        Av, Bv = A[1:m + 1, 2:k + 2], B[:, 1:n + 1]          # strided views (lda, ldb > k, n)
        C = C0.clone()
        call("pff_dgemm", m, n, k, -0.75, ptr(Av), Av.stride(0), ptr(Bv), Bv.stride(0), 1.5,
             ptr(C), C.stride(0), st)
        ref = 1.5 * C0 - 0.75 * (Av @ Bv)
        assert rel_l2(C.cpu().numpy(), ref.cpu().numpy()) <= 1e-14, (m, n, k)
        C = torch.full((m, n), float("nan"), dtype=torch.float64, device="cuda")
        call("pff_dgemm", m, n, k, 1.0, ptr(Av), Av.stride(0), ptr(Bv), Bv.stride(0), 0.0,
             ptr(C), C.stride(0), st)
        assert rel_l2(C.cpu().numpy(), (Av @ Bv).cpu().numpy()) <= 1e-14
    Y0, X, sv = rnd(40, 30), rnd(40, 30), rnd(40)
    Y = Y0.clone()
    call("pff_dmat_axpby", 40, 30, 0.5, ptr(Y), 30, -2.0, ptr(sv), ptr(X), 30, st)
    assert torch.allclose(Y, 0.5 * Y0 - 2.0 * sv[:, None] * X, rtol=1e-15, atol=1e-15)
    Y = torch.full((40, 30), float("nan"), dtype=torch.float64, device="cuda")
    call("pff_dmat_axpby", 40, 30, 0.0, ptr(Y), 30, 3.0, None, ptr(X), 30, st)
    assert torch.equal(Y, 3.0 * X)
    D = torch.empty(40, 40, dtype=torch.float64, device="cuda")
    call("pff_dmat_diag", 40, ptr(sv), ptr(D), 40, st)
    assert torch.equal(D, torch.diag(sv))
    x = torch.rand(1000, dtype=torch.float64, device="cuda", generator=g) + 0.1
    y = torch.empty_like(x)
    call("pff_recip", 1000, ptr(x), ptr(y), 1, st)
    assert torch.allclose(y, 1.0 / torch.sqrt(x), rtol=1e-15, atol=0)
    call("pff_recip", 1000, ptr(x), ptr(y), 0, st)
    assert torch.allclose(y, 1.0 / x, rtol=1e-15, atol=0)


@pytest.mark.parametrize("split", ["miehe", "none"])
@pytest.mark.parametrize("p,level", [(2, 2), (2, 3), (1, 3)])
def test_dense_jacobian_matches_sparse_assembly(split, p, level):
    """pff_dense_jacobian (the setup's masked dense coarse Jacobian) against the
    sparse assembled oracle (src/pff_operator.py:343-377)."""
    ost, _ = O.baseline_state(p, level, split, seed=2)
    h = P.build_hierarchy(max(level, 2), p)
    st = P.LinearizationState(h, level, ost.params, split=split)
    st.set_solution(ost.U); st.set_phi_tilde(ost.phi_tilde); st.set_phi_old(ost.phi_old)
    st.set_active(ost.active); st.set_dirichlet_nodes(np.flatnonzero(ost.dirichlet))
    st.refresh_cache()
    gmg = P.GmgPreconditioner(h, coarse_level=2)
    G = gmg._dense_jacobian(st).cpu().numpy()
    ref = P.operator.assemble_oracle(st).device.to_dense().cpu().numpy()
    assert np.max(np.abs(G - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("split", ["miehe", "none"])
def test_dense_level_vcycle_matches_matrix_free(split):
    """The V-cycle with the level-3 dense map and dense coarse maps equals the
    matrix-free one (the reference's algebra, kernel by kernel) on a 7-level
    hierarchy within 1e-13 per block."""
    import bench
    from paper_2005_00331_b200 import multigrid as MG
    level = 7
    h, params, U, pt, act, dirn, x = bench.baseline_inputs(2, level, split, seed=2, notch=True)
    st = P.LinearizationState(h, level, params, split=split)
    st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
    st.set_dirichlet_nodes(dirn)
    st.refresh_cache()
    g1 = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    g1.setup(st)
    assert g1._dense_l is not None and g1._dense is not None
    z1 = g1.apply(x)
    saved = (MG.DENSE_COARSE, MG.DENSE_LEVEL)
    try:
        MG.DENSE_COARSE, MG.DENSE_LEVEL = False, False
        g2 = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
        g2.setup(st)
        assert g2._dense_l is None and g2._dense is None
        z2 = g2.apply(x)
        MG.DENSE_COARSE, MG.DENSE_LEVEL = True, False   # coarse maps only
        g3 = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
        g3.setup(st)
        z3 = g3.apply(x)
    finally:
        MG.DENSE_COARSE, MG.DENSE_LEVEL = saved
    n = st.n_scalar
    assert max(block_rel(z1, z2, n)) <= 1e-13
    assert max(block_rel(z3, z2, n)) <= 1e-13
