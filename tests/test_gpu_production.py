"""Production-size parity: the multigrid and Krylov layers where the Q2 sweep
kernel and the large-level transfer paths actually run.

The small solver goldens (levels 4-5, tests/test_gpu_parity.py) sit below the
sweep kernel's threshold (64 cells per side), so these tests pin, against the
REFERENCE itself (fixtures tests/golden/prod_*.npz from
`make_golden.py --production`) and against the C oracle:

* level 7 (128^2 Q2, levels 6-7 on the sweep kernel): Lanczos ranges, one
  V-cycle and the GMRES(50) solve of the configs[3] inputs;
* level 10 (configs[3], 1024^2): the ranges and the V-cycle against a sketch
  of the reference's output (norms, projections, 4096 sampled entries per
  block) and the whole vector against oracle.Gmg;
* the PR1 goldens (32^2) with the sweep kernel forced onto that level;
* the fine-level transfer kernels bound to states (element-vector scratch,
  shared-memory-staged restriction, 32-bit prolongation) against P / P^T.

Reference: src/multigrid.py:123-162, 201-344; src/krylov.py:37-119.
"""

import numpy as np
import pytest
import torch

import bench
from conftest import block_rel, load_golden, rel_l2, sketch, sketch_rel
import paper_2005_00331_b200 as P
from paper_2005_00331_b200 import _lib
from oracle import oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _state(level, split, p=2):
    h, params, U, pt, act, dirn, x = bench.baseline_inputs(p, level, split, seed=0, notch=True)
    st = P.LinearizationState(h, level, params, split=split)
    st.set_solution(U); st.set_phi_tilde(pt); st.set_phi_old(pt); st.set_active(act)
    st.set_dirichlet_nodes(dirn)
    st.refresh_cache()
    return st, x


def _oracle_state(level, split, nt):
    ost, x = O.baseline_state(2, level, split, seed=0, notch=True)
    ost.refresh_cache(nthreads=nt)
    return ost, x


def _ranges(d, level):
    out = {}
    for l in range(2, level + 1):
        r = d[f"range_{l}"]
        out[l] = {"uu": (float(r[0]), float(r[1])), "phiphi": (float(r[2]), float(r[3]))}
    return out


def _check_ranges(gmg, d, level):
    for l in range(2, level + 1):
        got = gmg.ranges[l]
        assert np.allclose([got["uu"][0], got["uu"][1], got["phiphi"][0], got["phiphi"][1]],
                           d[f"range_{l}"], rtol=1e-10, atol=0), l


def _np(t):
    return t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


@pytest.mark.parametrize("split", ["miehe", "none"])
def test_level7_vcycle_and_gmres_vs_reference(split):
    """128^2 Q2 (configs[3] inputs): ranges, V-cycle (graph and eager, with
    estimated and with injected ranges) and GMRES(50) against the reference."""
    d = load_golden(f"prod_p2_l7_{split}")
    st, x = _state(7, split)
    n = st.n_scalar
    gmg = P.GmgPreconditioner(st.hierarchy, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    gmg.setup(st)
    _check_ranges(gmg, d, 7)
    z = _np(gmg.apply(x))
    assert max(block_rel(z, d["vcycle"], n)) <= TOL
    gmg.use_graph = False
    assert max(block_rel(_np(gmg.apply(x)), d["vcycle"], n)) <= TOL
    gmg.use_graph = True
    gi = P.GmgPreconditioner(st.hierarchy, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    gi.setup(st, ranges=_ranges(d, 7))
    assert max(block_rel(_np(gi.apply(x)), d["vcycle"], n)) <= TOL
    rhs = x.copy()
    rhs[st.constrained_mask()] = 0.0
    res = P.gmres_solve(P.JacobianOperator(st), rhs,
                        P.KrylovConfig(relative_tolerance=1e-8, restart=50),
                        preconditioner=gmg.apply)
    assert res.converged and bool(d["gmres_conv"][0])
    assert res.iterations == int(d["gmres_iters"][0])
    assert max(block_rel(_np(res.solution), d["gmres_x"], n)) <= 1e-8
    # the residual history follows the reference's to well below the tolerance
    h_ref = d["gmres_hist"]
    h_got = np.asarray(res.residual_history)
    assert h_got.shape == h_ref.shape
    assert np.max(np.abs(h_got - h_ref) / h_ref[0]) <= 1e-10


@pytest.mark.parametrize("split", ["miehe", "none"])
def test_level7_gmres_vs_oracle(split):
    """The same solve against the oracle's GMRES + V-cycle (iterations equal,
    solution <= 1e-8 per block)."""
    nt = O.max_threads()
    st, x = _state(7, split)
    ost, _ = _oracle_state(7, split, nt)
    n = st.n_scalar
    rhs = x.copy()
    rhs[st.constrained_mask()] = 0.0
    gmg = P.GmgPreconditioner(st.hierarchy, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    gmg.setup(st)
    og = O.Gmg(2, 7, coarse_level=2, cheb=O.ChebCfg(sweeps=3), nthreads=nt)
    og.setup(ost)
    res = P.gmres_solve(P.JacobianOperator(st), rhs,
                        P.KrylovConfig(relative_tolerance=1e-8, restart=50),
                        preconditioner=gmg.apply)
    ores = O.gmres(lambda v: O.apply_jacobian(ost, v, nt), rhs, tol=1e-8, restart=50,
                   preconditioner=og.apply)
    assert res.iterations == ores.iterations
    assert max(block_rel(_np(res.solution), ores.solution, n)) <= 1e-8


@pytest.mark.slow
@pytest.mark.parametrize("split", ["miehe", "none"])
def test_level10_vcycle_vs_reference_and_oracle(split):
    """configs[3] hierarchy (1024^2 Q2, 9 levels, every level >= 64^2 on the
    sweep kernel with its fused Chebyshev / emit / last forms, the staged
    restriction, the dense level-3 map): the ranges and the V-cycle against the
    reference (sketch) and the whole V-cycle against oracle.Gmg, once with the
    ranges estimated independently and once injected."""
    d = load_golden(f"prod_p2_l10_{split}")
    st, x = _state(10, split)
    n = st.n_scalar
    gmg = P.GmgPreconditioner(st.hierarchy, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    gmg.setup(st)
    _check_ranges(gmg, d, 10)
    z = _np(gmg.apply(torch.from_numpy(x).cuda()))
    want = {k[len("vcycle_"):]: d[k] for k in d if k.startswith("vcycle_") and k != "vcycle_s"}
    assert sketch_rel(sketch(z, n), want) <= TOL
    nt = O.max_threads()
    ost, _ = _oracle_state(10, split, nt)
    og = O.Gmg(2, 10, coarse_level=2, cheb=O.ChebCfg(sweeps=3), nthreads=nt)
    og.setup(ost, ranges=_ranges(d, 10))
    zo = og.apply(x)
    assert max(block_rel(z, zo, n)) <= TOL
    assert sketch_rel(sketch(zo, n), want) <= TOL   # the oracle itself, at full size
    gi = P.GmgPreconditioner(st.hierarchy, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    gi.setup(st, ranges=_ranges(d, 10))
    assert max(block_rel(_np(gi.apply(torch.from_numpy(x).cuda())), zo, n)) <= TOL


@pytest.mark.slow
@pytest.mark.parametrize("split", ["miehe", "none"])
def test_level11_newton_step_vs_reference(split):
    """2048^2 Q2 (50 M DoFs), the configs[3]/[4] inputs one level below
    configs[4]: the reference itself (fixture from make_golden.py --production
    11, an hour of serial numba GMRES) needs 43 (Miehe) GMRES(50) iterations --
    the growth 28 (1024^2) -> 43 (2048^2) -> 82 (4096^2) is the reference's own.
    Ranges on every level, the first V-cycle (sketch), the iteration count,
    the residual history and the solution (sketch) against it."""
    import os
    from conftest import GOLDEN
    name = f"prod_p2_l11_{split}"
    if not os.path.exists(os.path.join(GOLDEN, name + ".npz")):
        pytest.skip(f"{name} not generated")
    d = load_golden(name)
    st, x = _state(11, split)
    n = st.n_scalar
    gmg = P.GmgPreconditioner(st.hierarchy, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    gmg.setup(st)
    _check_ranges(gmg, d, 11)
    xd = torch.from_numpy(x).cuda()
    want = {k[len("vcycle_"):]: d[k] for k in d if k.startswith("vcycle_") and k != "vcycle_s"}
    assert sketch_rel(sketch(_np(gmg.apply(xd)), n), want) <= TOL
    rhs = x.copy()
    rhs[st.constrained_mask()] = 0.0
    res = P.gmres_solve(P.JacobianOperator(st), torch.from_numpy(rhs).cuda(),
                        P.KrylovConfig(relative_tolerance=1e-8, restart=50),
                        preconditioner=gmg.apply)
    assert res.converged and res.iterations == int(d["gmres_iters"][0])
    h_ref, h_got = d["gmres_hist"], np.asarray(res.residual_history)
    assert h_got.shape == h_ref.shape
    assert np.max(np.abs(h_got - h_ref) / h_ref[0]) <= 1e-10
    wx = {k[len("gmres_x_"):]: d[k] for k in d if k.startswith("gmres_x_")}
    assert sketch_rel(sketch(_np(res.solution), n), wx) <= 1e-8


@pytest.mark.slow
def test_level12_first_iterations_vs_oracle():
    """configs[4] (4096^2 Q2, 201 M DoFs): the C oracle's first 8 GMRES(50)
    iterations on the box's host cores (tools/pin_newton_oracle.py
    --max-iterations 8, fixture pin_oracle_l12_miehe_it8.json; the whole
    82-iteration oracle solve takes about an hour) -- Lanczos ranges on every
    level, the first V-cycle (sketch) and the residual history against the
    device solve's."""
    import json
    import os
    from conftest import GOLDEN
    with open(os.path.join(GOLDEN, "pin_oracle_l12_miehe_it8.json")) as f:
        d = json.load(f)
    st, x = _state(12, "miehe")
    n = st.n_scalar
    gmg = P.GmgPreconditioner(st.hierarchy, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    gmg.setup(st)
    for l, r in d["ranges"].items():
        got = gmg.ranges[int(l)]
        assert np.allclose([got["uu"][0], got["uu"][1], got["phiphi"][0], got["phiphi"][1]], r,
                           rtol=1e-10, atol=0), l
    xd = torch.from_numpy(x).cuda()
    want = {k: np.asarray(v) for k, v in d["vcycle_sketch"].items()}
    assert sketch_rel(sketch(_np(gmg.apply(xd)), n), want) <= TOL
    del xd
    rhs = x.copy()
    rhs[st.constrained_mask()] = 0.0
    res = P.gmres_solve(P.JacobianOperator(st), torch.from_numpy(rhs).cuda(),
                        P.KrylovConfig(relative_tolerance=1e-8, restart=50, max_iterations=8),
                        preconditioner=gmg.apply)
    h_ref, h_got = np.asarray(d["history"]), np.asarray(res.residual_history)
    assert res.iterations == 8 and h_got.shape == h_ref.shape
    # the last entry of both is the true residual of the returned iterate
    assert np.max(np.abs(h_got - h_ref) / h_ref[0]) <= 1e-10


@pytest.mark.parametrize("name", ["pr1_miehe", "pr1_none"])
def test_pr1_goldens_through_sweep_kernel(name):
    """PR1 (32^2 Q2) is below the sweep kernel's default threshold; force the
    sweep kernel onto it (PFF_OPT_SWEEP_MIN_NSIDE) and check the whole operator
    family against the reference's vectors, plus the V-cycle golden at level 5
    with every level >= 8^2 on the sweep kernel."""
    d = load_golden(name)
    split = "miehe" if int(d["meta"][3]) else "none"
    _lib.set_option(_lib.OPT_SWEEP_MIN_NSIDE, 8)
    try:
        h = P.build_hierarchy(5, 2)
        st = P.LinearizationState(h, 5, O.baseline_material(5), split=split)
        st.set_solution(d["U"]); st.set_phi_tilde(d["phi_tilde"]); st.set_phi_old(d["phi_old"])
        st.set_active(d["active"]); st.set_dirichlet_nodes(np.flatnonzero(d["dirichlet"]))
        st.refresh_cache()
        assert st.uses_sweep_kernel()
        n, x = st.n_scalar, d["x"]
        assert max(block_rel(_np(P.apply_jacobian(st, x)), d["jac"], n)) <= TOL
        assert max(block_rel(_np(P.apply_block_uu(st, x[:2 * n])), d["uu"], n)) <= TOL
        assert rel_l2(_np(P.apply_block_phiphi(st, x[2 * n:])), d["pp"]) <= TOL
        assert rel_l2(_np(P.apply_phi_row(st, x)), d["prow"]) <= TOL
        s = load_golden(f"solve_p2_l5_{split}_rand")
        st2 = P.LinearizationState(h, 5, O.baseline_material(5), split=split)
        st2.set_solution(s["U"]); st2.set_phi_tilde(s["phi_tilde"]); st2.set_phi_old(s["phi_old"])
        st2.set_active(s["active"]); st2.set_dirichlet_nodes(np.flatnonzero(s["dirichlet"]))
        st2.refresh_cache()
        gmg = P.GmgPreconditioner(h, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
        gmg.setup(st2)
        assert max(block_rel(_np(gmg.apply(s["x"])), s["vcycle"], n)) <= TOL
    finally:
        _lib.set_option(_lib.OPT_SWEEP_MIN_NSIDE, 0)


@pytest.mark.parametrize("level", [9, 10])
def test_bound_transfers_vs_csr(level):
    """The V-cycle's transfer kernels with both levels bound to states (the
    restriction's element-vector scratch, its shared-memory-staged stores on
    >= 256^2 coarse meshes, the 32-bit prolongation) against the oracle's CSR
    P / P^T (src/multigrid.py:44-120), unmasked and masked."""
    st, _ = _state(level, "miehe")
    gmg = P.GmgPreconditioner(st.hierarchy, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    gmg.setup(st)
    sf, sc = gmg.states[level], gmg.states[level - 1]
    nf, nc = sf.n_scalar, sc.n_scalar
    T = O.Transfer(2, level)
    g = torch.Generator(device="cuda").manual_seed(level)
    y = torch.rand(3 * nf, dtype=torch.float64, device="cuda", generator=g) - 0.5
    xc = torch.rand(3 * nc, dtype=torch.float64, device="cuda", generator=g) - 0.5
    yh, xh = y.cpu().numpy(), xc.cpu().numpy()
    cons_f, cons_c = sf.constrained_mask(), sc.constrained_mask()
    s = P.multigrid.stream_handle()
    for zero_cons in (0, 1):
        out = torch.empty(3 * nc, dtype=torch.float64, device="cuda")
        _lib.call("pff_restrict", sf.bind(), sc.bind(), _lib.ptr(y), _lib.ptr(out), zero_cons, s)
        want = T.restrict(yh)
        if zero_cons:
            want[cons_c] = 0.0
        assert max(block_rel(out.cpu().numpy(), want, nc)) <= 1e-14
    out = torch.empty(3 * nf, dtype=torch.float64, device="cuda")
    _lib.call("pff_prolongate", sf.bind(), sc.bind(), _lib.ptr(xc), _lib.ptr(out), 0, s)
    want = T.prolongate(xh)
    assert max(block_rel(out.cpu().numpy(), want, nf)) <= 1e-14
    base = torch.rand(3 * nf, dtype=torch.float64, device="cuda", generator=g)
    out = base.clone()
    _lib.call("pff_prolongate", sf.bind(), sc.bind(), _lib.ptr(xc), _lib.ptr(out), 1, s)
    want = base.cpu().numpy() + np.where(cons_f, 0.0, T.prolongate(xh))
    assert max(block_rel(out.cpu().numpy(), want, nf)) <= 1e-14


# ------------------------------------------------------------ Q4 write-once sweep

@pytest.mark.parametrize("name", ["op_p4_l3_miehe", "op_p4_l3_none"])
def test_q4_goldens_through_sweep_kernel(name):
    """The reference's p=4 operator goldens (8^2 Q4 cells) with the Q4 sweep
    kernel forced onto that level (PFF_OPT_SWEEP_MIN_NSIDE)."""
    d = load_golden(name)
    split = "miehe" if int(d["meta"][3]) else "none"
    _lib.set_option(_lib.OPT_SWEEP_MIN_NSIDE, 4)
    try:
        h = P.build_hierarchy(3, 4)
        st = P.LinearizationState(h, 3, O.baseline_material(3), split=split)
        st.set_solution(d["U"]); st.set_phi_tilde(d["phi_tilde"]); st.set_phi_old(d["phi_old"])
        st.set_active(d["active"]); st.set_dirichlet_nodes(np.flatnonzero(d["dirichlet"]))
        st.refresh_cache()
        assert st.uses_sweep_kernel()
        n, x = st.n_scalar, d["x"]
        assert max(block_rel(_np(P.apply_jacobian(st, x)), d["jac"], n)) <= TOL
        assert max(block_rel(_np(P.apply_block_uu(st, x[:2 * n])), d["uu"], n)) <= TOL
        assert rel_l2(_np(P.apply_block_phiphi(st, x[2 * n:])), d["pp"]) <= TOL
        assert rel_l2(_np(P.apply_phi_row(st, x)), d["prow"]) <= TOL
    finally:
        _lib.set_option(_lib.OPT_SWEEP_MIN_NSIDE, 0)


@pytest.mark.parametrize("split", ["none", "miehe"])
@pytest.mark.parametrize("level,rows", [(2, 0), (3, 1), (4, 3), (5, 0), (6, 7), (7, 0)])
def test_q4_sweep_matches_generic_all_modes(split, level, rows, monkeypatch):
    """The write-once Q4 kernel against the cooperative element-vector kernel
    (k_apply_coop + k_apply_gather), every mode, plain and fused, with extra
    active / Dirichlet nodes on the slit, over chunkings that put chunk edges
    on and off the slit row; and bitwise repeatable."""
    monkeypatch.setenv("PFF_SWEEP4_ROWS", str(rows))
    ost, x = O.baseline_state(4, level, split, seed=level)
    _lib.set_option(_lib.OPT_SWEEP_MIN_NSIDE, 4)
    try:
        h = P.build_hierarchy(max(level, 2), 4)
        st = P.LinearizationState(h, level, ost.params, split=split)
        st.set_solution(ost.U); st.set_phi_tilde(ost.phi_tilde); st.set_phi_old(ost.phi_old)
        act = ost.active.copy()
        act[np.random.default_rng(level).choice(st.n_scalar, 7, replace=False)] = True
        dn = ost.dirichlet.copy()
        dn[h.dof_map(level).slit_upper[:2]] = True
        st.set_active(act)
        st.set_dirichlet_nodes(np.flatnonzero(dn))
        st.refresh_cache()
        assert st.uses_sweep_kernel()
    finally:
        _lib.set_option(_lib.OPT_SWEEP_MIN_NSIDE, 0)
    n = st.n_scalar
    xd = torch.from_numpy(x).cuda()
    rhs = torch.from_numpy(np.random.default_rng(1).standard_normal(3 * n)).cuda()
    cases = [(0, xd, 3 * n), (1, xd[:2 * n], 2 * n), (2, xd[2 * n:], n), (3, xd, n)]
    try:
        for mode, src, nout in cases:
            outs = []
            for flag in (1, 0):
                _lib.set_option(_lib.OPT_GENERIC_APPLY, flag)
                y = torch.empty(nout, dtype=torch.float64, device="cuda")
                st.apply_into(mode, src, y)
                yf = torch.empty(nout, dtype=torch.float64, device="cuda")
                st.apply_into(mode, src, yf, rhs[:nout])
                outs.append((y.cpu().numpy(), yf.cpu().numpy()))
            (g, gf), (s, sf) = outs
            assert max(block_rel(s, g, n)) <= 1e-13, (mode, block_rel(s, g, n))
            assert max(block_rel(sf, gf, n)) <= 1e-13, mode
    finally:
        _lib.set_option(_lib.OPT_GENERIC_APPLY, 0)
    y1 = P.apply_jacobian(st, xd)
    y2 = P.apply_jacobian(st, xd)
    assert torch.equal(y1, y2)


@pytest.mark.parametrize("p,level,split", [(4, 6, "miehe"), (4, 6, "none"), (3, 6, "miehe"),
                                           (1, 7, "miehe")])
def test_other_degrees_vcycle_and_gmres_vs_oracle(p, level, split):
    """Q4 hierarchies mix the write-once Q4 sweep (the residual and phi-row
    applications on >= 64^2 levels) with the cooperative kernel (the fused
    Chebyshev forms, small levels); Q3 and Q1 run the cooperative kernel
    throughout.  V-cycle <= 1e-12 per block and GMRES(50) iterations against the
    oracle (src/multigrid.py:201-344, src/krylov.py:37-119), notch inputs."""
    nt = O.max_threads()
    st, x = _state(level, split, p=p)
    ost, _ = O.baseline_state(p, level, split, seed=0, notch=True)
    ost.refresh_cache(nthreads=nt)
    n = st.n_scalar
    gmg = P.GmgPreconditioner(st.hierarchy, coarse_level=2, cheb=P.ChebyshevConfig(sweeps=3))
    gmg.setup(st)
    og = O.Gmg(p, level, coarse_level=2, cheb=O.ChebCfg(sweeps=3), nthreads=nt)
    og.setup(ost)
    for l in range(2, level + 1):
        a, b = gmg.ranges[l], og.ranges[l]
        assert np.allclose([a["uu"][0], a["uu"][1], a["phiphi"][0], a["phiphi"][1]],
                           [b["uu"][0], b["uu"][1], b["phiphi"][0], b["phiphi"][1]], rtol=1e-10, atol=0)
    assert max(block_rel(_np(gmg.apply(x)), og.apply(x), n)) <= TOL
    rhs = x.copy()
    rhs[st.constrained_mask()] = 0.0
    res = P.gmres_solve(P.JacobianOperator(st), rhs,
                        P.KrylovConfig(relative_tolerance=1e-8, restart=50),
                        preconditioner=gmg.apply)
    ores = O.gmres(lambda v: O.apply_jacobian(ost, v, nt), rhs, tol=1e-8, restart=50,
                   preconditioner=og.apply)
    assert abs(res.iterations - ores.iterations) <= 1
    assert max(block_rel(_np(res.solution), ores.solution, n)) <= 1e-8
