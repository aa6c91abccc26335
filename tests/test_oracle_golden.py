"""Pin the CPU oracle against golden vectors made by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, block_rel, load_golden, rel_l2
from oracle import oracle as O

TOL = 1e-13   # oracle restates the reference op-for-op; observed ~1e-16


def state_from(d, split):
    p, level = int(d["meta"][0]), int(d["meta"][1])
    st = O.State(p, level, O.baseline_material(level), split)
    st.U = d["U"].copy()
    st.phi_tilde = d["phi_tilde"].copy()
    st.phi_old = d["phi_old"].copy()
    st.active = d["active"].copy()
    st.dirichlet = d["dirichlet"].copy()
    st.refresh_cache()
    return st


OP_CASES = sorted(os.path.basename(f)[:-4] for f in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if os.path.basename(f).startswith(("pr1_", "op_")))


@pytest.mark.parametrize("name", OP_CASES)
def test_operator_family(name):
    d = load_golden(name)
    split = "miehe" if int(d["meta"][3]) else "none"
    st = state_from(d, split)
    n = st.n
    x = d["x"]
    assert max(block_rel(O.apply_jacobian(st, x), d["jac"], n)) <= TOL
    assert max(block_rel(O.apply_block_uu(st, x[:2 * n]), d["uu"], n)) <= TOL
    assert rel_l2(O.apply_block_phiphi(st, x[2 * n:]), d["pp"]) <= TOL
    assert rel_l2(O.apply_phi_row(st, x), d["prow"]) <= TOL
    assert max(block_rel(O.block_diagonal(st, "uu"), d["diag_uu"], n)) <= TOL
    assert rel_l2(O.block_diagonal(st, "phiphi"), d["diag_pp"]) <= TOL
    r = O.residual(st)
    for k, v in enumerate(block_rel(r, d["residual"], n)):
        assert v <= TOL or np.abs(r[k * n:(k + 1) * n]).max() == 0.0
    assert max(block_rel(O.residual(st, mask_dirichlet=False), d["residual_raw"], n)) <= TOL


@pytest.mark.parametrize("split", ["none", "miehe"])
def test_cache_matches(split):
    d = load_golden(f"pr1_{split}")
    st = state_from(d, split)
    for k in ("e11", "e22", "e12", "gt", "dg", "esp", "pc"):
        assert rel_l2(st.cache[k], d["cache_" + k]) <= TOL, k


@pytest.mark.parametrize("split", ["none", "miehe"])
def test_colour_parallel_matches_serial(split):
    d = load_golden(f"pr1_{split}")
    st = state_from(d, split)
    y1 = O.apply_jacobian(st, d["x"], nthreads=1)
    y4 = O.apply_jacobian(st, d["x"], nthreads=4)
    assert max(block_rel(y4, y1, st.n)) <= 1e-15


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_transfer(p):
    d = load_golden(f"transfer_p{p}_l4")
    tr = O.Transfer(p, 4)
    assert np.array_equal(tr.P.indptr, d["P_indptr"])
    assert np.array_equal(tr.P.indices, d["P_indices"])
    assert np.abs(tr.P.data - d["P_data"]).max() == 0.0
    assert rel_l2(tr.prolongate(d["xc"]), d["Px"]) <= 1e-15
    assert rel_l2(tr.restrict(d["yf"]), d["Ry"]) <= 1e-15
    assert np.array_equal(O.injection(p, 4), d["inj"])


def test_transfer_level1():
    d = load_golden("transfer_p2_l1")
    tr = O.Transfer(2, 1)
    assert rel_l2(tr.prolongate(d["xc"]), d["Px"]) <= 1e-15
    assert rel_l2(tr.restrict(d["yf"]), d["Ry"]) <= 1e-15


def test_restrict_state():
    d = load_golden("restrict_p2_l5_l2")
    st = state_from(dict(d, meta=np.array([2, 5, 0, 1])), "miehe")
    c = O.restrict_state(st, 2)
    assert np.array_equal(c.U, d["cU"])
    assert np.array_equal(c.phi_tilde, d["cphi_tilde"])
    assert np.array_equal(c.active, d["cactive"])
    assert np.array_equal(c.dirichlet, d["cdirichlet"])


@pytest.mark.parametrize("p", [1, 2, 4])
def test_lumped_mass(p):
    d = load_golden(f"mass_p{p}_l3")
    assert rel_l2(O.lumped_mass(p, 3), d["m"]) <= TOL


SOLVE_CASES = sorted(os.path.basename(f)[:-4] for f in glob.glob(os.path.join(GOLDEN, "solve_*.npz")))


@pytest.mark.parametrize("name", SOLVE_CASES)
def test_solver_stack(name):
    d = load_golden(name)
    p, level, seed, miehe, notch, sweeps = (int(v) for v in d["meta"])
    split = "miehe" if miehe else "none"
    st = state_from(dict(d, meta=np.array([p, level, seed, miehe])), split)
    n = st.n
    gmg = O.Gmg(p, level, coarse_level=2, cheb=O.ChebCfg(sweeps=sweeps))
    gmg.setup(st)
    for l in range(2, level + 1):
        got = gmg.ranges[l]
        want = d[f"range_{l}"]
        assert np.allclose([got["uu"][0], got["uu"][1], got["phiphi"][0], got["phiphi"][1]],
                           want, rtol=1e-12, atol=0), l
    assert max(block_rel(gmg.apply(d["x"]), d["vcycle"], n)) <= 1e-12
    hi = gmg.ranges[level]["uu"][1]
    cheb = O.chebyshev_apply(lambda v: O.apply_block_uu(st, v), gmg.diags[level]["uu"],
                             d["x"][:2 * n], 0.24 * hi, 1.2 * hi, 5)
    assert max(block_rel(cheb, d["cheb_uu"], n)) <= 1e-12
    lz = O.estimate_lambda_range(lambda v: O.apply_block_uu(st, v), gmg.diags[level]["uu"], seed=7)
    assert np.allclose(lz, d["lanczos_uu"], rtol=1e-12, atol=0)
    rhs = d["x"].copy()
    rhs[st.constrained_mask()] = 0.0
    res = O.gmres(lambda v: O.apply_jacobian(st, v), rhs, tol=1e-8, restart=50,
                  preconditioner=gmg.apply)
    assert res.converged == bool(d["gmres_conv"][0])
    assert res.iterations == int(d["gmres_iters"][0])
    assert max(block_rel(res.solution, d["gmres_x"], n)) <= 1e-10


# ---- active-set loop (src/active_set_solver.py:101-163) -----------------------
AS_CASES = ["as_p1_l3_miehe_t40", "as_p1_l4_miehe_t1", "as_p2_l4_miehe_notch"]


def as_state(d):
    p, level, miehe = (int(v) for v in d["meta"][:3])
    lam, mu, gc, kappa, eps = (float(v) for v in d["material"])
    st = O.State(p, level, O.Material(lame_lambda=lam, mu=mu, g_c=gc, kappa=kappa, eps=eps),
                 "miehe" if miehe else "none")
    st.U = d["U0"].copy()
    st.phi_tilde = d["phi_tilde"].copy()
    st.phi_old = d["phi_old"].copy()
    st.dirichlet = d["dirichlet"].copy()
    return st


def test_boundary_program_and_values():
    d = load_golden("as_p1_l4_miehe_t1")
    st = O.State(1, 4, O.Material(), "miehe")
    O.apply_boundary_values(st, O.boundary_program("tension", *d["load"]))
    assert np.array_equal(st.U, d["U0"]) and np.array_equal(st.dirichlet, d["dirichlet"])
    with pytest.raises(ValueError):
        O.boundary_program("tension", -1.0)
    with pytest.raises(ValueError):
        O.boundary_program("torsion", 1.0)


@pytest.mark.parametrize("name", AS_CASES)
def test_active_set_step(name):
    d = load_golden(name)
    st = as_state(d)
    m = O.lumped_mass(st.p, st.level)
    assert np.array_equal(m, d["m"])
    gmg = O.Gmg(st.p, st.level, coarse_level=2, nthreads=O.max_threads())
    rep = O.active_set_solve_step(st, gmg, m, nthreads=O.max_threads())
    assert rep.converged and rep.as_iterations == int(d["as_iterations"][0])
    assert rep.gmres_iterations == d["gmres_iterations"].tolist()
    assert rep.active_counts == d["active_counts"].tolist()
    assert np.array_equal(st.active, d["active"])
    assert max(block_rel(st.U, d["U"], st.n)) <= 1e-10
    # the last norms sit at round-off: compare relative to the initial residual
    r0 = d["residual_norms"][0]
    assert np.abs(np.array(rep.residual_norms) - d["residual_norms"]).max() <= 1e-12 * r0
