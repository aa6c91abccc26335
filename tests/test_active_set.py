"""Active-set loop (src/active_set_solver.py): device
kernels and the device-resident PDAS loop against the oracle and the
reference's own fixtures (tests/golden/as_*.npz, lumped mass goldens)."""

import numpy as np
import pytest

from conftest import block_rel, load_golden
import paper_2005_00331_b200 as P
from oracle import oracle as O

gpu = pytest.mark.gpu


# ---- host logic (CPU) -------------------------------------------------------
def test_converged_logic():
    # src/active_set_solver.py:85-90 semantics (reference tests TestConverged)
    assert not P.converged(np.array([True]), None, 0.0, 1.0, 1e-8)
    a = np.array([True, False])
    assert P.converged(a, a.copy(), 0.0, 1.0, 1e-8)
    b = np.array([True])
    assert not P.converged(b, b.copy(), 1e-7, 1.0, 1e-8)
    assert P.converged(b, b.copy(), 0.9e-8, 1.0, 1e-8)
    assert not P.converged(np.array([True, False]), np.array([False, True]), 0.0, 1.0, 1e-8)


def test_params_and_boundary_program():
    with pytest.raises(ValueError):
        P.ActiveSetParams(complementarity_c=0.0)
    assert P.boundary_program("tension", 3.0, 2e-5) == O.boundary_program("tension", 3.0, 2e-5)
    assert P.boundary_program("shear", 3.0) == O.boundary_program("shear", 3.0)
    for bad in (("tension", -1.0), ("torsion", 1.0)):
        with pytest.raises(ValueError):
            P.boundary_program(*bad)
    assert P.SolveReport(gmres_iterations=[3, 4]).gmres_total == 7


# ---- lumped mass ---------------------------------------------------------------
@gpu
@pytest.mark.parametrize("p", [1, 2, 4])
def test_lumped_mass_golden_bitwise(p):
    got = P.lumped_mass_diagonal(P.build_hierarchy(3, p), 3)
    assert np.array_equal(got, load_golden(f"mass_p{p}_l3")["m"])


@gpu
@pytest.mark.parametrize("p,level", [(1, 0), (2, 1), (3, 4), (2, 7), (2, 10), (4, 9)])
def test_lumped_mass_oracle_bitwise(p, level):
    got = P.lumped_mass_diagonal(P.build_hierarchy(max(level, 2), p), level)
    want = O.lumped_mass(p, level)
    assert np.array_equal(got, want)
    assert got.sum() == pytest.approx(1.0, rel=1e-12)


# ---- complementarity pass ----------------------------------------------------
@gpu
def test_determine_active_set_reference_cases():
    # the reference's TestDetermineActiveSet cases
    n = 4
    rhs = np.zeros(3 * n)
    rhs[2 * n + 1] = 0.25
    got = P.determine_active_set(rhs, np.zeros(3 * n), np.zeros(n), np.full(n, 0.25), 100.0)
    assert got.tolist() == [False, True, False, False]
    rhs = np.zeros(3 * n)
    rhs[:2 * n] = 1e9
    assert not P.determine_active_set(rhs, np.zeros(3 * n), np.zeros(n), np.ones(n), 100.0).any()
    assert not P.determine_active_set(np.zeros(6), np.zeros(6), np.zeros(2), np.ones(2), 100.0).any()
    U = np.zeros(9)
    U[6:] = [0.5, 1.2, 0.9]
    got = P.determine_active_set(np.zeros(9), U, np.ones(3), np.ones(3), 100.0)
    assert got.tolist() == [False, True, False]


@gpu
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_determine_active_set_matches_oracle(seed):
    rng = np.random.default_rng(seed)
    n = 100_003
    m = rng.uniform(1e-6, 1e-3, n)
    rhs = rng.uniform(-1e-4, 1e-4, 3 * n)
    U = rng.uniform(0, 1, 3 * n)
    po = U[2 * n:] + rng.choice([0.0, 1e-7, -1e-7], n)     # many exact ties
    rhs[2 * n:][rng.random(n) < 0.1] = 0.0
    got = P.determine_active_set(rhs, U, po, m, 100.0)
    assert np.array_equal(got, O.determine_active_set(rhs, U, po, m, 100.0))


# ---- the loop --------------------------------------------------------------------
AS_CASES = ["as_p1_l3_miehe_t40", "as_p1_l4_miehe_t1", "as_p2_l4_miehe_notch",
            "as_p2_l6_none_notch", "as_p2_l6_miehe_notch"]


def build(d):
    p, level, miehe = (int(v) for v in d["meta"][:3])
    lam, mu, gc, kappa, eps = (float(v) for v in d["material"])
    h = P.build_hierarchy(level, p)
    st = P.LinearizationState(h, level, P.MaterialParams(lame_lambda=lam, mu=mu, g_c=gc,
                                                         kappa=kappa, eps=eps),
                              split="miehe" if miehe else "none")
    st.set_solution(d["U0"])
    st.set_phi_tilde(d["phi_tilde"])
    st.set_phi_old(d["phi_old"])
    st.set_dirichlet_nodes(np.flatnonzero(d["dirichlet"]))
    gmg = P.GmgPreconditioner(h, coarse_level=2)
    solver = P.ActiveSetSolver(gmg, P.KrylovConfig(), P.ActiveSetParams(),
                               P.lumped_mass_diagonal(h, level))
    return h, st, solver


@gpu
@pytest.mark.parametrize("name", AS_CASES)
def test_solve_step_matches_reference(name):
    d = load_golden(name)
    _, st, solver = build(d)
    rep = solver.solve_step(st)
    n = st.n_scalar
    assert rep.converged
    assert rep.as_iterations == int(d["as_iterations"][0])
    assert rep.active_counts == d["active_counts"].tolist()
    for got, want in zip(rep.gmres_iterations, d["gmres_iterations"]):
        assert abs(got - int(want)) <= 1
    assert np.array_equal(st.active, d["active"])
    # both loops end at the same discrete solution (residual <= 1e-8 r0)
    assert max(block_rel(st.U, d["U"], n)) <= 1e-7
    # irreversibility and complementarity (reference test_irreversibility_against_phi_old)
    phi, po = st.phi, st.phi_old
    assert np.all(phi <= po + 1e-10)
    assert np.array_equal(phi[st.active], po[st.active])


@gpu
def test_fully_active_phi_is_untouched():
    # reference TestActiveSetStep.test_fully_active_phi_is_untouched
    h = P.build_hierarchy(3, 1)
    st = P.LinearizationState(h, 3, P.MaterialParams())
    P.apply_boundary_values(st, P.boundary_program("tension", 5.0))
    st.set_active(np.ones(st.n_scalar, dtype=bool))
    st.refresh_cache()
    rhs = -P.residual(st, mask_active=True)
    rhs[st.constrained_mask()] = 0.0
    gmg = P.GmgPreconditioner(h, coarse_level=2)
    gmg.setup(st)
    res = P.gmres_solve(lambda v: P.apply_jacobian(st, v), rhs, P.KrylovConfig(),
                        preconditioner=gmg.apply)
    n = st.n_scalar
    assert res.converged
    assert np.all(res.solution[2 * n:] == 0.0)
    assert np.linalg.norm(res.solution[:2 * n]) > 0.0


@gpu
def test_linear_problem_converges_in_one_newton_step():
    h = P.build_hierarchy(3, 1)
    st = P.LinearizationState(h, 3, P.MaterialParams(), split="none")
    P.apply_boundary_values(st, P.boundary_program("tension", 1.0))
    st.set_active(np.ones(st.n_scalar, dtype=bool))
    st.refresh_cache()
    rhs = -P.residual(st, mask_active=True)
    rhs[st.constrained_mask()] = 0.0
    r0 = np.linalg.norm(rhs)
    gmg = P.GmgPreconditioner(h, coarse_level=2)
    gmg.setup(st)
    res = P.gmres_solve(lambda v: P.apply_jacobian(st, v), rhs,
                        P.KrylovConfig(relative_tolerance=1e-10), preconditioner=gmg.apply)
    st.set_solution(st.U + res.solution)
    st.refresh_cache()
    r = P.residual(st, mask_active=True)
    r[st.constrained_mask()] = 0.0
    assert np.linalg.norm(r) <= 1e-8 * r0


@gpu
def test_solver_failure_and_iteration_guard():
    d = load_golden("as_p1_l3_miehe_t40")
    _, st, solver = build(d)
    solver.krylov = P.KrylovConfig(relative_tolerance=1e-6, max_iterations=1, restart=2)
    with pytest.raises(P.SolverFailure):
        solver.solve_step(st)
    _, st, solver = build(d)
    solver.params = P.ActiveSetParams(tolerance=1e-30, max_iterations=2)
    with pytest.raises(P.SolverFailure):
        solver.solve_step(st)


@gpu
def test_reaction_load_matches_oracle():
    d = load_golden("as_p2_l4_miehe_notch")
    _, st, solver = build(d)
    solver.solve_step(st)
    fx, fy = P.reaction_load(st)
    ost = O.State(2, 4, O.Material(*(float(v) for v in d["material"])), "miehe")
    ost.U, ost.phi_tilde, ost.phi_old = st.U.copy(), st.phi_tilde.copy(), st.phi_old.copy()
    raw = O.residual(ost, mask_dirichlet=False)
    top = ost.lv.boundary_nodes("top")
    n = ost.n
    assert fx == pytest.approx(raw[:n][top].sum(), rel=1e-9, abs=1e-12 * abs(fy))
    assert fy == pytest.approx(raw[n:2 * n][top].sum(), rel=1e-9)
