"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container only (it imports fracturekit from
/root/reference/pkg/src, which does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Inputs are the BASELINE.json synthetic draws:
rng = default_rng(seed), u0 ~ U[-1e-3, 1e-3] (2n) -> phi0 ~ U[0,1] (n) ->
x ~ U[-1,1] (3n); phi_tilde = phi_old = phi0; active = phi0 < 0.05;
Dirichlet = top + bottom nodes; lambda=121.15e3, mu=80.77e3, Gc=2.7,
kappa=1e-10, eps=2h.  The fixtures store inputs and outputs so the tests
never need the reference at run time.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import fracturekit.pff_operator as op  # noqa: E402
from fracturekit.krylov import KrylovConfig, gmres_solve  # noqa: E402
from fracturekit.material_model import MaterialParams  # noqa: E402
from fracturekit.mesh_hierarchy import build_hierarchy  # noqa: E402
from fracturekit.multigrid import (ChebyshevConfig, GmgPreconditioner,  # noqa: E402
                                   TransferOperator, chebyshev_apply,
                                   estimate_lambda_range)
from fracturekit.active_set_solver import (ActiveSetParams, ActiveSetSolver,  # noqa: E402
                                           lumped_mass_diagonal)
from fracturekit.simulation_driver import (ScenarioConfig, apply_boundary_values,  # noqa: E402
                                           boundary_program, memory_report, run_simulation)
from fracturekit import io as ref_io  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def params(level):
    return MaterialParams(lame_lambda=121.15e3, mu=80.77e3, g_c=2.7, kappa=1e-10,
                          eps=2.0 / 2 ** level)


def notch(dm, eps):
    x, y = dm.coords[:, 0], dm.coords[:, 1]
    dx = np.maximum(x - 0.5, 0.0)
    return 1.0 - np.exp(-np.sqrt(dx * dx + (y - 0.5) ** 2) / eps)


def make(h, level, split, seed, notch_phi=False):
    st = op.LinearizationState(h, level, params(level), split=split)
    dm = h.dof_map(level)
    n = st.n_scalar
    rng = np.random.default_rng(seed)
    u0 = rng.uniform(-1e-3, 1e-3, 2 * n)
    phi0 = notch(dm, params(level).eps) if notch_phi else rng.uniform(0.0, 1.0, n)
    x = rng.uniform(-1.0, 1.0, 3 * n)
    st.set_solution(np.concatenate([u0, phi0]))
    st.set_phi_tilde(phi0)
    st.set_phi_old(phi0)
    st.set_active(phi0 < 0.05)
    st.set_dirichlet_nodes(np.unique(np.concatenate(
        [dm.boundary_nodes["top"], dm.boundary_nodes["bottom"]])))
    st.refresh_cache()
    return st, x


def inputs(st, x):
    return dict(U=st.U.copy(), phi_tilde=st.phi_tilde.copy(), phi_old=st.phi_old.copy(),
                active=st.active.copy(), dirichlet=st.dirichlet_nodes.copy(), x=x)


def operator_case(p, level, split, seed, with_cache=False):
    h = build_hierarchy(max(level, 2), p)
    st, x = make(h, level, split, seed)
    n = st.n_scalar
    d = inputs(st, x)
    d["jac"] = op.apply_jacobian(st, x)
    d["uu"] = op.apply_block_uu(st, x[:2 * n])
    d["pp"] = op.apply_block_phiphi(st, x[2 * n:])
    d["prow"] = op.apply_phi_row(st, x)
    d["diag_uu"] = op.block_diagonal(st, "uu")
    d["diag_pp"] = op.block_diagonal(st, "phiphi")
    d["residual"] = op.residual(st)
    d["residual_raw"] = op.residual(st, mask_dirichlet=False)
    if with_cache:
        for k, v in st.cache().items():
            if k not in ("C", "gs"):
                d["cache_" + k] = v.ravel().copy()
    d["meta"] = np.array([p, level, seed, 1 if split == "miehe" else 0])
    return d


def solver_case(p, level, split, seed, notch_phi, sweeps=3):
    h = build_hierarchy(level, p)
    st, x = make(h, level, split, seed, notch_phi)
    n = st.n_scalar
    d = inputs(st, x)
    gmg = GmgPreconditioner(h, coarse_level=2, cheb=ChebyshevConfig(sweeps=sweeps))
    gmg.setup(st)
    for l, rg in gmg.ranges.items():
        d[f"range_{l}"] = np.array([rg["uu"][0], rg["uu"][1], rg["phiphi"][0], rg["phiphi"][1]])
    d["vcycle"] = gmg.apply(x)
    # Chebyshev on the finest uu block with the smoothing interval
    lo, hi = gmg.ranges[level]["uu"]
    d["cheb_uu"] = chebyshev_apply(lambda v: op.apply_block_uu(st, v), gmg.diags[level]["uu"],
                                   x[:2 * n], 0.24 * hi, 1.2 * hi, 5)
    d["lanczos_uu"] = np.array(estimate_lambda_range(
        lambda v: op.apply_block_uu(st, v), gmg.diags[level]["uu"], seed=7))
    rhs = x.copy()
    rhs[st.constrained_mask()] = 0.0
    res = gmres_solve(lambda v: op.apply_jacobian(st, v), rhs,
                      KrylovConfig(relative_tolerance=1e-8, restart=50),
                      preconditioner=gmg.apply)
    d["gmres_x"] = res.solution
    d["gmres_iters"] = np.array([res.iterations])
    d["gmres_hist"] = np.array(res.residual_history)
    d["gmres_conv"] = np.array([int(res.converged)])
    d["meta"] = np.array([p, level, seed, 1 if split == "miehe" else 0, int(notch_phi), sweeps])
    return d


def transfer_case(p, fine_level, seed):
    h = build_hierarchy(max(fine_level, 2), p)
    tr = TransferOperator(h, fine_level)
    rng = np.random.default_rng(seed)
    xc = rng.uniform(-1, 1, 3 * tr.n_coarse)
    yf = rng.uniform(-1, 1, 3 * tr.n_fine)
    inj = h.injection(fine_level)
    return dict(xc=xc, yf=yf, Px=tr.prolongate(xc), Ry=tr.restrict(yf), inj=inj,
                P_indptr=tr.P.indptr, P_indices=tr.P.indices, P_data=tr.P.data,
                meta=np.array([p, fine_level, seed]))


def restrict_case(p, level, target, seed):
    h = build_hierarchy(level, p)
    st, x = make(h, level, "miehe", seed)
    c = op.restrict_state_to_level(st, target)
    d = inputs(st, x)
    d.update(cU=c.U, cphi_tilde=c.phi_tilde, cactive=c.active, cdirichlet=c.dirichlet_nodes,
             meta=np.array([p, level, target, seed]))
    return d


def activeset_case(p, level, split, t, du, notch_phi, baseline_material):
    """One ActiveSetSolver.solve_step (src/active_set_solver.py:101-163) from a
    tension load step; the reference tests' default material, or the BASELINE
    material with a pre-cracked (notch) phase field."""
    h = build_hierarchy(level, p)
    prm = params(level) if baseline_material else MaterialParams()
    st = op.LinearizationState(h, level, prm, split=split)
    n = st.n_scalar
    if notch_phi:
        phi0 = notch(h.dof_map(level), prm.eps)
        U = st.U.copy()
        U[2 * n:] = phi0
        st.set_solution(U)
        st.set_phi_tilde(phi0)
        st.set_phi_old(phi0)
    apply_boundary_values(st, boundary_program("tension", t, du))
    d = dict(U0=st.U.copy(), phi_tilde=st.phi_tilde.copy(), phi_old=st.phi_old.copy(),
             dirichlet=st.dirichlet_nodes.copy())
    m = lumped_mass_diagonal(h, level)
    gmg = GmgPreconditioner(h, coarse_level=2)
    solver = ActiveSetSolver(gmg, KrylovConfig(), ActiveSetParams(), m)
    rep = solver.solve_step(st)
    d.update(m=m, U=st.U.copy(), active=st.active.copy(),
             as_iterations=np.array([rep.as_iterations]),
             gmres_iterations=np.array(rep.gmres_iterations),
             active_counts=np.array(rep.active_counts),
             residual_norms=np.array(rep.residual_norms),
             converged=np.array([int(rep.converged)]),
             material=np.array([prm.lame_lambda, prm.mu, prm.g_c, prm.kappa, prm.eps]),
             meta=np.array([p, level, 1 if split == "miehe" else 0, int(notch_phi)]),
             load=np.array([t, du]))
    print(f"activeset p{p} l{level} {split}: as {rep.as_iterations} gmres {rep.gmres_iterations}"
          f" active {rep.active_counts}")
    return d


ACTIVESET = {
    "as_p1_l3_miehe_t40": (1, 3, "miehe", 40.0, 1e-5, False, False),
    "as_p1_l4_miehe_t1": (1, 4, "miehe", 1.0, 1e-5, False, False),
    "as_p2_l4_miehe_notch": (2, 4, "miehe", 1.0, 3e-3, True, True),
    "as_p2_l6_none_notch": (2, 6, "none", 1.0, 3e-3, True, True),
    "as_p2_l6_miehe_notch": (2, 6, "miehe", 1.0, 3e-3, True, True),
}


def simulation_case(scenario, level, degree, split, steps, du, vtk_every):
    """run_simulation (src/simulation_driver.py:189-259) on a small mesh."""
    cfg = ScenarioConfig(scenario=scenario, level=level, degree=degree, split=split, steps=steps,
                         du=du, vtk_every=vtk_every)
    res = run_simulation(cfg)
    rec = res.records
    d = dict(step=np.array([r.step for r in rec]), time_s=np.array([r.time_s for r in rec]),
             u=np.array([r.u_applied_mm for r in rec]),
             load_x=np.array([r.load_x_kN for r in rec]),
             load_y=np.array([r.load_y_kN for r in rec]),
             as_iters=np.array([r.as_iters for r in rec]),
             gmres_total=np.array([r.gmres_iters_total for r in rec]),
             active_dofs=np.array([r.active_dofs for r in rec]),
             snap_steps=np.array([s for s, _ in res.snapshots]),
             U_final=res.snapshots[-1][1],
             bounds=np.array([res.irreversibility_violation, res.phi_min, res.phi_max]),
             meta=np.array([level, degree, 1 if split == "miehe" else 0, steps, vtk_every,
                            0 if scenario == "tension" else 1]),
             du=np.array([du]))
    h = build_hierarchy(level, degree)
    d["vtk"] = np.frombuffer(ref_io.vtk_text(h.dof_map(level), res.snapshots[-1][1]).encode(),
                             dtype=np.uint8)
    print(f"simulation {scenario} p{degree} l{level} {split}: as {d['as_iters'].tolist()} "
          f"gmres {d['gmres_total'].tolist()} active {d['active_dofs'].tolist()}")
    return d


def assembled_case(p, level, split, seed):
    """cell_matrices / assemble_oracle (src/pff_operator.py:328-377)."""
    h = build_hierarchy(max(level, 2), p)
    st, x = make(h, level, split, seed)
    d = inputs(st, x)
    d["gk"] = op.cell_matrices(st)
    mat = op.assemble_oracle(st).matrix
    d["Ax"] = mat @ x
    d["nnz"] = np.array([mat.nnz])
    d["meta"] = np.array([p, level, seed, 1 if split == "miehe" else 0])
    return d


def memory_case():
    rows = []
    for level, degree in ((3, 2), (5, 1), (5, 4), (3, 4)):
        rep = memory_report(ScenarioConfig(scenario="tension", level=level, degree=degree, steps=1))
        rows.append([level, degree, rep.dofs, rep.csr_bytes])
    return dict(rows=np.array(rows, dtype=np.int64))


SIMULATION = {
    "sim_tension_p1_l3_miehe": ("tension", 3, 1, "miehe", 4, 1e-5, 2),
    "sim_shear_p2_l3_none": ("shear", 3, 2, "none", 3, 1e-5, 0),
    "sim_tension_p1_l4_miehe_fast": ("tension", 4, 1, "miehe", 6, 2e-3, 3),
}


sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from conftest import sketch  # noqa: E402  (the tests recompute it from the device result)


def production_case(p, level, split, seed, full, gmres=True, restart=50, sweeps=3):
    """The configs[3] Newton-step inputs (notch phi0) at `level`, solved by the
    reference (src/multigrid.py:228-344 + src/krylov.py:37-119).  full=True
    stores the V-cycle and GMRES vectors; otherwise only their sketches."""
    import time
    h = build_hierarchy(level, p)
    st, x = make(h, level, split, seed, True)
    n = st.n_scalar
    t0 = time.perf_counter()
    gmg = GmgPreconditioner(h, coarse_level=2, cheb=ChebyshevConfig(sweeps=sweeps))
    gmg.setup(st)
    d = {"setup_s": np.array([time.perf_counter() - t0])}
    for l, rg in gmg.ranges.items():
        d[f"range_{l}"] = np.array([rg["uu"][0], rg["uu"][1], rg["phiphi"][0], rg["phiphi"][1]])
    t0 = time.perf_counter()
    z = gmg.apply(x)
    d["vcycle_s"] = np.array([time.perf_counter() - t0])
    if full:
        d["vcycle"] = z
    else:
        for k, v in sketch(z, n).items():
            d["vcycle_" + k] = v
    if gmres:
        rhs = x.copy()
        rhs[st.constrained_mask()] = 0.0
        t0 = time.perf_counter()
        res = gmres_solve(lambda v: op.apply_jacobian(st, v), rhs,
                          KrylovConfig(relative_tolerance=1e-8, restart=restart),
                          preconditioner=gmg.apply)
        d["gmres_s"] = np.array([time.perf_counter() - t0])
        d["gmres_iters"] = np.array([res.iterations])
        d["gmres_hist"] = np.array(res.residual_history)
        d["gmres_conv"] = np.array([int(res.converged)])
        if full:
            d["gmres_x"] = res.solution
        else:
            for k, v in sketch(res.solution, n).items():
                d["gmres_x_" + k] = v
    d["meta"] = np.array([p, level, seed, 1 if split == "miehe" else 0, 1, sweeps, restart])
    return d


def main():
    if "--production" in sys.argv:   # production-size pins (the configs[3] inputs)
        # python make_golden.py --production LEVEL SPLIT {full|sketch|vcycle} [RESTART]
        i = sys.argv.index("--production")
        level, split, kind = int(sys.argv[i + 1]), sys.argv[i + 2], sys.argv[i + 3]
        restart = int(sys.argv[i + 4]) if len(sys.argv) > i + 4 else 50
        d = production_case(2, level, split, 0, full=(kind == "full"),
                            gmres=(kind != "vcycle"), restart=restart)
        tag = "" if restart == 50 else f"_r{restart}"
        name = f"prod_p2_l{level}_{split}{tag}" + ("_vcycle" if kind == "vcycle" else "")
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
        print(name, {k: v.tolist() for k, v in d.items()
                     if k.endswith(("_s", "iters")) or k.startswith("range_")})
        return
    if "--assembled" in sys.argv:   # only the assembled-path fixtures
        for p, level, split, seed in ((2, 2, "miehe", 4), (2, 2, "none", 4), (1, 3, "miehe", 8),
                                      (3, 2, "miehe", 2)):
            np.savez_compressed(os.path.join(OUT, f"asm_p{p}_l{level}_{split}.npz"),
                                **assembled_case(p, level, split, seed))
        np.savez_compressed(os.path.join(OUT, "memory_report.npz"), **memory_case())
        return
    if "--simulation" in sys.argv:   # only the run_simulation fixtures
        for name, args in SIMULATION.items():
            np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **simulation_case(*args))
        return
    if "--activeset" in sys.argv:   # only the active-set fixtures
        for name, args in ACTIVESET.items():
            np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **activeset_case(*args))
        return
    cases = {}
    for name, args in ACTIVESET.items():
        cases[name] = activeset_case(*args)
    for name, args in SIMULATION.items():
        cases[name] = simulation_case(*args)
    for split in ("none", "miehe"):
        cases[f"pr1_{split}"] = operator_case(2, 5, split, 0, with_cache=True)
        for p in (1, 3, 4):
            cases[f"op_p{p}_l3_{split}"] = operator_case(p, 3, split, p)
        cases[f"op_p2_l1_{split}"] = operator_case(2, 1, split, 5)
        cases[f"op_p1_l0_{split}"] = operator_case(1, 0, split, 6)
        cases[f"solve_p2_l5_{split}_rand"] = solver_case(2, 5, split, 0, False)
        cases[f"solve_p2_l5_{split}_notch"] = solver_case(2, 5, split, 0, True)
    cases["solve_p1_l4_miehe_notch_s5"] = solver_case(1, 4, "miehe", 1, True, sweeps=5)
    for p in (1, 2, 3, 4):
        cases[f"transfer_p{p}_l4"] = transfer_case(p, 4, 10 + p)
    cases["transfer_p2_l1"] = transfer_case(2, 1, 9)
    cases["restrict_p2_l5_l2"] = restrict_case(2, 5, 2, 3)
    for p in (1, 2, 4):
        h = build_hierarchy(3, p)
        cases[f"mass_p{p}_l3"] = dict(m=lumped_mass_diagonal(h, 3), meta=np.array([p, 3]))
    for name, d in cases.items():
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
        print(name, {k: np.asarray(v).shape for k, v in d.items() if k.startswith(("gmres_iters", "meta"))},
              d.get("gmres_iters", ""))


if __name__ == "__main__":
    main()
