"""Assembled-Jacobian comparison path (src/pff_operator.py:
328-377, src/simulation_driver.py:288-393) against the reference's fixtures
(tests/golden/asm_*.npz, memory_report.npz) and the matrix-free operator."""

import numpy as np
import pytest

from conftest import block_rel, load_golden, rel_l2
import paper_2005_00331_b200 as P
from paper_2005_00331_b200 import io as pio

pytestmark = pytest.mark.gpu
ASM = ["asm_p2_l2_miehe", "asm_p2_l2_none", "asm_p1_l3_miehe", "asm_p3_l2_miehe"]


def state_of(d, split):
    p, level = int(d["meta"][0]), int(d["meta"][1])
    h = P.build_hierarchy(max(level, 2), p)
    st = P.LinearizationState(h, level, P.MaterialParams(lame_lambda=121.15e3, mu=80.77e3, g_c=2.7,
                                                         kappa=1e-10, eps=2.0 / 2 ** level),
                              split=split)
    st.set_solution(d["U"])
    st.set_phi_tilde(d["phi_tilde"])
    st.set_phi_old(d["phi_old"])
    st.set_active(d["active"])
    st.set_dirichlet_nodes(np.flatnonzero(d["dirichlet"]))
    st.refresh_cache()
    return st


@pytest.mark.parametrize("name", ASM)
def test_cell_matrices_and_assembly_match_reference(name):
    d = load_golden(name)
    split = "miehe" if int(d["meta"][3]) else "none"
    st = state_of(d, split)
    gk = P.cell_matrices(st)
    assert gk.shape == d["gk"].shape
    # per component block of the local matrices (the phi rows are ~1e3x smaller)
    nl = st.dof_map.n_local
    for r in range(3):
        for c in range(3):
            blk = (slice(None), slice(r * nl, (r + 1) * nl), slice(c * nl, (c + 1) * nl))
            want = d["gk"][blk]
            if np.abs(want).max() == 0.0:
                assert np.abs(gk[blk]).max() == 0.0
            else:
                assert rel_l2(gk[blk], want) <= 1e-12, (r, c)
    orc = P.assemble_oracle(st)
    assert orc.nnz == int(d["nnz"][0]) and orc.state_version == st.version
    n = st.n_scalar
    assert max(block_rel(orc.matvec(d["x"]), d["Ax"], n)) <= 1e-12
    assert max(block_rel(orc.matrix @ d["x"], d["Ax"], n)) <= 1e-12


@pytest.mark.parametrize("degree", [1, 2, 3])
@pytest.mark.parametrize("level", [2, 3])
@pytest.mark.parametrize("split", ["none", "miehe"])
def test_matrix_free_matches_assembled(degree, level, split):
    # the reference's test_matches_assembled_oracle
    rng = np.random.default_rng(degree + level)
    h = P.build_hierarchy(level, degree)
    st = P.LinearizationState(h, level, P.MaterialParams(), split=split)
    n = st.n_scalar
    U = np.concatenate([rng.uniform(-1e-3, 1e-3, 2 * n), rng.uniform(0.2, 1.0, n)])
    st.set_solution(U)
    st.set_phi_tilde(U[2 * n:])
    st.set_active(rng.random(n) < 0.1)
    st.set_dirichlet_nodes(h.dof_map(level).boundary_nodes["bottom"])
    st.refresh_cache()
    mat = P.assemble_oracle(st)
    for _ in range(3):
        dvec = rng.standard_normal(3 * n)
        got, want = P.apply_jacobian(st, dvec), mat.matvec(dvec)
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


def test_memory_report_csr_bytes_match_reference():
    for level, degree, dofs, csr in load_golden("memory_report")["rows"].tolist():
        rep = P.memory_report(P.ScenarioConfig(scenario="tension", level=level, degree=degree,
                                               steps=1))
        assert rep.dofs == dofs and rep.csr_bytes == csr
        assert rep.mf_bytes > 0


def test_memory_report_directional_ratios():
    rep1 = P.memory_report(P.ScenarioConfig(scenario="tension", level=5, degree=1, steps=1))
    rep4 = P.memory_report(P.ScenarioConfig(scenario="tension", level=5, degree=4, steps=1))
    assert rep4.csr_bytes_per_dof / rep1.csr_bytes_per_dof >= 3.5
    assert rep4.mf_bytes_per_dof <= 2.0 * rep1.mf_bytes_per_dof


def test_benchmark_vmult_records_and_csv(tmp_path):
    cfg = P.ScenarioConfig(scenario="tension", level=3, degree=2, steps=1)
    recs = P.benchmark_vmult(cfg, reps=5)
    assert {r.kind for r in recs} == {"spmv", "mfmv", "assemble"}
    for r in recs:
        assert r.best_time_s > 0 and r.dofs == 3 * P.build_hierarchy(3, 2).dof_map(3).n_scalar
    pio.write_bench_csv(recs, tmp_path / "bench.csv")
    lines = (tmp_path / "bench.csv").read_text().strip().split("\n")
    assert lines[0] == "kind,degree,level,dofs,best_time_s,reps" and len(lines) == 4
