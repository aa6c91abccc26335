"""CPU checks of the C ABI and host logic (no kernel launches)."""

import ctypes
import os
import sys
import re

import numpy as np
import pytest

from conftest import ROOT
import paper_2005_00331_b200 as P
from paper_2005_00331_b200 import _lib
from oracle import oracle as O


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "pff_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(pff_\w+)\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    L = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_abi_version_and_host_only_calls():
    L = _lib.load()
    assert L.pff_abi_version() == 1
    assert L.pff_reduce_scratch_len() > 0
    s = P.shape_data(2)
    h = ctypes.c_void_p()
    mat = _lib.material(P.MaterialParams())
    E = s.embedding()
    rc = L.pff_level_create(ctypes.byref(h), 2, 10, 1, ctypes.byref(mat), s.values.ctypes.data,
                            s.derivatives.ctypes.data, s.quad_weights.ctypes.data, E.ctypes.data)
    assert rc == 0
    assert L.pff_level_n_scalar(h) == 4_199_425
    assert L.pff_level_n_cells(h) == 1024 * 1024
    # generic cache + strip-tiled Q2 tangent cache (34 strips x 1024 rows x 7 Miehe arrays x 9 q
    # x 32 lanes) + element-vector scratch (3 components x 9 nodes per cell)
    assert L.pff_level_qcache_len(h) == (6 * 9 * 1024 * 1024 + 34 * 1024 * 7 * 9 * 32
                                         + 3 * 9 * 1024 * 1024)
    rows = (ctypes.c_int64 * 6)()
    assert L.pff_level_set_window(h, 256, 512) == 0
    assert L.pff_level_window(h, rows) == 0
    assert list(rows) == [510, 1024, 1, 515 * 2049, 256, 512]
    assert L.pff_level_n_scalar(h) == (1024 - 510 + 1) * 2049 + 1024
    assert L.pff_level_set_window(h, 0, 1024) == 0
    assert L.pff_level_n_scalar(h) == 4_199_425
    assert L.pff_level_set_window(h, 10, 5) < 0
    # unbound state is an error, not a crash
    assert L.pff_apply(h, 0, None, None, None, None) < 0
    assert b"not bound" in L.pff_last_error()
    L.pff_level_destroy(h)
    bad = L.pff_level_create(ctypes.byref(h), 7, 3, 0, ctypes.byref(mat), s.values.ctypes.data,
                             s.derivatives.ctypes.data, s.quad_weights.ctypes.data, None)
    assert bad == _lib.load().pff_level_create.restype(-1) or bad < 0


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_shape_data_matches_oracle(p):
    a, b = P.shape_data(p), O.shape(p)
    assert np.array_equal(a.values, b.N) and np.array_equal(a.derivatives, b.D)
    assert np.array_equal(a.quad_weights, b.w)


@pytest.mark.parametrize("p,level", [(1, 0), (1, 3), (2, 1), (2, 5), (3, 3), (4, 4)])
def test_closed_form_numbering(p, level):
    dm = P.build_hierarchy(max(level, 2), p).dof_map(level)
    lv = O.Level(p, level)
    assert dm.n_scalar == lv.n
    assert np.array_equal(dm.conn, lv.conn())
    for tag in ("top", "bottom", "left", "right"):
        assert np.array_equal(dm.boundary_nodes[tag], lv.boundary_nodes(tag))


def test_dof_counts_match_configs():
    assert 3 * P.build_hierarchy(5, 2).dof_map(5).n_scalar == 12_771
    assert 3 * P.build_hierarchy(10, 2).dof_map(10).n_scalar == 12_598_275
    assert 3 * P.build_hierarchy(9, 4).dof_map(9).n_scalar == 12_598_275
    assert 3 * P.build_hierarchy(12, 2).dof_map(12).n_scalar == 201_388_035


@pytest.mark.parametrize("p", [1, 2, 3])
def test_injection_and_prolongation_matrix(golden, p):
    d = golden(f"transfer_p{p}_l4")
    h = P.build_hierarchy(4, p)
    assert np.array_equal(h.injection(4), d["inj"])
    Pm = P.build_prolongation(h, 4)
    assert np.array_equal(Pm.indptr, d["P_indptr"]) and np.array_equal(Pm.indices, d["P_indices"])
    assert np.array_equal(Pm.data, d["P_data"])


def test_config_validation():
    with pytest.raises(ValueError):
        P.KrylovConfig(relative_tolerance=1.5)
    with pytest.raises(ValueError):
        P.KrylovConfig(restart=1)
    with pytest.raises(ValueError):
        P.ChebyshevConfig(c=2.0)
    with pytest.raises(ValueError):
        P.build_hierarchy(1, 2)
    with pytest.raises(ValueError):
        P.MaterialParams(mu=-1.0)
    h = P.build_hierarchy(2, 1)
    with pytest.raises(ValueError):
        P.GmgPreconditioner(h, coarse_level=3)
    with pytest.raises(ValueError):
        P.LinearizationState(h, 2, P.MaterialParams(), split="bogus")
    with pytest.raises(ValueError):
        P.LinearizationState(h, 2, P.MaterialParams(), lane_width=3)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = P.build_hierarchy(2, 1)
    st = P.LinearizationState(h, 2, P.MaterialParams())
    with pytest.raises(RuntimeError, match="CUDA"):
        st.refresh_cache()


def test_host_argument_checks_of_session2_entries():
    """The new entry points reject bad arguments on the host (no launch)."""
    L = _lib.load()
    nul = ctypes.c_void_p(0)
    # pff_dense_matvec: rows/cols >= 1, non-null, x != y
    assert L.pff_dense_matvec(0, 4, nul, nul, nul, nul) != 0
    buf = ctypes.c_void_p(0x1000)
    assert L.pff_dense_matvec(4, 4, buf, buf, buf, nul) != 0          # x == y
    # pff_coarse_dense: n in 1..256
    assert L.pff_coarse_dense(0, buf, buf, buf, buf, buf, buf, nul) != 0
    assert L.pff_coarse_dense(257, buf, buf, buf, buf, buf, buf, nul) != 0
    # pff_apply_cheb_ex / pff_apply_emit / pff_smooth_init on an unbound level
    s = P.shape_data(2)
    h = ctypes.c_void_p()
    mat = _lib.material(P.MaterialParams())
    E = s.embedding()
    assert L.pff_level_create(ctypes.byref(h), 2, 6, 1, ctypes.byref(mat), s.values.ctypes.data,
                              s.derivatives.ctypes.data, s.quad_weights.ctypes.data,
                              E.ctypes.data) == 0
    try:
        assert L.pff_apply_cheb_ex(h, 1, buf, buf, buf, buf, buf, buf, ctypes.c_double(1.0),
                                   ctypes.c_double(1.0), 0, nul) != 0
        assert L.pff_apply_emit(h, 0, buf, buf, buf, buf, buf, ctypes.c_double(1.0), nul) != 0
        assert L.pff_smooth_init(h, buf, buf, buf, buf, buf, ctypes.c_double(1.0), nul) != 0
        assert L.pff_apply_host(h, 0, buf, buf, buf, buf, 0, nul) != 0     # unbound
    finally:
        L.pff_level_destroy(h)
    assert b"bad argument" in L.pff_last_error() or b"not bound" in L.pff_last_error()


def test_newton_floor_model():
    """bench.py's HBM-floor model of the Newton solve scales with
    the node count and the GPU count."""
    import bench
    n = 67_129_345                    # configs[4] scalar nodes
    a = bench.newton_floor(n, 28, 1, 1.0)
    b = bench.newton_floor(n, 28, 4, 1.0)
    assert abs(a["floor_s"] / b["floor_s"] - 4.0) < 0.01
    per_node = sum(2530 + 81 + 72 * (j + 2) for j in range(28))
    peak, _ = bench.peaks()
    assert abs(a["floor_s"] - n * per_node / (peak * 1e9)) < 1e-4
    assert abs(a["frac"] - a["floor_s"]) < 1e-3   # t = 1 s


def test_integration_doc_names_every_entry_point():
    """INTEGRATION.md maps every exported entry point to the reference
    interface it replaces (or says it has none)."""
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    missing = [s for s in header_symbols() if s not in doc]
    assert not missing, missing


def test_bench_gpus_flag_launches_its_own_ranks(monkeypatch):
    """bench.py --gpus N without WORLD_SIZE re-launches itself under
    torch.distributed.run with N local ranks on 127.0.0.1; under torchrun a
    WORLD_SIZE different from --gpus is an error."""
    import subprocess
    import bench
    seen = {}

    def fake_call(cmd):
        seen["cmd"] = cmd
        return 0
    monkeypatch.setattr(subprocess, "call", fake_call)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "5"])
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert e.value.code == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "5"][-3:]
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4"])
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert "WORLD_SIZE" in str(e.value.code)


def test_scaling_model_uses_the_slab_rule():
    """tools/scaling_model.py: the slab levels it models are the ones
    distributed.DistributedGmg builds, and more GPUs never model slower."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import scaling_model as SM
    from paper_2005_00331_b200 import distributed as D

    class _H:
        degree = 2
    import torch
    for world in (2, 4, 8):
        g = D.DistributedGmg(_H(), 12, 0, world, coarse_level=2, device=torch.device("cpu"))
        assert SM.slab_levels(12, world) == g.slab_levels
    d = {"iterations": 82, "operator_s": 2.6e-3, "ortho_s": 12e-3,
         "levels": [{"level": l, "floor_s": 95e-6, "prop_s": 0.37e-9 * (2 * 2 ** l + 1) ** 2}
                    for l in range(4, 13)] + [{"level": 3, "floor_s": 8e-6, "prop_s": 0.0}]}
    t = [SM.model(d, n)["gmres_s"] for n in (1, 2, 4, 8)]
    assert t[0] > t[1] > t[2] > t[3]
    assert SM.slab_levels(12, 8) == [12, 11, 10, 9, 8, 7]


@pytest.mark.parametrize("level", [1, 2, 3])
def test_vertex_mesh_topology(level):
    """MeshLevel's vertex mesh (src/mesh_hierarchy.py:36-59): boundary and slit
    edges belong to one cell, every other edge to two; dump_level has one
    record per line."""
    h = P.build_hierarchy(max(level, 2), 1)
    mesh = h.level(level)
    counts = mesh.edge_cell_counts()
    single = {tuple(sorted(map(int, e))) for es in mesh.boundary_edges.values() for e in es}
    single |= {tuple(sorted(map(int, e))) for e in mesh.slit_edges_lower}
    single |= {tuple(sorted(map(int, e))) for e in mesh.slit_edges_upper}
    for e, c in counts.items():
        assert c == (1 if e in single else 2), e
    assert len(h.dump_level(level).strip().split("\n")) == 1 + len(mesh.vertices) + mesh.n_cells
    assert h.slit_pairs(level).shape == (3 * h.dof_map(level).n_dup, 2)
