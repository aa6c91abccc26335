"""Run the reference's own tests (vendored by prepare.py, git-ignored) through
the drop-in: the ``fracturekit`` modules they import are mapped onto
paper_2005_00331_b200 -- pff_operator -> operator, multigrid -> multigrid,
krylov -> krylov, mesh_hierarchy -> mesh, tensor_basis -> basis -- except
material_model, the point-wise tensor algebra the tests use as their own
oracle (out of scope for the product), which stays the
reference's.  Collected only with PFF_REFSUITE=1 on a CUDA machine: the
product has no CPU path."""

import importlib.util
import os
import sys
import types

HERE = os.path.dirname(os.path.abspath(__file__))
VENDOR = os.path.join(HERE, "_vendor")


def _enabled():
    if os.environ.get("PFF_REFSUITE") != "1" or not os.path.isdir(VENDOR):
        return False
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


collect_ignore_glob = [] if _enabled() else ["_vendor/*"]


def _install_shim():
    import paper_2005_00331_b200 as P
    from paper_2005_00331_b200 import active_set, basis, io, krylov, mesh, multigrid, operator
    from paper_2005_00331_b200 import simulation
    pkg = types.ModuleType("fracturekit")
    pkg.__path__ = []
    sys.modules["fracturekit"] = pkg
    # material_model re-exports the reference's numba lane kernels at import; the
    # tests do not use them and the drop-in does not ship them: stubs that raise
    kern = types.ModuleType("fracturekit._kernels")

    def _absent(*_a, **_k):
        raise NotImplementedError("the reference's numba lane kernels are not part of the drop-in")
    for name in ("eig2_lanes", "positive_part_lanes", "d_positive_part_lanes",
                 "energy_split_lanes", "stress_split_lanes", "d_stress_plus_lanes"):
        setattr(kern, name, _absent)
    sys.modules["fracturekit._kernels"] = kern
    pkg._kernels = kern
    spec = importlib.util.spec_from_file_location("fracturekit.material_model",
                                                  os.path.join(VENDOR, "ref_material_model.py"),
                                                  submodule_search_locations=None)
    mm = importlib.util.module_from_spec(spec)
    sys.modules["fracturekit.material_model"] = mm
    spec.loader.exec_module(mm)
    mods = {"pff_operator": operator, "multigrid": multigrid, "krylov": krylov,
            "mesh_hierarchy": mesh, "tensor_basis": basis, "material_model": mm,
            "active_set_solver": active_set, "simulation_driver": simulation, "io": io}
    for name, mod in mods.items():
        sys.modules[f"fracturekit.{name}"] = mod
        setattr(pkg, name, mod)
    sys.modules["fracturekit"] = pkg
    pkg.__version__ = "drop-in:" + getattr(P, "__version__", "paper_2005_00331_b200")


# reference tests whose subject the drop-in does not ship:
# the command-line wrapper src/cli.py
OUT_OF_SCOPE = {"TestCli": "fracturekit.cli (argument parsing around run_simulation) is out of scope"}


def pytest_collection_modifyitems(config, items):
    import pytest
    for item in items:
        cls = getattr(item, "cls", None)
        if cls is not None and cls.__name__ in OUT_OF_SCOPE:
            item.add_marker(pytest.mark.xfail(reason=OUT_OF_SCOPE[cls.__name__], strict=True))


if _enabled():
    _install_shim()
