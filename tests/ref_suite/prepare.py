"""Copy the reference's own operator / multigrid / Krylov tests into
tests/ref_suite/_vendor/ (git-ignored; run in the build container, where
/root/reference exists; the copies travel to the GPU box with the snapshot).

Provenance: fracturekit 0.1.0, /root/reference/pkg/tests/test_pff_operator.py,
test_multigrid.py, test_krylov.py, test_mesh_hierarchy.py,
test_active_set_solver.py, test_simulation_driver.py, unmodified
(test_tensor_basis.py and test_material_model.py test the reference's numpy
batch helpers and point-wise algebra, out of scope for the drop-in); and its point-wise tensor algebra
src/fracturekit/material_model.py, which those tests use as their oracle
(out of scope for the product, test infrastructure here).
Nothing under _vendor/ is product code or committed; conftest.py maps the
``fracturekit`` modules the tests import onto paper_2005_00331_b200.

    python tests/ref_suite/prepare.py
    PFF_REFSUITE=1 python -m pytest tests/ref_suite -q     # on a GPU box
"""

import hashlib
import os
import shutil

SRC = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))
VENDOR = os.path.join(HERE, "_vendor")
FILES = {"tests/test_pff_operator.py": "test_pff_operator.py",
         "tests/test_multigrid.py": "test_multigrid.py",
         "tests/test_krylov.py": "test_krylov.py",
         "tests/test_mesh_hierarchy.py": "test_mesh_hierarchy.py",
         "tests/test_active_set_solver.py": "test_active_set_solver.py",
         "tests/test_simulation_driver.py": "test_simulation_driver.py",
         "src/fracturekit/material_model.py": "ref_material_model.py"}


def main():
    os.makedirs(VENDOR, exist_ok=True)
    lines = []
    for src, dst in FILES.items():
        path = os.path.join(SRC, src)
        shutil.copyfile(path, os.path.join(VENDOR, dst))
        with open(path, "rb") as f:
            lines.append(f"{dst}  <- {src}  sha256 {hashlib.sha256(f.read()).hexdigest()}")
    with open(os.path.join(VENDOR, "__init__.py"), "w") as f:
        f.write("")
    with open(os.path.join(VENDOR, "PROVENANCE.txt"), "w") as f:
        f.write("fracturekit 0.1.0 (/root/reference/pkg), copied unmodified by prepare.py\n")
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
