"""CSV and legacy-VTK writers for simulation output (src/io.py): the same
file formats, byte for byte (LF endings, '.' decimal separator)."""

from __future__ import annotations

from pathlib import Path

import numpy as np

from .mesh import DofMap

CSV_HEADER = ("step,time_s,u_applied_mm,load_x_kN,load_y_kN,as_iters,gmres_iters_total,"
              "active_dofs,wall_s")
BENCH_CSV_HEADER = "kind,degree,level,dofs,best_time_s,reps"


def format_load_row(rec) -> str:
    """One load-displacement row (src/io.py:14-19 formats)."""
    return ",".join([str(rec.step), f"{rec.time_s:.10g}", f"{rec.u_applied_mm:.10g}",
                     f"{rec.load_x_kN:.12g}", f"{rec.load_y_kN:.12g}", str(rec.as_iters),
                     str(rec.gmres_iters_total), str(rec.active_dofs), f"{rec.wall_s:.6g}"])


def _write_lines(lines, path):
    Path(path).write_text("\n".join(lines) + "\n", newline="\n")


def write_load_csv(records, path) -> None:
    _write_lines([CSV_HEADER] + [format_load_row(r) for r in records], path)


def write_bench_csv(records, path) -> None:
    rows = [BENCH_CSV_HEADER]
    rows += [f"{r.kind},{r.degree},{r.level},{r.dofs},{r.best_time_s:.9g},{r.reps}"
             for r in records]
    _write_lines(rows, path)


def vtk_text(dof_map: DofMap, U) -> str:
    """Legacy ASCII unstructured grid (src/io.py:37-80): points are the scalar
    Q_p nodes incl. the slit copies, every cell is written as p x p bilinear
    sub-quads, point data u (vector) and phi."""
    U = np.asarray(U.cpu() if hasattr(U, "cpu") else U)
    n, p = dof_map.n_scalar, dof_map.degree
    n1 = p + 1
    conn = dof_map.conn
    ux, uy, phi = U[:n], U[n:2 * n], U[2 * n:]
    # sub-quad corners (b, a), (b, a+1), (b+1, a+1), (b+1, a) of every cell
    b, a = np.meshgrid(np.arange(p), np.arange(p), indexing="ij")
    corners = np.stack([b * n1 + a, b * n1 + a + 1, (b + 1) * n1 + a + 1, (b + 1) * n1 + a],
                       axis=-1).reshape(-1, 4)
    quads = conn[:, corners].reshape(-1, 4)
    n_sub = quads.shape[0]
    g = "{:.12g}".format
    out = ["# vtk DataFile Version 3.0", "fracturekit snapshot", "ASCII",
           "DATASET UNSTRUCTURED_GRID", f"POINTS {n} double"]
    out += [f"{g(x)} {g(y)} 0" for x, y in dof_map.coords]
    out.append(f"CELLS {n_sub} {5 * n_sub}")
    out += [f"4 {q[0]} {q[1]} {q[2]} {q[3]}" for q in quads.tolist()]
    out.append(f"CELL_TYPES {n_sub}")
    out += ["9"] * n_sub
    out += [f"POINT_DATA {n}", "VECTORS u double"]
    out += [f"{g(x)} {g(y)} 0" for x, y in zip(ux.tolist(), uy.tolist())]
    out += ["SCALARS phi double 1", "LOOKUP_TABLE default"]
    out += [g(v) for v in phi.tolist()]
    return "\n".join(out) + "\n"


def write_vtk(dof_map: DofMap, U, path) -> None:
    Path(path).write_text(vtk_text(dof_map, U), newline="\n")
