"""Nested slit-square meshes with the reference's Q_p scalar numbering.

Closed-form replacement of src/mesh_hierarchy.py (whose per-cell Python
loops take 7 s at 1024^2): the device kernels never read a connectivity
array; ``DofMap.conn`` is materialised lazily (vectorised numpy) only for
callers that ask for it.  Numbering: grid node (i, j) -> j*n1 + i, upper
slit copies appended at n_grid + i (src/mesh_hierarchy.py:156-189).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import cached_property

import numpy as np

BOUNDARY_TAGS = ("bottom", "top", "left", "right")
COMPONENTS = ("u_x", "u_y", "phi")


@dataclass(frozen=True)
class MeshLevel:
    level_index: int

    @property
    def cells_per_side(self) -> int:
        return 2 ** self.level_index

    @property
    def h(self) -> float:
        return 1.0 / self.cells_per_side

    @property
    def n_cells(self) -> int:
        return self.cells_per_side ** 2

    # -- the vertex mesh (src/mesh_hierarchy.py:36-59, 228-276): host-side
    # geometry for topology checks and dumps; the kernels use the closed form
    @cached_property
    def _q1(self) -> "DofMap":
        return DofMap(self.level_index, 1)

    @cached_property
    def vertices(self) -> np.ndarray:
        return self._q1.coords

    @cached_property
    def cells(self) -> np.ndarray:
        """(n_cells, 4) vertex ids, counter-clockwise from the lower-left."""
        return np.ascontiguousarray(self._q1.conn[:, [0, 1, 3, 2]])

    @cached_property
    def boundary_edges(self) -> dict:
        """tag -> (n_edges, 2) vertex pairs along the boundary; left-boundary
        edges above the slit use the upper copy of the slit's end vertex."""
        q = self._q1
        n1, ng, im = q.nodes_per_side, q.n_grid, q.i_mid
        k = np.arange(n1, dtype=np.int64)
        runs = {"bottom": k, "top": (n1 - 1) * n1 + k, "left": k * n1, "right": k * n1 + n1 - 1}
        out = {}
        for tag in BOUNDARY_TAGS:
            e = np.column_stack([runs[tag][:-1], runs[tag][1:]])
            if tag == "left" and q.n_dup:
                e[im:, 0] = np.where(e[im:, 0] == im * n1, ng, e[im:, 0])
            out[tag] = e
        return out

    @cached_property
    def _slit_edges(self):
        q = self._q1
        if not q.n_dup:
            z = np.empty((0, 2), dtype=np.int64)
            return z, z
        tip = q.i_mid * q.nodes_per_side + q.i_mid
        lo = np.append(q.slit_lower, tip)
        up = np.append(q.slit_upper, tip)
        return (np.column_stack([lo[:-1], lo[1:]]).astype(np.int64),
                np.column_stack([up[:-1], up[1:]]).astype(np.int64))

    @property
    def slit_edges_lower(self) -> np.ndarray:
        return self._slit_edges[0]

    @property
    def slit_edges_upper(self) -> np.ndarray:
        return self._slit_edges[1]

    def edge_cell_counts(self) -> dict:
        """Undirected edge (vertex pair) -> number of cells referencing it."""
        c = self.cells
        e = np.stack([c, np.roll(c, -1, axis=1)], axis=2).reshape(-1, 2)
        e.sort(axis=1)
        keys, counts = np.unique(e, axis=0, return_counts=True)
        return {(int(a), int(b)): int(n) for (a, b), n in zip(keys, counts)}


@dataclass(frozen=True)
class DofMap:
    level_index: int
    degree: int

    @property
    def nodes_per_side(self) -> int:
        return self.degree * 2 ** self.level_index + 1

    @property
    def n_grid(self) -> int:
        return self.nodes_per_side ** 2

    @property
    def i_mid(self) -> int:
        return (self.nodes_per_side - 1) // 2

    @property
    def n_dup(self) -> int:
        return self.i_mid if self.level_index >= 1 else 0

    @property
    def n_scalar(self) -> int:
        return self.n_grid + self.n_dup

    @property
    def n_total(self) -> int:
        return 3 * self.n_scalar

    @property
    def n_local(self) -> int:
        return (self.degree + 1) ** 2

    @cached_property
    def conn(self) -> np.ndarray:
        p, ns, n1 = self.degree, 2 ** self.level_index, self.nodes_per_side
        cy, cx = np.divmod(np.arange(ns * ns, dtype=np.int64), ns)
        b, a = np.divmod(np.arange((p + 1) ** 2, dtype=np.int64), p + 1)
        j = cy[:, None] * p + b[None, :]
        i = cx[:, None] * p + a[None, :]
        gid = j * n1 + i
        if self.level_index >= 1:
            up = (cy[:, None] >= ns // 2) & (j == self.i_mid) & (i < self.i_mid)
            gid = np.where(up, self.n_grid + i, gid)
        return gid

    @cached_property
    def coords(self) -> np.ndarray:
        xs = np.arange(self.nodes_per_side) / (self.nodes_per_side - 1)
        gx, gy = np.meshgrid(xs, xs, indexing="xy")
        c = np.column_stack([gx.ravel(), gy.ravel()])
        if self.n_dup:
            c = np.vstack([c, np.column_stack([xs[: self.n_dup], np.full(self.n_dup, 0.5)])])
        return c

    @cached_property
    def boundary_nodes(self) -> dict:
        n1, ng = self.nodes_per_side, self.n_grid
        line = np.arange(n1, dtype=np.int64)
        out = {"bottom": line.copy(), "top": (n1 - 1) * n1 + line,
               "left": line * n1, "right": line * n1 + n1 - 1}
        if self.n_dup:
            out["left"] = np.sort(np.append(out["left"], ng))
        return out

    @property
    def slit_lower(self) -> np.ndarray:
        if not self.n_dup:
            return np.empty(0, dtype=np.int64)
        return self.i_mid * self.nodes_per_side + np.arange(self.n_dup, dtype=np.int64)

    @property
    def slit_upper(self) -> np.ndarray:
        if not self.n_dup:
            return np.empty(0, dtype=np.int64)
        return self.n_grid + np.arange(self.n_dup, dtype=np.int64)


@dataclass
class ConstraintSet:
    """Dirichlet dofs with prescribed values and the active phi dofs, in full
    (3n) dof ids (src/mesh_hierarchy.py:110-153).  Duplicate Dirichlet dofs
    must agree on their value (they are merged); active dofs must be phi dofs.
    The device path keeps the same information as per-node flag bytes."""

    dirichlet_dofs: np.ndarray
    dirichlet_values: np.ndarray
    active_dofs: np.ndarray
    n_total: int

    def __post_init__(self):
        d = np.asarray(self.dirichlet_dofs, dtype=np.int64)
        v = np.asarray(self.dirichlet_values, dtype=np.float64)
        order = np.argsort(d, kind="stable")
        d, v = d[order], v[order]
        if d.size:
            first = np.r_[True, d[1:] != d[:-1]]
            # every repeated dof must carry exactly the value of its first occurrence
            start = np.flatnonzero(first)
            owner = np.repeat(start, np.diff(np.r_[start, d.size]))
            if np.any(v != v[owner]):
                raise ValueError("conflicting Dirichlet values for the same dof")
            d, v = d[first], v[first]
        self.dirichlet_dofs, self.dirichlet_values = d, v
        a = np.asarray(self.active_dofs, dtype=np.int64)
        n = self.n_total // 3
        if a.size and (a.min() < 2 * n or a.max() >= self.n_total):
            raise ValueError("active-set entries must be phi-component dofs")
        self.active_dofs = a

    def kind_of(self, dof: int) -> str:
        if np.any(self.dirichlet_dofs == dof):
            return "dirichlet"
        if np.any(self.active_dofs == dof):
            return "active"
        return "free"

    def constrained_mask(self) -> np.ndarray:
        mask = np.zeros(self.n_total, dtype=bool)
        mask[self.dirichlet_dofs] = True
        mask[self.active_dofs] = True
        return mask


@dataclass
class MeshHierarchy:
    """Levels 0..max_level (src/mesh_hierarchy.py:279-338)."""

    max_level: int
    degree: int
    _injections: dict = field(default_factory=dict, repr=False)

    def level(self, l: int) -> MeshLevel:
        self._check(l)
        return MeshLevel(l)

    def dof_map(self, l: int) -> DofMap:
        self._check(l)
        return DofMap(l, self.degree)

    def _check(self, l):
        if not 0 <= l <= self.max_level:
            raise IndexError(f"level {l} outside 0..{self.max_level}")

    def boundary_dofs(self, level: int, tag: str) -> np.ndarray:
        if tag not in BOUNDARY_TAGS:
            raise ValueError(f"unknown boundary tag {tag!r}")
        dm = self.dof_map(level)
        nodes = dm.boundary_nodes[tag]
        return np.sort(np.concatenate([nodes, dm.n_scalar + nodes]))

    def slit_pairs(self, level: int) -> np.ndarray:
        """(lower, upper) full dof ids of every duplicated slit node, per
        component (src/mesh_hierarchy.py:304-314)."""
        if level < 1:
            raise ValueError("slit duplication starts at level 1")
        dm = self.dof_map(level)
        pairs = [np.column_stack([c * dm.n_scalar + dm.slit_lower, c * dm.n_scalar + dm.slit_upper])
                 for c in range(3)]
        return np.concatenate(pairs).astype(np.int64)

    def dump_level(self, level: int) -> str:
        """One record per line: header, vertices, cells (src/mesh_hierarchy.py:340-349)."""
        mesh, dm = self.level(level), self.dof_map(level)
        out = [f"level {level} cells {mesh.n_cells} scalar_dofs {dm.n_scalar}"]
        out += [f"vertex {i} {x:.12g} {y:.12g}" for i, (x, y) in enumerate(mesh.vertices)]
        out += ["cell {} {}".format(i, " ".join(str(int(v)) for v in c)) for i, c in enumerate(mesh.cells)]
        return "\n".join(out) + "\n"

    def injection(self, fine_level: int) -> np.ndarray:
        """coarse = fine[injection(fine_level)] (src/mesh_hierarchy.py:316-338)."""
        if fine_level in self._injections:
            return self._injections[fine_level]
        if fine_level < 1:
            raise ValueError("level 0 has no coarser level")
        fine, coarse = self.dof_map(fine_level), self.dof_map(fine_level - 1)
        idx = np.arange(coarse.nodes_per_side, dtype=np.int64) * 2
        jj, ii = np.meshgrid(idx, idx, indexing="ij")
        inj = (jj * fine.nodes_per_side + ii).ravel()
        if coarse.n_dup:
            inj = np.append(inj, fine.n_grid + 2 * np.arange(coarse.n_dup, dtype=np.int64))
        self._injections[fine_level] = inj
        return inj


def build_hierarchy(max_level: int, degree: int) -> MeshHierarchy:
    """src/mesh_hierarchy.py:352-366 (closed form, O(1) build)."""
    if max_level < 2:
        raise ValueError("max_level must be >= 2 (coarse solve is on level 2)")
    if degree < 1:
        raise ValueError("degree must be >= 1")
    if degree > 4:
        raise ValueError("degree must be <= 4 on the B200 kernels")
    return MeshHierarchy(max_level=max_level, degree=degree)
