"""Shape data and material parameters (host side, tiny tables).

Mirrors src/tensor_basis.py:16-81 and src/material_model.py:20-44 of the
reference so the kernels receive bit-identical N, D, w tables.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

LANE_WIDTHS = (1, 2, 4, 8)   # accepted for API compatibility; SIMT has no lanes


def gauss_legendre_01(q: int):
    pts, wts = np.polynomial.legendre.leggauss(q)
    return 0.5 * (pts + 1.0), 0.5 * wts


def support_points_01(degree: int) -> np.ndarray:
    if degree < 1:
        raise ValueError("degree must be >= 1")
    return np.linspace(0.0, 1.0, degree + 1)


def lagrange_matrices(support: np.ndarray, points: np.ndarray):
    n = support.size
    coeff = np.linalg.inv(np.vander(support, n, increasing=True))
    powers = np.vander(points, n, increasing=True)
    dpowers = np.zeros_like(powers)
    dpowers[:, 1:] = powers[:, :-1] * np.arange(1, n)
    return powers @ coeff, dpowers @ coeff


@dataclass(frozen=True)
class ShapeData:
    degree: int
    quad_points: np.ndarray
    quad_weights: np.ndarray
    support_points: np.ndarray
    values: np.ndarray
    derivatives: np.ndarray

    @property
    def q(self) -> int:
        return self.quad_points.size

    def embedding(self) -> np.ndarray:
        """(2, p+1, p+1): coarse basis at the child support points
        (src/multigrid.py:58-61)."""
        sup = self.support_points
        return np.ascontiguousarray(np.stack(
            [lagrange_matrices(sup, (child + sup) / 2.0)[0] for child in (0, 1)]))


_SHAPES: dict = {}


def shape_data(degree: int) -> ShapeData:
    if degree < 1:
        raise ValueError("degree must be >= 1")
    if degree not in _SHAPES:
        pts, wts = gauss_legendre_01(degree + 1)
        sup = support_points_01(degree)
        N, D = lagrange_matrices(sup, pts)
        _SHAPES[degree] = ShapeData(degree, pts, wts, sup, np.ascontiguousarray(N),
                                    np.ascontiguousarray(D))
    return _SHAPES[degree]


@dataclass(frozen=True)
class MaterialParams:
    """Material and regularisation parameters (src/material_model.py:20-44)."""

    lame_lambda: float = 121.15
    mu: float = 80.77
    g_c: float = 2.7e-3
    kappa: float = 1e-10
    eps: float = 4e-3

    def __post_init__(self):
        if self.mu <= 0:
            raise ValueError("mu must be positive")
        if self.lame_lambda < 0:
            raise ValueError("lame_lambda must be nonnegative")
        if self.g_c <= 0:
            raise ValueError("g_c must be positive")
        if not 0 < self.kappa < 1:
            raise ValueError("kappa must lie in (0, 1)")
        if self.eps <= 0:
            raise ValueError("eps must be positive")
