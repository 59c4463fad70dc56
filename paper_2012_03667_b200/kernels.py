"""Model parameters of the qDSE sweep (reference kernels.py:36-79).

The integrand itself (row_rhs, kernels.py:178-226) lives in the CUDA library
(csrc/dse_device.cuh: point_exact / point_fast); `row_rhs` here evaluates one
external row through it.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ParameterError

__all__ = ["ModelParams", "row_rhs"]


@dataclass
class ModelParams:
    """D (GeV^2), omega (GeV): Gaussian interaction; m0 current mass; z1
    renormalisation constant; xi convergence accuracy; N, m_rad, m_ang grid
    sizes over [p2_min, p2_max]; relaxation 1.0 = plain substitution."""

    D: float = 0.550
    omega: float = 0.678
    m0: float = 0.0
    z1: float = 1.0
    xi: float = 0.005
    N: int = 150
    m_rad: int = 100
    m_ang: int = 32
    p2_min: float = 1e-6
    p2_max: float = 1e4
    max_iterations: int = 500
    relaxation: float = 1.0

    def validate(self) -> None:
        checks = [
            ("D", self.D >= 0.0),
            ("omega", self.omega > 0.0),
            ("m0", self.m0 >= 0.0),
            ("xi", self.xi > 0.0),
            ("N", self.N >= 2),
            ("M_rad", self.m_rad >= 2),
            ("M_ang", self.m_ang >= 1),
            ("p2_min/p2_max", 0.0 < self.p2_min < self.p2_max),
            ("max_iterations", self.max_iterations >= 1),
            ("relaxation", 0.0 < self.relaxation <= 1.0),
        ]
        for key, good in checks:
            if not good:
                raise ParameterError(f"parameter out of range: {key}")

    @property
    def interaction_coeff(self) -> float:
        """8 pi^2 D / omega^4, evaluated exactly as kernels.py:79 does."""
        return 8.0 * np.pi**2 * self.D / self.omega**4


def row_rhs(p2: float, a_p: float, b_p: float, a_q, b_q, grid, params: ModelParams,
            row: int | None = None) -> tuple[float, float]:
    """(A', B') for one external momentum (kernels.py:178-226), on the GPU.

    One-row sweep through the C ABI (dse_row_rhs) in the exact arithmetic,
    with the caller's dressing values a_q, b_q at the internal nodes.
    """
    from .solver import _row_rhs_gpu
    return _row_rhs_gpu(p2, a_p, b_p, a_q, b_q, grid, params, row)
