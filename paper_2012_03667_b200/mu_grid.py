"""Finite chemical potential (BASELINE configs 3-4): parameters and grids.

The reference has NO finite-mu path (SURVEY.md §8c "Missing from the
container", §8f rank 3).  This module is the
host-side input producer of the self-derived finite-mu extension of the
reference's vacuum equation; DESIGN.md "Finite chemical potential" states the
equations.  It follows the vacuum construction of grid.py:96-154 axis by axis:

  external |p|  : logspace over [p_min, p_max]      (vacuum p2_ext, grid.py:116-117)
  internal |q|  : Gauss-Legendre in s = ln|q|        (vacuum q2_int, grid.py:118-119)
  external p4   : uniform midpoints in sigma, p4 = s0 sinh(sigma), sigma in [-S, S],
                  S = asinh(lam / s0)                (nodes dense where the Gaussian
                                                      interaction lives, spanning [-lam, lam])
  internal q4   : Gauss-Legendre in sigma (same map)
  angle         : Gauss-Legendre in z = cos(theta) on [-1, 1] (3-D angular measure 2 pi dz)

with the vacuum grid's coincidence rule (shift the external nodes half a step
when an external/internal pair coincides within 1e-12, grid.py:122-130) on
each axis.  The measure of d^4q/(2 pi)^4 = (1/(8 pi^3)) |q|^2 d|q| dq4 dz is
split into per-axis factors meas_s[j_s] = (1/(8 pi^3)) |q|^3 w_s and
meas_4[j_4] = s0 cosh(sigma) w_4; the kernel and the oracle both form the
node weight as the single product meas_s * meas_4 (np.outer).

Dressing functions A, B, C are complex arrays of shape (n_s, n_4); external
point i = i_s * n_4 + i_4, internal node j = j_s * m_4 + j_4.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import GridConstructionError, ParameterError
from .quadrature import gauss_legendre

__all__ = ["MuParams", "MuGrid", "build_mu_grid", "mu_bracket_indices", "THREE_VOLUME_COEFF"]

# d^4q/(2 pi)^4 = (1/(2 pi)^4) dq4 |q|^2 d|q| (2 pi) dz  ->  1/(8 pi^3)
THREE_VOLUME_COEFF = 1.0 / (8.0 * np.pi**3)
VERTICES = ("bc", "bc1", "bcb")  # order = DSE_MU_VERTEX_* codes
MODES = ("direct", "moments")    # order = DSE_MU_MODE_* codes
_COINCIDENCE_RTOL = 1e-12


@dataclass
class MuParams:
    """ModelParams (kernels.py:36-79) plus the finite-mu grid sizes.

    Defaults are BASELINE config 3: mu = 0.2 GeV, T = 0, 128 x 128 external
    (|p|, p4) nodes, 128 x 128 x 32 internal (|q|, q4, cos theta) nodes,
    xi = 1e-9, the reference's default interaction (D, omega) and m0.
    """

    D: float = 0.550
    omega: float = 0.678
    m0: float = 0.0
    z1: float = 1.0
    mu: float = 0.2
    xi: float = 1e-9
    n_s: int = 128
    n_4: int = 128
    m_s: int = 128
    m_4: int = 128
    m_ang: int = 32
    p_min: float = 1e-3
    p_max: float = 1e2
    lam: float = 1e2
    p4_scale: float = 0.2
    max_iterations: int = 500
    relaxation: float = 1.0
    # quark-gluon vertex: "bcb" (default) Ball-Chiu Sigma structures in every
    # channel + Delta_A/Delta_C in the B channel; "bc" the full in-medium
    # Ball-Chiu vertex (diverges under successive approximation on these grids,
    # DESIGN.md); "bc1" the Sigma structure only
    vertex: str = "bcb"
    # "direct": every integrand point every iteration; "moments": the angular
    # moments built once per grid (shared by every mu) and contracted per iteration
    mode: str = "direct"

    def validate(self) -> None:
        checks = [
            ("mode", self.mode in MODES),
            ("vertex", self.vertex in VERTICES),
            ("D", self.D >= 0.0),
            ("omega", self.omega > 0.0),
            ("m0", self.m0 >= 0.0),
            ("mu", np.isfinite(self.mu) and self.mu >= 0.0),
            ("xi", self.xi > 0.0),
            ("n_s", self.n_s >= 2),
            ("n_4", self.n_4 >= 2),
            ("m_s", self.m_s >= 2),
            ("m_4", self.m_4 >= 2),
            ("m_ang", self.m_ang >= 1),
            ("p_min/p_max", 0.0 < self.p_min < self.p_max),
            ("lam", self.lam > 0.0),
            ("p4_scale", self.p4_scale > 0.0),
            ("max_iterations", self.max_iterations >= 1),
            ("relaxation", 0.0 < self.relaxation <= 1.0),
        ]
        for key, ok in checks:
            if not ok:
                raise ParameterError(f"parameter out of range: {key}")

    @property
    def interaction_coeff(self) -> float:
        """8 pi^2 D / omega^4, evaluated as kernels.py:79 does."""
        return 8.0 * np.pi**2 * self.D / self.omega**4


@dataclass(frozen=True)
class MuGrid:
    p_ext: np.ndarray        # [n_s] external |p|
    ps2_ext: np.ndarray      # [n_s] |p|^2 (interpolation coordinate, linear as the vacuum p^2)
    p4_ext: np.ndarray       # [n_4]
    q_int: np.ndarray        # [m_s] internal |q|
    qs2_int: np.ndarray      # [m_s] |q|^2
    q4_int: np.ndarray       # [m_4]
    meas_s: np.ndarray       # [m_s] (1/(8 pi^3)) |q|^3 w_s
    meas_4: np.ndarray       # [m_4] s0 cosh(sigma) w_4
    z_nodes: np.ndarray      # [m_ang] Gauss-Legendre on [-1, 1]
    z_weights: np.ndarray    # [m_ang]
    brk_s: np.ndarray        # [m_s] int64 bracket of qs2_int in ps2_ext (-1 below, n_s-1 at/after)
    brk_4: np.ndarray        # [m_4] int64 bracket of q4_int in p4_ext
    node_measure: np.ndarray = field(repr=False)  # [m_s, m_4] np.outer(meas_s, meas_4)

    @property
    def n_s(self) -> int:
        return self.p_ext.size

    @property
    def n_4(self) -> int:
        return self.p4_ext.size

    @property
    def m_s(self) -> int:
        return self.q_int.size

    @property
    def m_4(self) -> int:
        return self.q4_int.size

    @property
    def m_ang(self) -> int:
        return self.z_nodes.size

    @property
    def n_ext(self) -> int:
        return self.n_s * self.n_4

    @property
    def m_int(self) -> int:
        return self.m_s * self.m_4

    @property
    def nominal_points(self) -> int:
        return self.n_ext * self.m_int * self.m_ang


def mu_bracket_indices(x_ext: np.ndarray, q_int: np.ndarray) -> np.ndarray:
    """searchsorted(side='right') - 1: the vacuum merge pass (grid.py:67-83) per axis."""
    return np.searchsorted(np.asarray(x_ext), np.asarray(q_int), side="right").astype(np.int64) - 1


def _min_gap(x_ext: np.ndarray, q_int: np.ndarray, scale: np.ndarray) -> float:
    pos = np.searchsorted(x_ext, q_int)
    last = x_ext.size - 1
    worst = np.inf
    for nb in (np.clip(pos - 1, 0, last), np.clip(pos, 0, last)):
        gap = np.abs(q_int - x_ext[nb]) / scale(q_int, x_ext[nb])
        worst = min(worst, float(np.min(gap)))
    return worst


def build_mu_grid(n_s: int, n_4: int, m_s: int, m_4: int, m_ang: int, p_min: float = 1e-3,
                  p_max: float = 1e2, lam: float = 1e2, p4_scale: float = 0.2, shared_p4: bool = False) -> MuGrid:
    if n_s < 2 or n_4 < 2 or m_s < 2 or m_4 < 2 or m_ang < 1:
        raise ParameterError(f"grid sizes out of range: n_s={n_s} n_4={n_4} m_s={m_s} m_4={m_4} m_ang={m_ang}")
    if not (0.0 < p_min < p_max) or not (lam > 0.0) or not (p4_scale > 0.0):
        raise ParameterError(f"grid ranges out of range: p=[{p_min}, {p_max}] lam={lam} p4_scale={p4_scale}")

    # spatial axis: the vacuum construction in |p| (logspace external, GL in ln internal)
    lg_lo, lg_hi = np.log10(p_min), np.log10(p_max)
    p_ext = np.logspace(lg_lo, lg_hi, n_s)
    radial = gauss_legendre(m_s, np.log(p_min), np.log(p_max))
    q_int = np.exp(radial.nodes)
    rel = lambda a, b: np.maximum(a, b)  # noqa: E731
    if _min_gap(p_ext, q_int, rel) <= _COINCIDENCE_RTOL:
        half = 0.5 * (lg_hi - lg_lo) / (n_s - 1)
        p_ext = p_ext * 10.0**-half
        if _min_gap(p_ext, q_int, rel) <= _COINCIDENCE_RTOL:
            raise GridConstructionError(f"could not separate |p| and |q| nodes for n_s={n_s}, m_s={m_s}")

    # temporal axis: sinh map, uniform midpoints external, GL internal
    big_s = float(np.arcsinh(lam / p4_scale))
    h = 2.0 * big_s / n_4
    sig_ext = -big_s + (np.arange(n_4) + 0.5) * h
    temporal = gauss_legendre(m_4, -big_s, big_s)
    q4_int = p4_scale * np.sinh(temporal.nodes)
    absolute = lambda a, b: np.full_like(a, lam)  # noqa: E731
    p4_ext = p4_scale * np.sinh(sig_ext)
    if shared_p4:
        if n_4 != m_4:
            raise ParameterError(f"shared p4 nodes need n_4 == m_4, got {n_4} and {m_4}")
        p4_ext = q4_int.copy()
    elif _min_gap(p4_ext, q4_int, absolute) <= _COINCIDENCE_RTOL:
        sig_ext = sig_ext - 0.25 * h
        p4_ext = p4_scale * np.sinh(sig_ext)
        if _min_gap(p4_ext, q4_int, absolute) <= _COINCIDENCE_RTOL:
            raise GridConstructionError(f"could not separate p4 and q4 nodes for n_4={n_4}, m_4={m_4}")

    angular = gauss_legendre(m_ang, -1.0, 1.0)
    meas_s = THREE_VOLUME_COEFF * q_int**3 * radial.weights
    meas_4 = p4_scale * np.cosh(temporal.nodes) * temporal.weights
    ps2 = p_ext * p_ext
    qs2 = q_int * q_int
    arrays = dict(p_ext=p_ext, ps2_ext=ps2, p4_ext=p4_ext, q_int=q_int, qs2_int=qs2, q4_int=q4_int,
                  meas_s=meas_s, meas_4=meas_4, z_nodes=np.array(angular.nodes), z_weights=np.array(angular.weights),
                  brk_s=mu_bracket_indices(ps2, qs2), brk_4=mu_bracket_indices(p4_ext, q4_int),
                  node_measure=np.outer(meas_s, meas_4))
    for arr in arrays.values():
        arr.flags.writeable = False
    return MuGrid(**arrays)


def grid_for(params: MuParams) -> MuGrid:
    return build_mu_grid(params.n_s, params.n_4, params.m_s, params.m_4, params.m_ang, params.p_min,
                         params.p_max, params.lam, params.p4_scale)
