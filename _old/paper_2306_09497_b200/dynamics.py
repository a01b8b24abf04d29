"""Batched GPU prognostic state and SWE tendencies (mirror of dynamics.py).

Mirror of `/root/reference/pkg/src/pintswe/dynamics.py`: Tendency (:25-35),
PrognosticState (:38-104), ViscositySpec (:107-118), linear_gravity /
linear_coriolis / nonlinear terms / full_rhs (:121-165), viscosity helpers
(:168-200).  A state holds B independent slices in one CUDA tensor of shape
[B, 3, K] (complex128; fields Phi total, xi, delta) plus phibar [B]; B = 1 is
the reference's single state.  Arithmetic keeps the reference's rules
(`+`/`-` only on the same grid, phibar of the left operand).
"""

from __future__ import annotations

import ctypes
import dataclasses
import math
from typing import NamedTuple

import numpy as np
import torch

from . import _lib
from .spharm import SphereGrid, _ptr, _stream, truncate_pad

SQRT2 = math.sqrt(2.0)


class Tendency(NamedTuple):
    phi: torch.Tensor
    xi: torch.Tensor
    delta: torch.Tensor

    def __add__(self, other):
        return Tendency(self.phi + other.phi, self.xi + other.xi, self.delta + other.delta)

    def scaled(self, c: float) -> "Tendency":
        return Tendency(c * self.phi, c * self.xi, c * self.delta)


def _as_dev(x, grid: SphereGrid, dtype):
    if isinstance(x, torch.Tensor):
        return x.to(device=f"cuda:{grid.device}", dtype=dtype)
    return torch.as_tensor(np.asarray(x), dtype=dtype, device=f"cuda:{grid.device}")


class PrognosticState:
    """Spectral (Phi, xi, delta) of B slices; Phi stores the total geopotential."""

    def __init__(self, grid: SphereGrid, data: torch.Tensor, phibar):
        if data.ndim != 3 or data.shape[1] != 3 or data.shape[2] != grid.n_modes:
            raise ValueError(f"state data must be [B, 3, {grid.n_modes}]")
        self.grid = grid
        self.data = data.contiguous()
        pb = _as_dev(phibar, grid, torch.float64).reshape(-1)
        if pb.numel() == 1 and data.shape[0] > 1:
            pb = pb.expand(data.shape[0]).contiguous()
        self.phibar_t = pb.contiguous()

    @classmethod
    def from_fields(cls, grid, phi, xi, delta, phibar):
        """Build from per-field arrays, (K,) or (B, K), numpy or torch."""
        f = [_as_dev(x, grid, torch.complex128) for x in (phi, xi, delta)]
        if f[0].ndim == 1:
            f = [x[None] for x in f]
        return cls(grid, torch.stack(f, dim=1), phibar)

    # -- views -------------------------------------------------------------------
    @property
    def batch(self) -> int:
        return self.data.shape[0]

    @property
    def phi(self):
        return self.data[:, 0]

    @property
    def xi(self):
        return self.data[:, 1]

    @property
    def delta(self):
        return self.data[:, 2]

    @property
    def phibar(self) -> float:
        """Scalar mean geopotential (all slices of an engine share it)."""
        return float(self.phibar_t[0])

    def to_numpy(self):
        """(phi, xi, delta) as numpy arrays of shape (B, K), phibar (B,)."""
        d = self.data.cpu().numpy()
        return d[:, 0], d[:, 1], d[:, 2], self.phibar_t.cpu().numpy()

    # -- reference API (dynamics.py:47-104) ---------------------------------------
    def copy(self) -> "PrognosticState":
        return PrognosticState(self.grid, self.data.clone(), self.phibar_t.clone())

    def phi_prime(self):
        c = self.phi.clone()
        c[:, 0] -= self.phibar_t * SQRT2
        return c

    def add_tendency(self, tend: Tendency, dt: float) -> "PrognosticState":
        t = torch.stack([tend.phi, tend.xi, tend.delta], dim=1)
        return PrognosticState(self.grid, self.data + dt * t, self.phibar_t)

    def max_abs_each(self) -> torch.Tensor:
        out = torch.empty(self.batch, dtype=torch.float64, device=self.data.device)
        fin = torch.empty(self.batch, dtype=torch.int32, device=self.data.device)
        _lib.check(self.grid._lib.swe_state_stats(self.grid.plan, _ptr(self.data), self.batch,
                                                  _ptr(out), _ptr(fin), _stream()),
                   "swe_state_stats")
        self._fin = fin
        return out

    def is_finite_each(self) -> torch.Tensor:
        self.max_abs_each()
        return self._fin.bool()

    def max_abs(self) -> float:
        return float(self.max_abs_each().max())

    def is_finite(self) -> bool:
        return bool(self.is_finite_each().all())

    def to_truncation(self, grid_dst: SphereGrid) -> "PrognosticState":
        if grid_dst is self.grid:
            return self.copy()
        out = truncate_pad(self.data, self.grid, grid_dst)
        return PrognosticState(grid_dst, out, self.phibar_t.clone())

    def _require_compatible(self, other: "PrognosticState"):
        if other.grid is not self.grid:
            raise ValueError("states live on different grids")

    def __add__(self, other: "PrognosticState") -> "PrognosticState":
        self._require_compatible(other)
        return PrognosticState(self.grid, self.data + other.data, self.phibar_t)

    def __sub__(self, other: "PrognosticState") -> "PrognosticState":
        self._require_compatible(other)
        return PrognosticState(self.grid, self.data - other.data, self.phibar_t)

    def winds(self):
        return self.grid.uv_from_vortdiv(self.xi, self.delta)

    # -- batching helpers ---------------------------------------------------------
    def slice(self, idx) -> "PrognosticState":
        idx = torch.as_tensor(np.atleast_1d(idx), device=self.data.device)
        return PrognosticState(self.grid, self.data[idx], self.phibar_t[idx])

    @staticmethod
    def stack(states) -> "PrognosticState":
        g = states[0].grid
        for s in states:
            if s.grid is not g:
                raise ValueError("states live on different grids")
        return PrognosticState(g, torch.cat([s.data for s in states]),
                               torch.cat([s.phibar_t for s in states]))


@dataclasses.dataclass(frozen=True)
class ViscositySpec:
    """(Hyper)viscosity order q (even, >= 2) and coefficient nu (dynamics.py:107-118)."""

    order_q: int = 2
    coeff_nu: float = 0.0

    def __post_init__(self):
        if self.order_q < 2 or self.order_q % 2 != 0:
            raise ValueError("viscosity order must be an even integer >= 2")
        if self.coeff_nu < 0:
            raise ValueError("viscosity coefficient must be non-negative")


TEND_GRAVITY, TEND_CORIOLIS, TEND_NONLINEAR, TEND_FULL = 0, 1, 2, 3
TEND_ADVECTION, TEND_REST = 4, 5


def _tendency(state: PrognosticState, kind: int) -> Tendency:
    out = torch.empty_like(state.data)
    _lib.check(state.grid._lib.swe_tendency(state.grid.plan, kind, _ptr(state.data),
                                            _ptr(state.phibar_t), _ptr(out), state.batch,
                                            _stream()), "swe_tendency")
    return Tendency(out[:, 0], out[:, 1], out[:, 2])


def linear_gravity(state: PrognosticState) -> Tendency:
    """(-phibar delta, 0, -lap Phi) (dynamics.py:121-126)."""
    return _tendency(state, TEND_GRAVITY)


def linear_coriolis(state: PrognosticState) -> Tendency:
    """(0, -div(f V), curl(f V)) pseudospectrally (dynamics.py:129-135)."""
    return _tendency(state, TEND_CORIOLIS)


def linear_combined(state: PrognosticState) -> Tendency:
    return linear_gravity(state) + linear_coriolis(state)


def nonlinear(state: PrognosticState) -> Tendency:
    """nonlinear_advection + nonlinear_rest (dynamics.py:142-160), fused on the GPU:
    one grid pass computes -V.grad Phi - Phi' delta, V.V/2 and xi V."""
    return _tendency(state, TEND_NONLINEAR)


def nonlinear_advection(state: PrognosticState) -> Tendency:
    """(-V.grad Phi, -div(xi V), -lap(V.V/2) + curl(xi V)) (dynamics.py:142-151):
    the fused grid pass without the -Phi' delta product."""
    return _tendency(state, TEND_ADVECTION)


def nonlinear_rest(state: PrognosticState) -> Tendency:
    """(-Phi' delta, 0, 0) via a dealiased grid product (dynamics.py:154-160)."""
    return _tendency(state, TEND_REST)


def full_rhs(state: PrognosticState) -> Tendency:
    """L_G + L_C + N_A + N_R (dynamics.py:163-165)."""
    return _tendency(state, TEND_FULL)


def viscosity_coefficient_from_damping_time(M: int, order_q: int, tau: float,
                                            radius_a: float) -> float:
    """nu = (1/tau) (M(M+1)/a^2)^(-q/2) (dynamics.py:168-178)."""
    if tau <= 0:
        raise ValueError("damping time must be positive")
    if order_q < 2 or order_q % 2 != 0:
        raise ValueError("viscosity order must be an even integer >= 2")
    return (1.0 / tau) * (M * (M + 1) / radius_a ** 2) ** (-order_q / 2.0)


def viscosity_damping(grid: SphereGrid, vspec: ViscositySpec, dt: float) -> np.ndarray:
    """b(n) = 1/(1 + dt nu (n(n+1)/a^2)^(q/2)) per packed mode (dynamics.py:181-188)."""
    nn1 = grid.n_of * (grid.n_of + 1.0) / grid.geometry.radius_a ** 2
    return 1.0 / (1.0 + dt * vspec.coeff_nu * nn1 ** (vspec.order_q / 2.0))


def viscosity_step(state: PrognosticState, vspec: ViscositySpec, dt: float) -> PrognosticState:
    """Backward-Euler damping of Phi', xi, delta (dynamics.py:191-200); b(0) = 1
    keeps the mean geopotential.  (The IMEX step applies it fused in k_cn_fused /
    k_cn_finish; this is the standalone API call.)"""
    if dt <= 0:
        raise ValueError("dt must be positive")
    if vspec.coeff_nu == 0.0:
        return state.copy()
    b = torch.from_numpy(viscosity_damping(state.grid, vspec, dt)).to(state.data.device)
    return PrognosticState(state.grid, state.data * b, state.phibar_t.clone())
