"""Batched GPU fine propagator with the reference's stepper interface.

Mirror of `/root/reference/pkg/src/pintswe/steppers.py`: StepperConfig
(:31-50), StepperState (:53-58), ImplicitSolveError (:27-28), imex_step
(:155-168), advance (:215-222), propagate (:225-237).  One call advances every
slice of a batched PrognosticState through libswe_b200.so's swe_imex_step;
the implicit Coriolis fixed point keeps per-slice convergence (each slice
stops at its own iteration, exactly as a serial call would).

The SL-SI-SETTLS scheme (:171-212) is a coarse-level-only scheme and is out of
scope for the GPU path; configuring it raises
NotImplementedError at step time.
"""

from __future__ import annotations

import ctypes
import dataclasses
from typing import Optional

import numpy as np
import torch

from . import _lib
from .dynamics import PrognosticState, ViscositySpec
from .spharm import _ptr, _stream

IMEX = "imex"
SL_SI_SETTLS = "sl_si_settls"
TWO_STEP = "two_step"
ONE_STEP = "one_step"


class ImplicitSolveError(RuntimeError):
    """The Coriolis fixed-point iteration failed to reach tolerance."""


@dataclasses.dataclass(frozen=True)
class StepperConfig:
    scheme: str = IMEX
    dt: float = 60.0
    viscosity: ViscositySpec = ViscositySpec(2, 0.0)
    settls_mode: str = TWO_STEP
    coriolis_treatment: str = "implicit"    # "implicit" | "explicit"
    include_nonlinear: bool = True
    implicit_tol: float = 1e-12
    implicit_max_iter: int = 200

    def __post_init__(self):
        if self.dt <= 0:
            raise ValueError("dt must be positive")
        if self.scheme not in (IMEX, SL_SI_SETTLS):
            raise ValueError(f"unknown scheme {self.scheme!r}")
        if self.settls_mode not in (TWO_STEP, ONE_STEP):
            raise ValueError(f"unknown SETTLS mode {self.settls_mode!r}")
        if self.coriolis_treatment not in ("implicit", "explicit"):
            raise ValueError("coriolis_treatment must be implicit or explicit")

    def to_c(self) -> _lib.StepperCfgC:
        return _lib.StepperCfgC(self.dt, self.viscosity.order_q, self.viscosity.coeff_nu,
                                1 if self.coriolis_treatment == "implicit" else 0,
                                1 if self.include_nonlinear else 0, self.implicit_tol,
                                self.implicit_max_iter)


@dataclasses.dataclass
class StepperState:
    """Current state plus the one-step history used by two-step SETTLS."""

    current: PrognosticState
    previous: Optional[PrognosticState] = None


def imex_steps_inplace(state: PrognosticState, cfg: StepperConfig, nsteps: int = 1,
                       iters: Optional[np.ndarray] = None) -> PrognosticState:
    """Advance `state` by `nsteps` IMEX steps IN PLACE (device data mutated).

    iters, if given, is an int32 array [nsteps, B, 2] receiving the fixed-point
    iteration counts of the two Crank-Nicolson solves of every step.
    """
    if cfg.scheme != IMEX:
        raise NotImplementedError("the GPU propagator implements the IMEX scheme only")
    grid = state.grid
    c = cfg.to_c()
    resid = np.zeros(state.batch)
    ip = None
    if iters is not None:
        assert iters.shape == (nsteps, state.batch, 2) and iters.dtype == np.int32
        ip = iters.ctypes.data_as(ctypes.c_void_p)
    rc = grid._lib.swe_imex_step(grid.plan, _ptr(state.data), _ptr(state.phibar_t), state.batch,
                                 ctypes.byref(c), int(nsteps), ip,
                                 resid.ctypes.data_as(ctypes.c_void_p), _stream())
    try:
        _lib.check(rc, "swe_imex_step")
    except _lib.NoConvergence as exc:
        raise ImplicitSolveError(str(exc)) from None
    return state


def imex_step(state: PrognosticState, cfg: StepperConfig) -> PrognosticState:
    """Implicit half step, explicit Heun step on N, implicit half step, viscosity
    (steppers.py:155-168).  Returns a new state; the input is untouched."""
    return imex_steps_inplace(state.copy(), cfg, 1)


def advance(sstate: StepperState, cfg: StepperConfig) -> StepperState:
    """One step of the configured scheme (steppers.py:215-222)."""
    if cfg.scheme == IMEX:
        return StepperState(imex_step(sstate.current, cfg), None)
    raise NotImplementedError("SL-SI-SETTLS is a coarse-level scheme outside the GPU path")


def propagate(sstate: StepperState, t0: float, t1: float, cfg: StepperConfig) -> StepperState:
    """Advance over [t0, t1], an integral number of steps (steppers.py:225-237)."""
    span = t1 - t0
    if span < 0:
        raise ValueError("t1 must not precede t0")
    steps_f = span / cfg.dt
    nsteps = int(round(steps_f))
    if abs(steps_f - nsteps) > 1e-9:
        raise ValueError(f"slice [{t0}, {t1}] is not an integral number of dt")
    if cfg.scheme != IMEX:
        raise NotImplementedError("SL-SI-SETTLS is a coarse-level scheme outside the GPU path")
    if nsteps == 0:
        return StepperState(sstate.current.copy(), None)
    return StepperState(imex_steps_inplace(sstate.current.copy(), cfg, nsteps), None)
