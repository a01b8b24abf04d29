"""Oracle SWE tendencies and the IMEX fine propagator, batched over slices.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
`/root/reference/pkg/src/pintswe/dynamics.py` and `steppers.py`:

* PrognosticState (Phi total, xi, delta, phibar) ... dynamics.py:38-104
* linear gravity / Coriolis ......................... dynamics.py:121-139
* nonlinear advection + rest ........................ dynamics.py:142-160
* backward-Euler (hyper)viscosity ................... dynamics.py:181-200
* per-mode Helmholtz solve .......................... steppers.py:61-71
* Coriolis fixed-point implicit solve ............... steppers.py:74-118
* Crank-Nicolson half / IMEX Strang step ............ steppers.py:121-168

A batch of B slices is advanced in lockstep; the implicit solve keeps the
reference's per-slice semantics by freezing each slice at the iteration
where *its* convergence test passes.
"""

from __future__ import annotations

import dataclasses
import math

import numpy as np

from .sht import OracleSphere, truncate_pad

SQRT2 = math.sqrt(2.0)


class ImplicitSolveError(RuntimeError):
    """Coriolis fixed point did not converge (steppers.py:27-28)."""


@dataclasses.dataclass
class OracleState:
    """Batched prognostic state: fields (B, K) complex, phibar (B,)."""

    sph: OracleSphere
    phi: np.ndarray
    xi: np.ndarray
    delta: np.ndarray
    phibar: np.ndarray

    @property
    def batch(self):
        return self.phi.shape[0]

    def copy(self):
        return OracleState(self.sph, self.phi.copy(), self.xi.copy(),
                           self.delta.copy(), self.phibar.copy())

    def fields(self):
        return (self.phi, self.xi, self.delta)

    def replace(self, phi, xi, delta):
        return OracleState(self.sph, phi, xi, delta, self.phibar)

    def phi_prime(self):
        c = self.phi.copy()                       # dynamics.py:52-56
        c[:, 0] -= self.phibar * SQRT2
        return c

    def axpy(self, tend, dt):                     # dynamics.py:58-63
        return self.replace(self.phi + dt * tend[0], self.xi + dt * tend[1],
                            self.delta + dt * tend[2])

    def __add__(self, o):                         # dynamics.py:91-95
        return self.replace(self.phi + o.phi, self.xi + o.xi, self.delta + o.delta)

    def __sub__(self, o):                         # dynamics.py:97-101
        return self.replace(self.phi - o.phi, self.xi - o.xi, self.delta - o.delta)

    def max_abs(self):
        """Per-slice max |coefficient| over the three fields (dynamics.py:65-67)."""
        return np.max([np.abs(f).max(axis=1) for f in self.fields()], axis=0)

    def is_finite(self):
        return np.all([np.isfinite(f).all(axis=1) for f in self.fields()], axis=0)

    def to_truncation(self, dst: OracleSphere):   # dynamics.py:73-83
        if dst is self.sph:
            return self.copy()
        return OracleState(dst, truncate_pad(self.phi, self.sph, dst),
                           truncate_pad(self.xi, self.sph, dst),
                           truncate_pad(self.delta, self.sph, dst),
                           self.phibar.copy())

    def slice(self, idx):
        idx = np.atleast_1d(idx)
        return OracleState(self.sph, self.phi[idx].copy(), self.xi[idx].copy(),
                           self.delta[idx].copy(), self.phibar[idx].copy())

    @staticmethod
    def stack(states):
        s0 = states[0]
        return OracleState(s0.sph, np.concatenate([s.phi for s in states]),
                           np.concatenate([s.xi for s in states]),
                           np.concatenate([s.delta for s in states]),
                           np.concatenate([s.phibar for s in states]))


@dataclasses.dataclass(frozen=True)
class StepCfg:
    """Mirror of StepperConfig for the IMEX scheme (steppers.py:31-50)."""

    dt: float = 60.0
    visc_order: int = 2
    visc_nu: float = 0.0
    coriolis_treatment: str = "implicit"
    include_nonlinear: bool = True
    tol: float = 1e-12
    max_iter: int = 200
    scheme: str = "imex"             # or "sl_si_settls" (oracle/semilag.py)
    settls_mode: str = "two_step"


# -- tendencies ----------------------------------------------------------------


def linear_gravity(s: OracleState):
    """(-phibar delta, 0, -lap Phi) (dynamics.py:121-126)."""
    return (-s.phibar[:, None] * s.delta, np.zeros_like(s.xi),
            -s.sph.laplacian(s.phi))


def linear_coriolis(s: OracleState):
    """(0, -div(fV), curl(fV)) pseudospectrally (dynamics.py:129-135)."""
    sph = s.sph
    u, v = sph.uv_from_vortdiv(s.xi, s.delta)
    f = sph.f_grid[:, None]
    curl, div = sph.vortdiv_from_uv(f * u, f * v)
    return (np.zeros_like(s.phi), -div, curl)


def _tsum(a, b):
    return tuple(x + y for x, y in zip(a, b))


def nonlinear_advection(s: OracleState):
    """(-V.grad Phi, -div(xi V), -lap(V.V/2) + curl(xi V)) (dynamics.py:142-151)."""
    sph = s.sph
    u, v = sph.uv_from_vortdiv(s.xi, s.delta)
    gx, gy = sph.grad_grid(s.phi)
    tphi = -sph.analysis(u * gx + v * gy)
    xg = sph.synthesis(s.xi)
    curl, div = sph.vortdiv_from_uv(xg * u, xg * v)
    ke = sph.analysis(0.5 * (u * u + v * v))
    return (tphi, -div, curl - sph.laplacian(ke))


def nonlinear_rest(s: OracleState):
    """(-Phi' delta, 0, 0) (dynamics.py:154-160)."""
    sph = s.sph
    prod = sph.synthesis(s.phi_prime()) * sph.synthesis(s.delta)
    z = np.zeros_like(s.xi)
    return (-sph.analysis(prod), z, z.copy())


def viscosity_factor(sph: OracleSphere, order, nu, dt):
    """b(n) = 1/(1 + dt nu (n(n+1)/a^2)^(q/2)) (dynamics.py:181-188)."""
    nn1 = sph.n_of * (sph.n_of + 1.0) / sph.radius ** 2
    return 1.0 / (1.0 + dt * nu * nn1 ** (order / 2.0))


def viscosity_step(s: OracleState, cfg: StepCfg):
    """dynamics.py:191-200."""
    if cfg.visc_nu == 0.0:
        return s.copy()
    b = viscosity_factor(s.sph, cfg.visc_order, cfg.visc_nu, cfg.dt)
    return s.replace(s.phi * b, s.xi * b, s.delta * b)


# -- implicit solve --------------------------------------------------------------


def helmholtz(sph, phibar, r, alpha):
    """Exact per-mode solve of (I - alpha L_G) U = r (steppers.py:61-71)."""
    eps = -sph.lap
    pb = phibar[:, None]
    denom = 1.0 + alpha * alpha * pb * eps
    phi = (r[0] - alpha * pb * r[2]) / denom
    delta = r[2] + alpha * eps * phi
    return phi, r[1].copy(), delta


def implicit_solve(rhs: OracleState, alpha, cfg: StepCfg, include_coriolis=True,
                   stats=None):
    """(I - alpha L) U = rhs with per-slice fixed point (steppers.py:74-118)."""
    sph = rhs.sph
    if alpha == 0.0:
        return rhs.copy()
    u = rhs.replace(*helmholtz(sph, rhs.phibar, rhs.fields(), alpha))
    if not include_coriolis or sph.omega == 0.0:
        return u
    active = np.ones(rhs.batch, dtype=bool)
    iters = np.zeros(rhs.batch, dtype=np.int64)
    for _ in range(cfg.max_iter):
        idx = np.flatnonzero(active)
        sub = u.slice(idx)
        lc = linear_coriolis(sub)
        r = [f[idx] + alpha * t for f, t in zip(rhs.fields(), lc)]
        new = helmholtz(sph, rhs.phibar[idx], r, alpha)
        overall = np.maximum(np.max([np.abs(f).max(axis=1) for f in new], axis=0), 1e-300)
        done = np.ones(idx.size, dtype=bool)
        for nf, of in zip(new, sub.fields()):
            scale = np.maximum(np.abs(nf).max(axis=1), 1e-13 * overall)
            # NaN differences count as converged, exactly like `>` in steppers.py:107
            done &= ~(np.abs(nf - of).max(axis=1) > cfg.tol * scale)
        u.phi[idx], u.xi[idx], u.delta[idx] = new
        iters[idx] += 1
        active[idx[done]] = False
        if not active.any():
            if stats is not None:
                stats.append(iters)
            return u
    bad = np.flatnonzero(active)
    sub = u.slice(bad)
    lin = _tsum(linear_gravity(sub), linear_coriolis(sub))
    rf = rhs.slice(bad).fields()
    res = max(np.abs(f - alpha * l - r).max() for f, l, r in zip(sub.fields(), lin, rf))
    raise ImplicitSolveError(f"Coriolis iteration did not converge; residual {res:.3e}")


def _implicit_tendency(s, cfg):                   # steppers.py:121-124
    if cfg.coriolis_treatment == "implicit":
        return _tsum(linear_gravity(s), linear_coriolis(s))
    return linear_gravity(s)


def explicit_tendency(s, cfg):                    # steppers.py:127-140
    parts = []
    if cfg.include_nonlinear:
        parts.append(nonlinear_advection(s))
        parts.append(nonlinear_rest(s))
    if cfg.coriolis_treatment == "explicit":
        parts.append(linear_coriolis(s))
    if not parts:
        z = np.zeros_like(s.phi)
        return (z, z.copy(), z.copy())
    out = parts[0]
    for p in parts[1:]:
        out = _tsum(out, p)
    return out


def cn_half(s, alpha, cfg, stats=None):           # steppers.py:143-152
    rhs = s.axpy(_implicit_tendency(s, cfg), alpha)
    return implicit_solve(rhs, alpha, cfg,
                          include_coriolis=cfg.coriolis_treatment == "implicit",
                          stats=stats)


def imex_step(s: OracleState, cfg: StepCfg, stats=None) -> OracleState:
    """CN(dt/4) -> Heun on N -> CN(dt/4) -> viscosity (steppers.py:155-168)."""
    dt = cfg.dt
    us = cn_half(s, dt / 4.0, cfg, stats)
    k1 = explicit_tendency(us, cfg)
    mid = us.axpy(k1, dt)
    k2 = explicit_tendency(mid, cfg)
    ue = us.axpy(_tsum(k1, k2), 0.5 * dt)
    un = cn_half(ue, dt / 4.0, cfg, stats)
    return viscosity_step(un, cfg)


def full_rhs(s: OracleState):                      # dynamics.py:163-165
    out = _tsum(linear_gravity(s), linear_coriolis(s))
    out = _tsum(out, nonlinear_advection(s))
    return _tsum(out, nonlinear_rest(s))


# -- scenario ---------------------------------------------------------------------

BUMP_AMPLITUDE = 6000.0                                  # scenarios.py:23
BUMP_WIDTHS = (20.0, 80.0, 360.0)                        # scenarios.py:24
BUMP_CENTERS = ((np.pi / 5.0, np.pi / 3.0),              # scenarios.py:25-27
                (6.0 * np.pi / 5.0, np.pi / 5.0),
                (8.0 * np.pi / 5.0, -np.pi / 4.0))
BUMP_MEAN_DEPTH = 29400.0                                # scenarios.py:28


def gaussian_bumps_grid(sph: OracleSphere):
    """Grid geopotential of the Gaussian-bumps scenario (scenarios.py:62-72)."""
    lam = sph.lons[None, :] * np.ones((sph.nlat, 1))
    th = sph.lats[:, None] * np.ones((1, sph.nlon))
    phibar = sph.gravity * BUMP_MEAN_DEPTH
    phi = np.full_like(lam, phibar)
    for (l0, t0), wdt in zip(BUMP_CENTERS, BUMP_WIDTHS):
        c = np.sin(th) * np.sin(t0) + np.cos(th) * np.cos(t0) * np.cos(lam - l0)
        d = np.arccos(np.clip(c, -1.0, 1.0))
        phi += BUMP_AMPLITUDE * np.exp(-wdt * d * d)
    return phi, phibar


def gaussian_bumps(sph: OracleSphere, batch=1) -> OracleState:
    phi_g, phibar = gaussian_bumps_grid(sph)
    phi = np.repeat(sph.analysis(phi_g)[None, :], batch, axis=0)
    z = np.zeros_like(phi)
    return OracleState(sph, phi, z, z.copy(), np.full(batch, phibar))
