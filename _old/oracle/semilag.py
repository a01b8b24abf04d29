"""CPU restatement of the reference's semi-Lagrangian pieces and the SL-SI-SETTLS
step (test infrastructure only: tests/ and the bench's CPU legs use it as the
checker; the product path never calls it).

Follows pintswe/semilag.py:25-179 and steppers.py:171-212:
  * bicubic Lagrange interpolation on the Gaussian grid: uniform cubic weights
    in longitude, 4-point Lagrange weights on the true latitudes, two ghost
    rows past each pole taken from the rows next to it shifted by half a
    revolution (semilag.py:25-88);
  * departure points by the two-time-level extrapolation: start from a
    great-circle displacement with the arrival wind, then `iterations` times
    interpolate the extrapolated wind (Cartesian components) at the departure
    guess, project it onto the tangent plane there, transport it back to the
    arrival point, average with the arrival wind and displace again
    (semilag.py:108-170);
  * the SETTLS step G = U + dt/2 (L U + 2 N_R(U) - N_R(U_prev)) taken at the
    departure points, plus dt/2 N_R(U), solved with (I - dt/2 L) and damped by
    the viscosity factor (steppers.py:171-212).
"""

from __future__ import annotations

import numpy as np

from .sht import OracleSphere
from .swe import (OracleState, StepCfg, _tsum, implicit_solve, linear_coriolis, linear_gravity,
                  nonlinear_rest, viscosity_step)


class DeparturePointError(RuntimeError):
    pass


class GridInterp:
    """Bicubic interpolation of grid fields [J, I] (north-to-south rows)."""

    def __init__(self, sph: OracleSphere):
        self.J, self.I = sph.nlat, sph.nlon
        self.dlon = 2.0 * np.pi / self.I
        up = sph.lats[::-1]                               # ascending latitudes
        self.nodes = np.concatenate([[-np.pi - up[1], -np.pi - up[0]], up,
                                     [np.pi - up[-1], np.pi - up[-2]]])

    def extended(self, g):
        """[J+4, I] ascending rows with the pole ghost rows (semilag.py:45-53)."""
        a = g[::-1]
        h = self.I // 2
        ghost = lambda row: np.roll(row, h)                # noqa: E731
        return np.vstack([ghost(a[1]), ghost(a[0]), a, ghost(a[-1]), ghost(a[-2])])

    def stencil(self, lam, th):
        """Latitude rows, longitude columns and their weights (semilag.py:55-80)."""
        lam = np.mod(lam, 2.0 * np.pi)
        x = lam / self.dlon
        i0 = np.floor(x).astype(np.int64)
        t = x - i0
        wl = np.stack([-t * (t - 1.0) * (t - 2.0) / 6.0,
                       (t + 1.0) * (t - 1.0) * (t - 2.0) / 2.0,
                       -(t + 1.0) * t * (t - 2.0) / 2.0,
                       (t + 1.0) * t * (t - 1.0) / 6.0], axis=-1)
        cols = (i0[..., None] + np.arange(-1, 3)) % self.I
        j = np.clip(np.searchsorted(self.nodes, th) - 1, 1, self.nodes.size - 3)
        rows = j[..., None] + np.arange(-1, 3)
        nd = self.nodes[rows]
        wt = np.ones_like(nd)
        for k in range(4):
            for l in range(4):
                if l != k:
                    wt[..., k] = wt[..., k] * (th - nd[..., l]) / 1.0
        den = np.ones_like(nd)
        for k in range(4):
            for l in range(4):
                if l != k:
                    den[..., k] = den[..., k] * (nd[..., k] - nd[..., l])
        return rows, cols, wt / den, wl

    def apply(self, g, st):
        rows, cols, wt, wl = st
        ext = self.extended(g)
        patch = ext[rows[..., :, None], cols[..., None, :]]
        return (patch * wt[..., :, None] * wl[..., None, :]).sum(axis=(-2, -1))


def _frame(sph: OracleSphere):
    lam = sph.lons[None, :] * np.ones((sph.nlat, 1))
    mu = sph.mu[:, None] * np.ones((1, sph.nlon))
    c = sph.cos_lat[:, None] * np.ones((1, sph.nlon))
    xa = np.stack([c * np.cos(lam), c * np.sin(lam), mu])
    el = np.stack([-np.sin(lam), np.cos(lam), np.zeros_like(lam)])
    et = np.stack([-mu * np.cos(lam), -mu * np.sin(lam), c])
    return xa, el, et


def _back(xa, w, dt, a):
    """Great-circle step of length |w| dt / a backward from xa along w."""
    sp = np.sqrt((w * w).sum(axis=0))
    sig = sp * dt / a
    with np.errstate(invalid="ignore", divide="ignore"):
        dirn = np.where(sp > 0.0, w / np.where(sp > 0.0, sp, 1.0), 0.0)
    xd = np.cos(sig) * xa - np.sin(sig) * dirn
    return xd / np.sqrt((xd * xd).sum(axis=0))


def _transport(v, src, dst):
    """Rotate the tangent vector v at src into the tangent plane at dst."""
    k = np.cross(src, dst, axis=0)
    s2 = (k * k).sum(axis=0)
    c = (src * dst).sum(axis=0)
    tiny = s2 < 1e-24
    out = c * v + np.cross(k, v, axis=0) + k * ((k * v).sum(axis=0) * (1.0 - c)
                                                / np.where(tiny, 1.0, s2))
    return np.where(tiny, v, out)


def _lonlat(xd):
    return (np.mod(np.arctan2(xd[1], xd[0]), 2.0 * np.pi),
            np.arcsin(np.clip(xd[2], -1.0, 1.0)))


def departure_points(sph: OracleSphere, ua, va, ue, ve, dt, iterations=2):
    """(lambda_d, theta_d) of every grid point of one slice (semilag.py:140-170)."""
    a = sph.radius
    xa, el, et = _frame(sph)
    wa = ua[None] * el + va[None] * et
    vc = ue[None] * el + ve[None] * et
    gi = GridInterp(sph)
    xd = _back(xa, wa, dt, a)
    for _ in range(iterations):
        st = gi.stencil(*_lonlat(xd))
        we = np.stack([gi.apply(vc[c], st) for c in range(3)])
        we = we - (we * xd).sum(axis=0) * xd
        xd = _back(xa, 0.5 * (_transport(we, xd, xa) + wa), dt, a)
    lam, th = _lonlat(xd)
    if not (np.isfinite(lam).all() and np.isfinite(th).all()):
        raise DeparturePointError("departure-point iteration diverged")
    return lam, th


def settls_step(u: OracleState, prev, cfg: StepCfg) -> OracleState:
    """One SL-SI-SETTLS step per slice (steppers.py:171-212); prev (same batch)
    or None = one-step mode (prev := u)."""
    sph, dt = u.sph, cfg.dt
    prev = u if prev is None else prev
    half = 0.5 * dt
    un, vn = sph.uv_from_vortdiv(u.xi, u.delta)
    up, vp = sph.uv_from_vortdiv(prev.xi, prev.delta)
    lin = _tsum(linear_gravity(u), linear_coriolis(u))
    nr, nrp = nonlinear_rest(u), nonlinear_rest(prev)
    g = [f + half * (lf + 2.0 * nf - pf)
         for f, lf, nf, pf in zip(u.fields(), lin, nr, nrp)]
    gi = GridInterp(sph)
    out = [np.empty_like(f) for f in g]
    for b in range(u.batch):
        lam, th = departure_points(sph, un[b], vn[b], 2.0 * un[b] - up[b],
                                   2.0 * vn[b] - vp[b], dt)
        st = gi.stencil(lam, th)
        for f in range(3):
            out[f][b] = sph.analysis(gi.apply(sph.synthesis(g[f][b]), st)) + half * nr[f][b]
    rhs = u.replace(*out)
    return viscosity_step(implicit_solve(rhs, half, cfg, include_coriolis=True), cfg)
