"""Semi-Lagrangian building blocks on the GPU (reference semilag.py:1-179).

`departure_points` and `advect_scalar` keep the reference's names and
arguments over swe_departure_points / swe_interpolate (csrc/settls.cu):
great-circle departure points with the two-time-level extrapolated wind and
bicubic Lagrange interpolation with pole ghost rows.  Grids may be numpy or
torch, one [nlat, nlon] field or a [B, nlat, nlon] batch.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .spharm import SphereGrid, _ptr, _stream


class DeparturePointError(RuntimeError):
    """Trajectory iteration produced non-finite departure points (semilag.py:167-170)."""


def _grids(grid: SphereGrid, *xs):
    out, tt = [], False
    for x in xs:
        if isinstance(x, torch.Tensor):
            tt = True
            t = x.to(device=f"cuda:{grid.device}", dtype=torch.float64)
        else:
            t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(f"cuda:{grid.device}")
        single = t.ndim == 2
        t = t.reshape(-1, grid.nlat, grid.nlon).contiguous()
        out.append(t)
    return out, tt, single


def departure_points(grid: SphereGrid, u_arr, v_arr, u_ext, v_ext, dt: float,
                     iterations: int = 2):
    """Departure longitudes/latitudes of every grid point (semilag.py:140-170)."""
    (ua, va, ue, ve), tt, single = _grids(grid, u_arr, v_arr, u_ext, v_ext)
    lam = torch.empty_like(ua)
    th = torch.empty_like(ua)
    try:
        _lib.check(grid._lib.swe_departure_points(grid.plan, _ptr(ua), _ptr(va), _ptr(ue),
                                                  _ptr(ve), ua.shape[0], float(dt),
                                                  int(iterations), _ptr(lam), _ptr(th),
                                                  _stream()), "swe_departure_points")
    except _lib.NonFinite as exc:
        raise DeparturePointError(str(exc)) from None
    if single:
        lam, th = lam[0], th[0]
    return (lam, th) if tt else (lam.cpu().numpy(), th.cpu().numpy())


def advect_scalar(grid: SphereGrid, values, lam_d, th_d):
    """Interpolate grid scalars at the departure points (semilag.py:173-179)."""
    (v, lam, th), tt, single = _grids(grid, values, lam_d, th_d)
    out = torch.empty_like(v)
    _lib.check(grid._lib.swe_interpolate(grid.plan, _ptr(v), _ptr(lam), _ptr(th), v.shape[0],
                                         _ptr(out), _stream()), "swe_interpolate")
    if single:
        out = out[0]
    return out if tt else out.cpu().numpy()
