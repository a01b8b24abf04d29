"""Gaussian-bumps initial condition (mirror of scenarios.py:62-72).

The three-bump geopotential is evaluated on the host grid (analytic input
generation, not the hot path) and transformed with the GPU analysis.
"""

from __future__ import annotations

import numpy as np
import torch

from .dynamics import PrognosticState
from .spharm import SphereGrid

GAUSSIAN_BUMP_AMPLITUDE = 6000.0
GAUSSIAN_BUMP_WIDTHS = (20.0, 80.0, 360.0)
GAUSSIAN_BUMP_CENTERS = ((np.pi / 5.0, np.pi / 3.0),
                         (6.0 * np.pi / 5.0, np.pi / 5.0),
                         (8.0 * np.pi / 5.0, -np.pi / 4.0))
GAUSSIAN_BUMP_MEAN_DEPTH = 29400.0


def great_circle_distance(lam, theta, lam0, theta0):
    c = (np.sin(theta) * np.sin(theta0)
         + np.cos(theta) * np.cos(theta0) * np.cos(lam - lam0))
    return np.arccos(np.clip(c, -1.0, 1.0))


def gaussian_bumps_grid(grid: SphereGrid):
    """Grid geopotential and phibar of the Gaussian-bumps scenario."""
    phibar = grid.geometry.gravity_g * GAUSSIAN_BUMP_MEAN_DEPTH
    lam = grid.lons[None, :] * np.ones((grid.nlat, 1))
    theta = grid.lats[:, None] * np.ones((1, grid.nlon))
    phi = np.full_like(lam, phibar)
    for (lam0, th0), width in zip(GAUSSIAN_BUMP_CENTERS, GAUSSIAN_BUMP_WIDTHS):
        d = great_circle_distance(lam, theta, lam0, th0)
        phi += GAUSSIAN_BUMP_AMPLITUDE * np.exp(-width * d * d)
    return phi, phibar


def gaussian_bumps(grid: SphereGrid, batch: int = 1) -> PrognosticState:
    """Resting geopotential with three Gaussian bumps, V = 0; `batch` copies."""
    phi_g, phibar = gaussian_bumps_grid(grid)
    phi = grid.analysis(torch.from_numpy(phi_g).cuda(grid.device))
    data = torch.zeros((batch, 3, grid.n_modes), dtype=torch.complex128, device=phi.device)
    data[:, 0] = phi
    return PrognosticState(grid, data, torch.full((batch,), phibar, dtype=torch.float64,
                                                  device=phi.device))
