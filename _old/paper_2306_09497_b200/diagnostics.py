"""Error norms, kinetic-energy spectra and their record types, on the device.

Mirror of the reference `pintswe.diagnostics` (diagnostics.py:1-118) over the
library's deterministic reductions (csrc/diag.cu): swe_window_maxdiff for the
windowed spectral error (diagnostics.py:46-65), swe_grid_sqdiff for the
physical-space RMS error (:68-75) and swe_ke_spectrum for the kinetic-energy
spectrum (:78-87).  States stay on the GPU; only the scalar results (and the
M-point spectrum) come back to the host.
"""

from __future__ import annotations

import ctypes
import dataclasses
import math

import numpy as np
import torch

from . import _lib
from .dynamics import PrognosticState
from .spharm import SphereGrid, _ptr, _stream, truncate_pad


@dataclasses.dataclass(frozen=True)
class ErrorRecord:
    iteration: int
    rnorm: str          # wavenumber cap as digits, or "l2"
    target: str         # "fine" | "reference"
    value: float

    def row(self):
        return (self.iteration, self.rnorm, self.target, self.value)


ERROR_HEADER = ("k", "rnorm", "target", "value")
SPECTRUM_HEADER = ("series", "iteration", "n", "wavelength_m", "energy")


@dataclasses.dataclass
class KESpectrumRecord:
    n: np.ndarray
    wavelength: np.ndarray
    energy: np.ndarray


def _dev(x, grid: SphereGrid, dtype):
    if isinstance(x, torch.Tensor):
        return x.to(device=f"cuda:{grid.device}", dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x)).to(f"cuda:{grid.device}", dtype)


def _window_terms(coeffs, grid: SphereGrid, ref, ref_grid: SphereGrid, rnorms):
    """max|c - c_ref| and max|c_ref| over m, n <= R for every R in rnorms."""
    for r in rnorms:
        if r < 1 or r > grid.M or r > ref_grid.M:
            raise ValueError(f"rnorm {r} outside 1..{min(grid.M, ref_grid.M)}")
    c = _dev(coeffs, grid, torch.complex128).reshape(grid.n_modes)
    rf = _dev(ref, ref_grid, torch.complex128).reshape(ref_grid.n_modes)
    if ref_grid is not grid:  # same (m, n) values on the window (n <= min M)
        rf = truncate_pad(rf, ref_grid, grid)
    out = torch.empty(2 * len(rnorms), dtype=torch.float64, device=c.device)
    rn = (ctypes.c_int * len(rnorms))(*[int(r) for r in rnorms])
    _lib.check(grid._lib.swe_window_maxdiff(grid.plan, _ptr(c), _ptr(rf), rn, len(rnorms),
                                            _ptr(out), _stream()), "swe_window_maxdiff")
    return out.cpu().numpy().reshape(-1, 2)


def spectral_error(coeffs, grid: SphereGrid, ref_coeffs, ref_grid: SphereGrid,
                   rnorm: int) -> float:
    """Relative max-coefficient error over the window m, n <= rnorm (diagnostics.py:51-65)."""
    num, den = _window_terms(coeffs, grid, ref_coeffs, ref_grid, [rnorm])[0]
    if den == 0.0:
        raise ZeroDivisionError("reference field vanishes on the error window")
    return float(num / den)


def l2_error(values, ref_values) -> float:
    """Relative RMS error on a uniform-weight physical grid (diagnostics.py:68-75)."""
    if tuple(values.shape) != tuple(ref_values.shape):
        raise ValueError("grids differ in shape")
    dev = values.device if isinstance(values, torch.Tensor) else torch.device("cuda")
    v = values if isinstance(values, torch.Tensor) else torch.from_numpy(np.asarray(values))
    r = ref_values if isinstance(ref_values, torch.Tensor) else torch.from_numpy(np.asarray(ref_values))
    v = v.to(dev, torch.float64).contiguous()
    r = r.to(dev, torch.float64).contiguous()
    out = torch.empty(2, dtype=torch.float64, device=dev)
    _lib.check(_lib.load().swe_grid_sqdiff(_ptr(v), _ptr(r), v.numel(), _ptr(out), _stream()),
               "swe_grid_sqdiff")
    num, den = out.cpu().numpy()
    n = v.numel()
    if den == 0.0:
        raise ZeroDivisionError("reference field vanishes")
    return float(math.sqrt(num / n) / math.sqrt(den / n))


def ke_spectrum_batch(state: PrognosticState) -> np.ndarray:
    """Energy per total wavenumber n = 1..M for every slice: [B, M]."""
    grid = state.grid
    e = torch.empty((state.batch, grid.M), dtype=torch.float64, device=state.data.device)
    _lib.check(grid._lib.swe_ke_spectrum(grid.plan, _ptr(state.data), state.batch, _ptr(e),
                                         _stream()), "swe_ke_spectrum")
    return e.cpu().numpy()


def ke_spectrum(state: PrognosticState, index: int = 0) -> KESpectrumRecord:
    """Kinetic-energy spectrum per total wavenumber (n >= 1) (diagnostics.py:78-87)."""
    grid = state.grid
    a = grid.geometry.radius_a
    n = np.arange(1, grid.M + 1)
    return KESpectrumRecord(n=n, wavelength=2.0 * np.pi * a / n,
                            energy=ke_spectrum_batch(state)[index])


def spectrum_rows(series: str, iteration, record: KESpectrumRecord):
    """Rows for spectrum.csv: (series, iteration, n, wavelength_m, energy)."""
    return [(series, iteration, int(nn), float(wl), float(en))
            for nn, wl, en in zip(record.n, record.wavelength, record.energy)]


def phi_error_records(iteration: int, state: PrognosticState, target_name: str,
                      target: PrognosticState, rnorms, include_l2: bool = False):
    """Geopotential error records of one iterate against one target, both projected
    onto the common truncation min(M, M_target) (diagnostics.py:99-118)."""
    common = state.grid if state.grid.M <= target.grid.M else target.grid
    s = state.to_truncation(common)
    t = target.to_truncation(common)
    terms = _window_terms(s.phi[0], common, t.phi[0], common, [int(r) for r in rnorms])
    records = []
    for r, (num, den) in zip(rnorms, terms):
        if den == 0.0:
            raise ZeroDivisionError("reference field vanishes on the error window")
        records.append(ErrorRecord(iteration, str(int(r)), target_name, float(num / den)))
    if include_l2:
        val = l2_error(common.synthesis(s.phi[0:1])[0], common.synthesis(t.phi[0:1])[0])
        records.append(ErrorRecord(iteration, "l2", target_name, val))
    return records
