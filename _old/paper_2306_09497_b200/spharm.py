"""GPU spherical-harmonic transform with the reference's SphereGrid interface.

Mirror of `/root/reference/pkg/src/pintswe/spharm.py` (SphereGeometry :30-42,
Truncation :45-72, SphereGrid :146-343, get_grid :346-349, truncate_pad
:352-368).  Same names, argument meaning and errors; the transforms run in
libswe_b200.so (parity-folded FP64 DMMA Legendre GEMMs + in-place mixed-radix
longitude FFT).  Every transform also accepts a leading batch dimension and
torch CUDA tensors (which stay on the device); numpy inputs return numpy.
"""

from __future__ import annotations

import ctypes
import dataclasses
import functools
import math

import numpy as np
import torch

from . import _lib

EARTH_RADIUS = 6371.22e3      # m
EARTH_OMEGA = 7.292e-5        # s^-1
EARTH_GRAVITY = 9.80616       # m s^-2


@dataclasses.dataclass(frozen=True)
class SphereGeometry:
    """Sphere radius, rotation rate and gravity (spharm.py:30-42)."""

    radius_a: float = EARTH_RADIUS
    omega: float = EARTH_OMEGA
    gravity_g: float = EARTH_GRAVITY

    def __post_init__(self):
        if not (self.radius_a > 0 and self.gravity_g > 0):
            raise ValueError("radius and gravity must be strictly positive")
        if self.omega < 0:
            raise ValueError("omega must be non-negative")


@dataclasses.dataclass(frozen=True)
class Truncation:
    """Triangular truncation M with its 3/2-rule Gaussian grid (spharm.py:45-72)."""

    M: int
    nlat: int
    nlon: int

    def __post_init__(self):
        if self.M < 1:
            raise ValueError("truncation M must be >= 1")
        if self.nlat < math.ceil((3 * self.M + 1) / 2):
            raise ValueError("nlat violates the 3/2 rule")
        if self.nlon < 3 * self.M + 1 or self.nlon % 2 != 0:
            raise ValueError("nlon must be even and satisfy the 3/2 rule")

    @classmethod
    def for_wavenumber(cls, M: int) -> "Truncation":
        nlat = -(-(3 * M + 1) // 2)
        nlon = 3 * M + 1 + (3 * M + 1) % 2
        return cls(M=M, nlat=nlat, nlon=nlon)

    @property
    def n_modes(self) -> int:
        return (self.M + 1) * (self.M + 2) // 2


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())


class SphereGrid:
    """Gaussian grid + device transform plan for one truncation and geometry.

    Public transforms are pure functions of their inputs (spharm.py:146-152).
    """

    def __init__(self, trunc: Truncation, geometry: SphereGeometry = SphereGeometry(),
                 device: int | None = None):
        if trunc != Truncation.for_wavenumber(trunc.M):
            raise ValueError("only the for_wavenumber grid of a truncation is supported")
        lib = _lib.load()
        if not torch.cuda.is_available():
            raise RuntimeError("SphereGrid needs a CUDA device (no CPU fallback)")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.trunc = trunc
        self.geometry = geometry
        self.M, self.nlat, self.nlon = trunc.M, trunc.nlat, trunc.nlon
        plan = ctypes.c_void_p()
        _lib.check(lib.swe_plan_create(self.M, geometry.radius_a, geometry.omega,
                                       geometry.gravity_g, self.device, ctypes.byref(plan)),
                   "swe_plan_create")
        self._plan = plan
        self._lib = lib
        mu = np.empty(self.nlat)
        w = np.empty(self.nlat)
        _lib.check(lib.swe_plan_grid(plan, mu.ctypes.data_as(ctypes.c_void_p),
                                     w.ctypes.data_as(ctypes.c_void_p)))
        self.mu, self.weights = mu, w
        self.lats = np.arcsin(mu)
        self.lons = 2.0 * np.pi * np.arange(self.nlon) / self.nlon
        self.cos_lat = np.sqrt(1.0 - mu ** 2)
        M = self.M
        self.offsets = np.zeros(M + 2, dtype=np.int64)
        for m in range(M + 1):
            self.offsets[m + 1] = self.offsets[m] + (M + 1 - m)
        self.n_modes = int(self.offsets[M + 1])
        self.m_of = np.repeat(np.arange(M + 1), M + 1 - np.arange(M + 1))
        self.n_of = np.arange(self.n_modes) - self.offsets[self.m_of] + self.m_of
        a = geometry.radius_a
        nn1 = self.n_of * (self.n_of + 1.0)
        self.laplacian_eig = -nn1 / (a * a)
        self.inv_laplacian_eig = np.zeros(self.n_modes)
        self.inv_laplacian_eig[nn1 > 0] = -(a * a) / nn1[nn1 > 0]
        self._dev_cache = {}

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan is not None and plan.value:
            try:
                self._lib.swe_plan_destroy(plan)
            except Exception:
                pass
            self._plan = None

    @property
    def plan(self):
        return self._plan

    # -- layout helpers (spharm.py:206-218) -----------------------------------

    def mode_index(self, m: int, n: int) -> int:
        if not (0 <= m <= self.M and m <= n <= self.M):
            raise IndexError(f"mode ({m},{n}) outside truncation M={self.M}")
        return int(self.offsets[m]) + (n - m)

    def zeros_spectral(self) -> np.ndarray:
        return np.zeros(self.n_modes, dtype=np.complex128)

    def zeros_grid(self) -> np.ndarray:
        return np.zeros((self.nlat, self.nlon))

    def _check_grid(self, values):
        if tuple(values.shape[-2:]) != (self.nlat, self.nlon) or values.ndim > 3:
            raise ValueError(f"grid shape {tuple(values.shape)} != ({self.nlat}, {self.nlon})")

    def _check_spec(self, coeffs):
        if coeffs.shape[-1] != self.n_modes or coeffs.ndim > 2:
            raise ValueError(f"expected {self.n_modes} packed coefficients")

    # -- device staging ----------------------------------------------------------

    def _to_dev(self, x, dtype):
        if isinstance(x, torch.Tensor):
            return x.to(device=f"cuda:{self.device}", dtype=dtype).contiguous(), True
        arr = np.ascontiguousarray(x, dtype=np.complex128 if dtype == torch.complex128 else np.float64)
        return torch.from_numpy(arr).to(f"cuda:{self.device}"), False

    @staticmethod
    def _out(t: torch.Tensor, as_torch: bool, single: bool):
        if single:
            t = t[0]
        return t if as_torch else t.cpu().numpy()

    # -- scalar transforms -------------------------------------------------------

    def synthesis(self, coeffs):
        """Packed coefficients -> grid values (spharm.py:249-257)."""
        self._check_spec(coeffs)
        c, tt = self._to_dev(coeffs, torch.complex128)
        single = c.ndim == 1
        c = c.reshape(-1, self.n_modes)
        g = torch.empty((c.shape[0], self.nlat, self.nlon), dtype=torch.float64, device=c.device)
        _lib.check(self._lib.swe_synthesis(self._plan, _ptr(c), _ptr(g), c.shape[0], _stream()),
                   "swe_synthesis")
        return self._out(g, tt, single)

    def analysis(self, values):
        """Grid values -> packed coefficients (spharm.py:238-247)."""
        self._check_grid(values)
        g, tt = self._to_dev(values, torch.float64)
        single = g.ndim == 2
        g = g.reshape(-1, self.nlat, self.nlon)
        c = torch.empty((g.shape[0], self.n_modes), dtype=torch.complex128, device=g.device)
        _lib.check(self._lib.swe_analysis(self._plan, _ptr(g), _ptr(c), g.shape[0], _stream()),
                   "swe_analysis")
        return self._out(c, tt, single)

    def _synthesis_pair(self, cp, ch):
        """sum_m (P cp_m + H ch_m) e^{i m lambda} on the grid (spharm.py:259-267)."""
        self._check_spec(cp)
        self._check_spec(ch)
        p, tt = self._to_dev(cp, torch.complex128)
        h, _ = self._to_dev(ch, torch.complex128)
        single = p.ndim == 1
        p, h = p.reshape(-1, self.n_modes), h.reshape(-1, self.n_modes)
        if p.shape != h.shape:
            raise ValueError("cp and ch must have the same shape")
        g = torch.empty((p.shape[0], self.nlat, self.nlon), dtype=torch.float64, device=p.device)
        _lib.check(self._lib.swe_synthesis_pair(self._plan, _ptr(p), _ptr(h), _ptr(g), p.shape[0],
                                                _stream()), "swe_synthesis_pair")
        return self._out(g, tt, single)

    def grad_grid(self, coeffs):
        """(gx, gy) = (1/(a cos) d/dlambda, 1/a d/dtheta) on the grid (spharm.py:282-294)."""
        self._check_spec(coeffs)
        c, tt = self._to_dev(coeffs, torch.complex128)
        single = c.ndim == 1
        c = c.reshape(-1, self.n_modes)
        gx = torch.empty((c.shape[0], self.nlat, self.nlon), dtype=torch.float64, device=c.device)
        gy = torch.empty_like(gx)
        _lib.check(self._lib.swe_grad_grid(self._plan, _ptr(c), _ptr(gx), _ptr(gy), c.shape[0],
                                           _stream()), "swe_grad_grid")
        return self._out(gx, tt, single), self._out(gy, tt, single)

    def laplacian(self, coeffs):
        self._check_spec(coeffs)
        return coeffs * self._eig("lap", self.laplacian_eig, coeffs)

    def inverse_laplacian(self, coeffs):
        """Inverse Laplacian; the (0,0) mode maps to zero (spharm.py:275-278)."""
        self._check_spec(coeffs)
        return coeffs * self._eig("inv", self.inv_laplacian_eig, coeffs)

    def _eig(self, key, arr, like):
        if isinstance(like, torch.Tensor):
            k = (key, like.device)
            if k not in self._dev_cache:
                self._dev_cache[k] = torch.from_numpy(arr).to(like.device)
            return self._dev_cache[k]
        return arr

    def uv_from_vortdiv(self, xi, delta):
        """Winds from vorticity/divergence (spharm.py:296-313)."""
        self._check_spec(xi)
        self._check_spec(delta)
        x, tt = self._to_dev(xi, torch.complex128)
        d, _ = self._to_dev(delta, torch.complex128)
        single = x.ndim == 1
        x, d = x.reshape(-1, self.n_modes), d.reshape(-1, self.n_modes)
        u = torch.empty((x.shape[0], self.nlat, self.nlon), dtype=torch.float64, device=x.device)
        v = torch.empty_like(u)
        _lib.check(self._lib.swe_uv_from_vortdiv(self._plan, _ptr(x), _ptr(d), _ptr(u), _ptr(v),
                                                 x.shape[0], _stream()), "swe_uv_from_vortdiv")
        return self._out(u, tt, single), self._out(v, tt, single)

    def vortdiv_from_uv(self, u, v):
        """(xi, delta) of a grid wind (spharm.py:315-343)."""
        self._check_grid(u)
        self._check_grid(v)
        gu, tt = self._to_dev(u, torch.float64)
        gv, _ = self._to_dev(v, torch.float64)
        single = gu.ndim == 2
        gu = gu.reshape(-1, self.nlat, self.nlon)
        gv = gv.reshape(-1, self.nlat, self.nlon)
        xi = torch.empty((gu.shape[0], self.n_modes), dtype=torch.complex128, device=gu.device)
        de = torch.empty_like(xi)
        _lib.check(self._lib.swe_vortdiv_from_uv(self._plan, _ptr(gu), _ptr(gv), _ptr(xi),
                                                 _ptr(de), gu.shape[0], _stream()),
                   "swe_vortdiv_from_uv")
        return self._out(xi, tt, single), self._out(de, tt, single)

    def device_bytes(self) -> int:
        return int(self._lib.swe_plan_bytes(self._plan))


@dataclasses.dataclass
class SpectralField:
    """Packed complex coefficients of one real scalar field (spharm.py:374-386)."""

    grid: SphereGrid
    coeffs: object

    def __post_init__(self):
        self.grid._check_spec(self.coeffs)

    def to_grid(self) -> "GridField":
        return GridField(self.grid, self.grid.synthesis(self.coeffs))


@dataclasses.dataclass
class GridField:
    """Real values on the Gaussian grid, latitudes north first (spharm.py:389-399)."""

    grid: SphereGrid
    values: object

    def __post_init__(self):
        self.grid._check_grid(self.values)

    def to_spectral(self) -> SpectralField:
        return SpectralField(self.grid, self.grid.analysis(self.values))


@functools.lru_cache(maxsize=64)
def get_grid(M: int, geometry: SphereGeometry = SphereGeometry()) -> SphereGrid:
    """Shared, cached transform engine for (M, geometry) (spharm.py:346-349)."""
    return SphereGrid(Truncation.for_wavenumber(M), geometry)


def truncate_pad(coeffs, grid_src: SphereGrid, grid_dst: SphereGrid):
    """Map packed coefficients between truncations (spharm.py:352-368).

    `coeffs` may carry leading dimensions; all are treated as independent
    packed arrays.
    """
    if grid_src.geometry != grid_dst.geometry:
        raise ValueError("truncate_pad requires matching geometries")
    grid_src._check_spec(coeffs) if getattr(coeffs, "ndim", 1) <= 2 else None
    c, tt = grid_src._to_dev(coeffs, torch.complex128)
    lead = tuple(c.shape[:-1])
    flat = c.reshape(-1, grid_src.n_modes)
    out = torch.empty((flat.shape[0], grid_dst.n_modes), dtype=torch.complex128, device=c.device)
    _lib.check(grid_src._lib.swe_truncate_pad(grid_src.plan, grid_dst.plan, _ptr(flat), _ptr(out),
                                              flat.shape[0], _stream()), "swe_truncate_pad")
    out = out.reshape(lead + (grid_dst.n_modes,))
    return out if tt else out.cpu().numpy()
