"""Oracle spherical-harmonic transform, batched over fields/slices.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
`/root/reference/pkg/src/pintswe/spharm.py`:

* Gaussian grid sizing .................. spharm.py:61-68
* Gauss-Legendre nodes (Newton) ......... spharm.py:75-108
* orthonormal P_mn recurrence ........... spharm.py:111-143
* H = (1-mu^2) dP/dmu tables ............ spharm.py:179-187
* analysis / synthesis / pair synthesis . spharm.py:238-267
* Laplacian, gradient, winds, vort/div .. spharm.py:271-343
* truncate_pad .......................... spharm.py:352-368

Spectral arrays are complex128 with shape (..., K) in the packed m-major
layout (block m holds n = m..M); grid arrays are float64 (..., nlat, nlon),
latitudes north to south.  Leading dimensions are a batch.
"""

from __future__ import annotations

import math

import numpy as np

EARTH_RADIUS = 6371.22e3      # spharm.py:21
EARTH_OMEGA = 7.292e-5        # spharm.py:22
EARTH_GRAVITY = 9.80616       # spharm.py:23


def grid_shape(M: int):
    """(nlat, nlon) of the 3/2-rule dealiased grid (spharm.py:61-68)."""
    nlat = -(-(3 * M + 1) // 2)
    nlon = 3 * M + 1
    nlon += nlon % 2
    return nlat, nlon


def gauss_nodes(n: int, tol: float = 1e-15, max_iter: int = 100):
    """Gauss-Legendre nodes (decreasing) and weights (spharm.py:75-108)."""
    x = np.cos(np.pi * (np.arange(n) + 0.75) / (n + 0.5))
    for _ in range(max_iter):
        lo, hi = np.ones_like(x), x.copy()          # P_0, P_1
        for k in range(2, n + 1):
            lo, hi = hi, ((2 * k - 1) * x * hi - (k - 1) * lo) / k
        deriv = n * (x * hi - lo) / (x * x - 1.0)
        step = hi / deriv
        x = x - step
        if np.all(np.abs(step) <= tol * np.maximum(1.0, np.abs(x))):
            break
    else:
        raise RuntimeError(f"Gauss-Legendre Newton failed for n={n}")
    w = 2.0 / ((1.0 - x * x) * deriv * deriv)
    order = np.argsort(-x)
    return x[order], w[order]


def _eps(m, n):
    """sqrt((n^2-m^2)/(4n^2-1)), zero for n <= m (spharm.py:111-115)."""
    m = np.asarray(m, dtype=np.float64)
    n = np.asarray(n, dtype=np.float64)
    num = np.where(n > m, n * n - m * m, 0.0)
    return np.sqrt(num / (4.0 * n * n - 1.0))


def legendre_tables(M: int, mu: np.ndarray):
    """P[m] of shape (nlat, M+2-m) for n = m..M+1 (spharm.py:118-143).

    Computed diagonal by diagonal (d = n - m) for all orders at once; the
    per-element arithmetic is the reference's three-term recurrence.
    """
    nlat = mu.shape[0]
    cos_t = np.sqrt(np.maximum(1.0 - mu * mu, 0.0))
    sect = np.empty((M + 1, nlat))
    sect[0] = 1.0 / math.sqrt(2.0)
    for m in range(1, M + 1):
        sect[m] = sect[m - 1] * cos_t * math.sqrt((2.0 * m + 1.0) / (2.0 * m))
    ms = np.arange(M + 1)
    diag = np.zeros((M + 2, M + 1, nlat))           # diag[d, m, j] = P_{m,m+d}
    diag[0] = sect
    diag[1] = np.sqrt(2.0 * ms + 3.0)[:, None] * mu[None, :] * sect
    for d in range(2, M + 2):
        e_n = _eps(ms, ms + d)[:, None]
        e_nm1 = _eps(ms, ms + d - 1)[:, None]
        with np.errstate(divide="ignore", invalid="ignore"):
            nxt = (mu[None, :] * diag[d - 1] - e_nm1 * diag[d - 2]) / e_n
        diag[d] = np.where(ms[:, None] + d <= M + 1, nxt, 0.0)
    return [np.ascontiguousarray(diag[: M + 2 - m, m, :].T) for m in range(M + 1)]


class OracleSphere:
    """Transform tables for one truncation M (spharm.py:146-202)."""

    def __init__(self, M: int, radius=EARTH_RADIUS, omega=EARTH_OMEGA,
                 gravity=EARTH_GRAVITY):
        self.M = M
        self.radius, self.omega, self.gravity = radius, omega, gravity
        self.nlat, self.nlon = grid_shape(M)
        self.mu, self.weights = gauss_nodes(self.nlat)
        self.lats = np.arcsin(self.mu)
        self.lons = 2.0 * np.pi * np.arange(self.nlon) / self.nlon
        self.cos_lat = np.sqrt(1.0 - self.mu ** 2)
        k_m = M + 1 - np.arange(M + 1)
        self.offsets = np.concatenate([[0], np.cumsum(k_m)]).astype(np.int64)
        self.n_modes = int(self.offsets[-1])
        self.m_of = np.repeat(np.arange(M + 1), k_m)
        self.n_of = np.arange(self.n_modes) - self.offsets[self.m_of] + self.m_of
        full = legendre_tables(M, self.mu)
        self.P, self.H = [], []
        for m, tab in enumerate(full):
            n = np.arange(m, M + 1, dtype=np.float64)
            h = (-n * _eps(m, n + 1))[None, :] * tab[:, 1:]
            lower = np.zeros_like(h)
            lower[:, 1:] = ((n[1:] + 1.0) * _eps(m, n[1:]))[None, :] * tab[:, :-2]
            h = h + lower
            self.P.append(np.ascontiguousarray(tab[:, :-1]))
            self.H.append(h)
        nn1 = self.n_of * (self.n_of + 1.0)
        self.lap = -nn1 / radius ** 2
        self.inv_lap = np.zeros(self.n_modes)
        self.inv_lap[nn1 > 0] = -(radius ** 2) / nn1[nn1 > 0]
        self.w_sin2 = self.weights / (1.0 - self.mu ** 2)
        self.f_grid = 2.0 * omega * self.mu

    # -- shape helpers ------------------------------------------------------

    def _blocks(self):
        for m in range(self.M + 1):
            yield m, slice(int(self.offsets[m]), int(self.offsets[m + 1]))

    @staticmethod
    def _flat(a, tail):
        lead = a.shape[: a.ndim - tail]
        return a.reshape((-1,) + a.shape[a.ndim - tail:]), lead

    def check_spec(self, c):
        if c.shape[-1] != self.n_modes:
            raise ValueError(f"expected {self.n_modes} packed coefficients")

    def check_grid(self, g):
        if g.shape[-2:] != (self.nlat, self.nlon):
            raise ValueError(f"grid shape {g.shape[-2:]} != ({self.nlat}, {self.nlon})")

    # -- Legendre stage (batched real GEMMs on (re, im) rows) ----------------

    def _legendre_to_half(self, terms):
        """half[b, j, m] = sum_t T_t[m] @ c_t[b, block m] (spharm.py:249-267)."""
        c0 = terms[0][1]
        nb = c0.shape[0]
        half = np.zeros((nb, self.nlat, self.nlon // 2 + 1), dtype=np.complex128)
        for m, sl in self._blocks():
            acc = None
            for tabs, c in terms:
                blk = c[:, sl]
                ri = np.concatenate([blk.real, blk.imag], axis=0)   # (2B, k)
                prod = ri @ tabs[m].T                                # (2B, J)
                acc = prod if acc is None else acc + prod
            half[:, :, m] = acc[:nb] + 1j * acc[nb:]
        return half

    def _half_to_grid(self, half):
        return np.fft.irfft(half * self.nlon, n=self.nlon, axis=-1)

    def _project(self, tabs, fm):
        """out[b, block m] = T[m]^T @ fm[b, :, m] (spharm.py:238-247)."""
        nb = fm.shape[0]
        out = np.empty((nb, self.n_modes), dtype=np.complex128)
        for m, sl in self._blocks():
            col = fm[:, :, m]
            ri = np.concatenate([col.real, col.imag], axis=0)       # (2B, J)
            r = ri @ tabs[m]                                         # (2B, k)
            out[:, sl] = r[:nb] + 1j * r[nb:]
        return out

    # -- public transforms ----------------------------------------------------

    def synthesis(self, c):
        """Packed spectral -> grid (spharm.py:249-257)."""
        self.check_spec(c)
        cf, lead = self._flat(np.asarray(c, dtype=np.complex128), 1)
        g = self._half_to_grid(self._legendre_to_half([(self.P, cf)]))
        return g.reshape(lead + g.shape[1:])

    def synthesis_pair(self, cp, ch):
        """sum_m (P cp + H ch) e^{im lambda} (spharm.py:259-267)."""
        cpf, lead = self._flat(np.asarray(cp, dtype=np.complex128), 1)
        chf, _ = self._flat(np.asarray(ch, dtype=np.complex128), 1)
        g = self._half_to_grid(self._legendre_to_half([(self.P, cpf), (self.H, chf)]))
        return g.reshape(lead + g.shape[1:])

    def analysis(self, g):
        """Grid -> packed spectral (spharm.py:238-247)."""
        self.check_grid(g)
        gf, lead = self._flat(np.asarray(g, dtype=np.float64), 2)
        fm = np.fft.rfft(gf, axis=-1) / self.nlon
        fm = fm * self.weights[None, :, None]
        out = self._project(self.P, fm)
        return out.reshape(lead + (self.n_modes,))

    def laplacian(self, c):
        return c * self.lap                                   # spharm.py:271-273

    def inverse_laplacian(self, c):
        return c * self.inv_lap                               # spharm.py:275-278

    def grad_grid(self, c):
        """(gx, gy) = (d_lambda / (a cos), d_theta / a) (spharm.py:282-294)."""
        a = self.radius
        gx = self.synthesis(c * (1j * self.m_of)) / (a * self.cos_lat[:, None])
        gy = self.synthesis_pair(np.zeros_like(c), c) / (a * self.cos_lat[:, None])
        return gx, gy

    def uv_from_vortdiv(self, xi, delta):
        """Winds from vorticity/divergence (spharm.py:296-313)."""
        a = self.radius
        psi = self.inverse_laplacian(xi)
        chi = self.inverse_laplacian(delta)
        im = 1j * self.m_of
        u = self.synthesis_pair(chi * im, -psi)
        v = self.synthesis_pair(psi * im, chi)
        s = 1.0 / (a * self.cos_lat[:, None])
        return u * s, v * s

    def vortdiv_from_uv(self, u, v):
        """(xi, delta) of a grid wind (spharm.py:315-343)."""
        self.check_grid(u)
        a = self.radius
        uf, lead = self._flat(np.asarray(u, dtype=np.float64), 2)
        vf, _ = self._flat(np.asarray(v, dtype=np.float64), 2)
        cos = self.cos_lat[:, None]
        amx = np.fft.rfft(uf * cos, axis=-1) / self.nlon
        bmx = np.fft.rfft(vf * cos, axis=-1) / self.nlon
        ws = self.w_sin2[None, :, None]
        amx, bmx = amx * ws, bmx * ws
        pa, pb = self._project(self.P, amx), self._project(self.P, bmx)
        ha, hb = self._project(self.H, amx), self._project(self.H, bmx)
        im = 1j * self.m_of
        delta = im * pa - hb
        xi = im * pb + ha
        return (xi / a).reshape(lead + (self.n_modes,)), \
            (delta / a).reshape(lead + (self.n_modes,))


def truncate_pad(c, src: OracleSphere, dst: OracleSphere):
    """Copy n <= min(M_src, M_dst) per m; zero elsewhere (spharm.py:352-368)."""
    c = np.asarray(c)
    out = np.zeros(c.shape[:-1] + (dst.n_modes,), dtype=np.complex128)
    mm = min(src.M, dst.M)
    for m in range(mm + 1):
        k = mm - m + 1
        out[..., dst.offsets[m]: dst.offsets[m] + k] = c[..., src.offsets[m]: src.offsets[m] + k]
    return out


def random_bandlimited(sph: OracleSphere, rng, batch=(), n_max=None):
    """Random valid coefficients, m = 0 real (test_spharm.py:16-22)."""
    shape = tuple(batch) + (sph.n_modes,)
    c = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    c[..., : sph.M + 1] = c[..., : sph.M + 1].real
    if n_max is not None:
        c[..., sph.n_of > n_max] = 0.0
    return c
