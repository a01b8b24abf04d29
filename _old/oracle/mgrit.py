"""Oracle FAS-MGRIT / Parareal driver and error diagnostics.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
`/root/reference/pkg/src/pintswe/pint.py` (IMEX and SL-SI-SETTLS levels with
the two-step history policy, pint.py:103-119) and the parts of
`diagnostics.py` that the frozen fixtures exercise:

* level sizes / validation ........ pint.py:55-95
* SweProblem protocol ............. pint.py:157-194
* F- / C-relaxation sweeps ........ pint.py:223-263
* residual, FAS restriction ....... pint.py:267-304
* coarsest serial sweep ........... pint.py:306-320
* recursive cycle ................. pint.py:322-337
* initial guess, run, blow-up ..... pint.py:341-400
* serial fine C-points ............ pint.py:421-430
* spectral / l2 errors, KE spectrum diagnostics.py:46-118

Slices are processed one state at a time (batch 1) so the control flow reads
like the reference; the batched GPU engine is checked against this.
"""

from __future__ import annotations

import dataclasses

import numpy as np

from .sht import OracleSphere
from .swe import OracleState, StepCfg, imex_step

SETTLS, ONE_STEP, TWO_STEP = "sl_si_settls", "one_step", "two_step"


def settls_boundary_policy(nlevels, level, nsteps, cfactor, chunk_size):   # pint.py:103-119
    """Per-step SETTLS mode: one-step below the coarsest level; on the coarsest,
    two-step except where the history would cross a chunk boundary."""
    if level < nlevels - 1:
        return [ONE_STEP] * nsteps
    spacing = cfactor ** (nlevels - 2)
    return [ONE_STEP if chunk_size > 0 and ((j - 1) * spacing) % chunk_size == 0 else TWO_STEP
            for j in range(1, nsteps + 1)]


class PintBlowUp(RuntimeError):
    def __init__(self, iteration, slice_index, trace):
        super().__init__(f"blow-up at iteration {iteration}, slice {slice_index}")
        self.iteration, self.slice_index, self.trace = iteration, slice_index, trace


@dataclasses.dataclass(frozen=True)
class Level:
    M: int
    cfg: StepCfg


@dataclasses.dataclass(frozen=True)
class PintCfg:
    levels: tuple
    T: float
    N0: int
    cfactor: int = 2
    nrelax: int = 0
    max_iters: int = 10
    cycle: str = "F_then_V"
    chunk_size: int = 0

    def points_on(self, level):                       # pint.py:89-90
        return self.N0 // self.cfactor ** level


class OracleProblem:
    """Per-level sphere + stepper (pint.py:157-194), one state per call."""

    def __init__(self, pcfg: PintCfg, spheres=None):
        cache = {} if spheres is None else dict(spheres)
        self.spheres = []
        for lv in pcfg.levels:
            if lv.M not in cache:
                cache[lv.M] = OracleSphere(lv.M)
            self.spheres.append(cache[lv.M])
        self.cfgs = [lv.cfg for lv in pcfg.levels]
        self.step_calls = 0

    def step(self, level, value, prev=None):
        """steppers.advance (steppers.py:215-222): SETTLS uses prev unless one-step."""
        self.step_calls += 1
        cfg = self.cfgs[level]
        if cfg.scheme == SETTLS:
            from .semilag import settls_step
            return settls_step(value, None if cfg.settls_mode == ONE_STEP else prev, cfg)
        return imex_step(value, cfg)

    def tracks_history(self, level):                  # pint.py:192-194
        cfg = self.cfgs[level]
        return cfg.scheme == SETTLS and cfg.settls_mode == TWO_STEP

    def restrict(self, level, value):
        return value.to_truncation(self.spheres[level + 1])

    def prolong(self, level, value):
        return value.to_truncation(self.spheres[level - 1])


@dataclasses.dataclass
class Trace:
    snapshots: list
    blowup: dict = None


class OracleMgrit:
    """Same control flow as MgritEngine (pint.py:197-400)."""

    def __init__(self, problem: OracleProblem, pcfg: PintCfg):
        self.p, self.c, self.m, self.L = problem, pcfg, pcfg.cfactor, len(pcfg.levels)

    def tracks(self, level):
        f = getattr(self.p, "tracks_history", None)
        return bool(f(level)) if f is not None else False

    def step(self, level, value, prev=None):
        return self.p.step(level, value) if prev is None else self.p.step(level, value, prev)

    def f_sweep(self, level, u, g):                   # pint.py:223-241
        m = self.m
        for i in range(1, len(u) // m + 1):
            v = u[m * (i - 1)]
            for j in range(m * (i - 1) + 1, m * i):
                v = self.p.step(level, v)
                if g is not None:
                    v = v + g[j]
                u[j] = v

    def c_sweep(self, level, u, g):                   # pint.py:243-256
        m = self.m
        new = {}
        for i in range(1, len(u) // m + 1):
            v = self.p.step(level, u[m * i - 1])
            new[m * i] = v if g is None else v + g[m * i]
        for k, v in new.items():
            u[k] = v

    def relax(self, level, u, g):                     # pint.py:258-263
        self.f_sweep(level, u, g)
        for _ in range(self.c.nrelax):
            self.c_sweep(level, u, g)
            self.f_sweep(level, u, g)

    def fas_restrict(self, level, u, g):              # pint.py:267-304
        m = self.m
        n = len(u) // m
        ubar = [self.p.restrict(level, u[m * i]) for i in range(n + 1)]
        res = [None]
        for i in range(1, n + 1):
            prop = self.p.step(level, u[m * i - 1])
            if g is not None:
                prop = prop + g[m * i]
            res.append(prop - u[m * i])
        modes = None                                  # pint.py:287-299
        if self.tracks(level + 1):
            modes = settls_boundary_policy(self.L, level + 1, n, m, self.c.chunk_size)
        gbar = [None]
        for i in range(1, n + 1):
            prev = ubar[i - 2] if modes and i >= 2 and modes[i - 1] == TWO_STEP else None
            tau = ubar[i] - self.step(level + 1, ubar[i - 1], prev)
            gbar.append(self.p.restrict(level, res[i]) + tau)
        return ubar, gbar

    def coarsest(self, u, g):                         # pint.py:306-320
        lv = self.L - 1
        modes = settls_boundary_policy(self.L, lv, len(u) - 1, self.m, self.c.chunk_size)
        track = self.tracks(lv)
        prev = None
        for j in range(1, len(u)):
            hist = prev if track and modes[j - 1] == TWO_STEP else None
            v = self.step(lv, u[j - 1], hist)
            prev = u[j - 1]
            u[j] = v if g is None else v + g[j]

    def cycle(self, level, u, g, kind):               # pint.py:322-337
        if level == self.L - 1:
            self.coarsest(u, g)
            return
        m = self.m
        self.relax(level, u, g)
        ubar, gbar = self.fas_restrict(level, u, g)
        v = [x.copy() for x in ubar]
        self.cycle(level + 1, v, gbar, kind)
        for i in range(1, len(u) // m + 1):
            u[m * i] = u[m * i] + self.p.prolong(level + 1, v[i] - ubar[i])
        self.f_sweep(level, u, g)
        if kind == "F_then_V" and level + 1 < self.L - 1:
            self.cycle(level, u, g, "V")

    def initial_guess(self, u0):                      # pint.py:341-353
        n1 = self.c.points_on(1)
        v = [self.p.restrict(0, u0)]
        track = self.tracks(1) and self.L == 2
        modes = settls_boundary_policy(self.L, 1, n1, self.m, self.c.chunk_size)
        prev = None
        for j in range(1, n1 + 1):
            hist = prev if track and modes[j - 1] == TWO_STEP else None
            prev = v[j - 1]
            v.append(self.step(1, v[j - 1], hist))
        return [self.p.prolong(1, x) for x in v]

    def run(self, u0: OracleState, iters=None) -> Trace:   # pint.py:355-394
        m, n0, n1 = self.m, self.c.N0, self.c.points_on(1)
        guess = self.initial_guess(u0)
        trace = Trace(snapshots=[guess])
        # np.atleast_1d: the oracle's batched states return arrays, a per-state
        # problem's states (the reference protocol, pint.py:185-189) plain scalars
        limit = 1e10 * max(float(np.atleast_1d(u0.max_abs())[0]), 1e-300)
        self.check(trace, 0, guess, limit)
        u = [None] * (n0 + 1)
        u[0] = u0.copy()
        for i in range(1, n1 + 1):
            u[m * i] = guess[i].copy()
            for j in range(m * (i - 1) + 1, m * i):
                u[j] = guess[i - 1].copy()
        for k in range(1, (self.c.max_iters if iters is None else iters) + 1):
            with np.errstate(over="ignore", invalid="ignore"):
                self.cycle(0, u, None, self.c.cycle)
            snap = [u[m * i].copy() for i in range(n1 + 1)]
            trace.snapshots.append(snap)
            self.check(trace, k, snap, limit)
        return trace

    @staticmethod
    def check(trace, k, snap, limit):                 # pint.py:396-400
        for i, v in enumerate(snap):
            if (not bool(np.atleast_1d(v.is_finite())[0])
                    or float(np.atleast_1d(v.max_abs())[0]) > limit):
                trace.blowup = {"iteration": k, "slice": i}
                raise PintBlowUp(k, i, trace)


def fine_serial_cpoints(problem: OracleProblem, pcfg: PintCfg, u0):   # pint.py:421-430
    out = [u0.copy()]
    v = u0.copy()
    for _ in range(pcfg.points_on(1)):
        for _ in range(pcfg.cfactor):
            v = problem.step(0, v)
        out.append(v.copy())
    return out


# -- diagnostics ------------------------------------------------------------------


def spectral_error(c, sph, cref, sph_ref, rnorm):      # diagnostics.py:46-65
    sel = (sph.m_of <= rnorm) & (sph.n_of <= rnorm)
    sel_r = (sph_ref.m_of <= rnorm) & (sph_ref.n_of <= rnorm)
    w, wr = c[..., sel], cref[..., sel_r]
    return float(np.abs(w - wr).max() / np.abs(wr).max())


def l2_error(g, gref):                                 # diagnostics.py:68-75
    den = np.sqrt(np.mean(gref ** 2))
    return float(np.sqrt(np.mean((g - gref) ** 2)) / den)


def phi_error_records(k, state, target_name, target, rnorms, include_l2=False):
    """Rows (k, rnorm, target, value) (diagnostics.py:99-118)."""
    common = state.sph if state.sph.M <= target.sph.M else target.sph
    s, t = state.to_truncation(common), target.to_truncation(common)
    rows = [(k, str(int(r)), target_name,
             spectral_error(s.phi[0], common, t.phi[0], common, r)) for r in rnorms]
    if include_l2:
        rows.append((k, "l2", target_name,
                     l2_error(common.synthesis(s.phi[0]), common.synthesis(t.phi[0]))))
    return rows


def ke_spectrum(state: OracleState):                   # diagnostics.py:78-87
    sph = state.sph
    a = sph.radius
    mult = np.where(sph.m_of == 0, 1.0, 2.0)
    power = mult * (np.abs(state.xi[0]) ** 2 + np.abs(state.delta[0]) ** 2)
    per_n = np.bincount(sph.n_of, weights=power, minlength=sph.M + 1)
    n = np.arange(1, sph.M + 1)
    energy = 0.25 * a * a / (n * (n + 1.0)) * per_n[1:]
    return n, 2.0 * np.pi * a / n, energy
