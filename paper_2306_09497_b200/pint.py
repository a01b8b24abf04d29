"""Batched (and slice-sharded) FAS-MGRIT / Parareal driver.

Mirror of `/root/reference/pkg/src/pintswe/pint.py`: PintBlowUpError (:33-41),
LevelSpec (:44-53), PintConfig (:55-95), IterationTrace (:122-135),
speedup_report (:146-154), SweProblem (:157-194), MgritEngine (:197-400),
mgrit_run / parareal_run / fine_serial_cpoints (:403-430).

Differences are in execution only, never in the iterates:
* every sweep (F, C, residual, tau) is ONE batched propagator call over all
  slices instead of a thread-pool task per slice (pint.py:209-219);
* level arrays are tensors [points, ...] (for the SWE: [points, 3, K]
  complex128 on the GPU);
* with a `comm` (torch.distributed), level-0 slices are sharded in
  contiguous blocks over ranks; a rank sends its last C-point to rank+1 before
  every F-sweep (the only data dependence between slices, pint.py:229-231),
  the coarsest serial sweep (pint.py:306-320) runs redundantly on every rank
  after an all-gather of its forcing, and blow-up flags are all-reduced.
Rank-count determinism (the reference's worker-count contract):
a rank's share of a sweep is stepped with the kernels chosen for the sweep's
GLOBAL point count (`select_batch`, see steppers.py), and the serial sweeps
(coarsest level, initial guess) run one point per call on every rank, so each
point's arithmetic is the same for any number of ranks and the traces are
bitwise identical (tests/test_gpu_multirank.py).
The SL-SI-SETTLS history policy (pint.py:103-119) is followed in the FAS tau,
the coarsest sweep and the initial guess.
"""

from __future__ import annotations

import dataclasses
import time
from typing import Optional, Sequence

import numpy as np
import torch

from ._lib import NoConvergence as _NoConv
from ._lib import check as _lib_check

F_THEN_V = "F_then_V"
SL_SI_SETTLS, ONE_STEP, TWO_STEP = "sl_si_settls", "one_step", "two_step"


def settls_boundary_policy(nlevels: int, level_index: int, nsteps: int, cfactor: int,
                           chunk_size: int):
    """Per-step SETTLS mode of one level (pint.py:103-119): one-step below the
    coarsest level; on the coarsest, two-step except where the step's history
    would sit in another chunk of `chunk_size` fine C-point slices."""
    if level_index < nlevels - 1:
        return [ONE_STEP] * nsteps
    spacing = cfactor ** (nlevels - 2)
    return [ONE_STEP if chunk_size > 0 and ((j - 1) * spacing) % chunk_size == 0 else TWO_STEP
            for j in range(1, nsteps + 1)]
V_CYCLE = "V"


class PintBlowUpError(RuntimeError):
    """Non-finite or runaway state detected; carries the partial trace."""

    def __init__(self, iteration: int, slice_index: int, trace: "IterationTrace"):
        super().__init__(f"blow-up at iteration {iteration}, slice {slice_index}")
        self.iteration = iteration
        self.slice_index = slice_index
        self.trace = trace


@dataclasses.dataclass(frozen=True)
class LevelSpec:
    index: int
    M: int
    stepper: object  # steppers.StepperConfig

    @property
    def dt(self) -> float:
        return self.stepper.dt


@dataclasses.dataclass(frozen=True)
class PintConfig:
    levels: tuple
    T: float
    N0: int
    cfactor: int = 2
    nrelax: int = 0
    max_iters: int = 10
    chunk_size: int = 0
    cycle: str = F_THEN_V

    def __post_init__(self):
        L = len(self.levels)
        if L < 2:
            raise ValueError("need at least two levels")
        if self.cfactor < 2:
            raise ValueError("coarsening factor must be >= 2")
        if self.nrelax < 0 or self.max_iters < 0 or self.chunk_size < 0:
            raise ValueError("nrelax, max_iters and chunk_size must be >= 0")
        if self.cycle not in (F_THEN_V, V_CYCLE):
            raise ValueError(f"unknown cycle {self.cycle!r}")
        dt0 = self.levels[0].dt
        if abs(self.N0 * dt0 - self.T) > 1e-9 * max(self.T, 1.0):
            raise ValueError("N0 * dt_0 must equal the horizon T")
        for lv in range(1, L):
            ratio = self.levels[lv].dt / self.levels[lv - 1].dt
            if abs(ratio - self.cfactor) > 1e-9:
                raise ValueError("level time steps must follow dt_{l+1} = cfactor*dt_l")
            if self.levels[lv].M > self.levels[0].M:
                raise ValueError("coarse levels cannot exceed the fine truncation")
        if self.N0 % self.cfactor ** (L - 1) != 0:
            raise ValueError("N0 must be divisible by cfactor^(nlevels-1)")

    @property
    def nlevels(self) -> int:
        return len(self.levels)

    def points_on(self, level: int) -> int:
        return self.N0 // self.cfactor ** level

    @property
    def exact_convergence_bound(self) -> int:
        return int(np.ceil(self.N0 / ((self.nrelax + 1) * self.cfactor)))


class SnapshotList(list):
    """One iteration's C-point snapshots; items materialise as problem states."""

    def __init__(self, problem, tensor):
        super().__init__(range(tensor.shape[0]))
        self.tensor = tensor
        self._problem = problem

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        n = len(self)
        if i < 0:
            i += n
        return self._problem.wrap(0, self.tensor[i:i + 1])

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]


@dataclasses.dataclass
class IterationTrace:
    """Level-0 C-point snapshots per iteration (iteration 0: initial guess)."""

    times: np.ndarray
    snapshots: list
    wall_times: list
    config: PintConfig
    blowup: Optional[dict] = None
    fine_reference: Optional[Sequence] = None
    fine_steps: list = dataclasses.field(default_factory=list)

    @property
    def iterations(self) -> int:
        return len(self.snapshots) - 1


@dataclasses.dataclass(frozen=True)
class SpeedupRecord:
    iteration: int
    wall_time: float
    cumulative_time: float
    speedup: float


def speedup_report(trace: IterationTrace, t_ref: float):
    """pint.py:146-154."""
    out, cum = [], 0.0
    for k, wt in enumerate(trace.wall_times):
        cum += wt
        out.append(SpeedupRecord(k, wt, cum, t_ref / cum if cum > 0 else 0.0))
    return out


class Comm:
    """Slice-block exchange over torch.distributed.

    NCCL (one rank per GPU): device buffers go over NVLink directly.  Any other
    backend (gloo: CPU tests, or several ranks sharing one GPU in the multi-rank
    parity test) stages device tensors through host memory, so no kernel of one
    rank ever waits on another rank's kernels.
    """

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.stage = dist.get_backend(group) != "nccl"

    def _wire(self, t: torch.Tensor) -> torch.Tensor:
        t = t.contiguous()
        return t.cpu() if self.stage and t.is_cuda else t

    def halo(self, send: torch.Tensor, recv: torch.Tensor):
        """send -> rank+1, recv <- rank-1 (first/last rank skip)."""
        d = self.dist
        ops = []
        if self.rank + 1 < self.size:
            ops.append(d.P2POp(d.isend, self._wire(send), self.rank + 1, self.group))
        buf = None
        if self.rank > 0:
            buf = torch.empty(recv.shape, dtype=recv.dtype,
                              device="cpu" if self.stage else recv.device)
            ops.append(d.P2POp(d.irecv, buf, self.rank - 1, self.group))
        if ops:
            for req in d.batch_isend_irecv(ops):
                req.wait()
        if buf is not None:
            recv.copy_(buf)

    def all_gather(self, local: torch.Tensor) -> torch.Tensor:
        src = self._wire(local)
        out = torch.empty((self.size * local.shape[0],) + tuple(local.shape[1:]),
                          dtype=local.dtype, device=src.device)
        if out.is_complex():
            self.dist.all_gather_into_tensor(torch.view_as_real(out), torch.view_as_real(src),
                                             group=self.group)
        else:
            self.dist.all_gather_into_tensor(out, src, group=self.group)
        return out.to(local.device)

    def min_int(self, v: int) -> int:
        t = torch.tensor([v], dtype=torch.int64,
                         device="cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return int(t[0])


class LevelWindow:
    """Rows [base, base + n) of a level array of `total` rows, addressed with the
    global row indices the engine uses (ints, slices, index tensors); row 0 (the
    initial condition) is kept separately when it lies outside the window.  A
    rank holding a contiguous block of slices keeps O(N0 / ranks) level-0 states
    instead of all N0 + 1."""

    def __init__(self, data: torch.Tensor, base: int, total: int, row0: torch.Tensor):
        self.data, self.base, self.total, self.row0 = data, base, total, row0

    @property
    def shape(self):
        return (self.total,) + tuple(self.data.shape[1:])

    @property
    def device(self):
        return self.data.device

    def _loc(self, i):
        if isinstance(i, slice):
            start = 0 if i.start is None else i.start
            stop = self.total if i.stop is None else i.stop
            return slice(start - self.base, stop - self.base, i.step)
        return i - self.base

    def __getitem__(self, i):
        if self.base > 0 and isinstance(i, slice) and i.start in (0, None) and i.stop == 1:
            return self.row0
        return self.data[self._loc(i)]

    def __setitem__(self, i, v):
        self.data[self._loc(i)] = v


class MgritEngine:
    """FAS-MGRIT / Parareal over a batched problem (pint.py:197-400 semantics).

    The problem provides step_batch(level, x), restrict_batch(level, x),
    prolong_batch(level, x), stats_batch(level, x) -> (finite, max_abs) and
    wrap(level, x) (tensors with a leading point axis).
    """

    def __init__(self, problem, config: PintConfig, comm: Optional[Comm] = None):
        self.problem = problem
        self.cfg = config
        self.m = config.cfactor
        self.L = config.nlevels
        self.comm = comm
        self.G = comm.size if comm else 1
        self.g = comm.rank if comm else 0
        self.fine_steps = 0
        for lv in range(self.L - 1):
            n = config.points_on(lv) // self.m
            if n % self.G:
                raise ValueError(f"level {lv}: {n} slices do not split over {self.G} ranks")
        if self.G > 1:
            n1 = config.points_on(1) // self.G     # coarse points per rank, level 1
            if self.L > 2 and n1 % self.m:
                raise ValueError("rank blocks must align with coarse slices")

    # slices owned by this rank on `level` (1-based slice indices)
    def _own(self, level: int, n: int):
        S = n // self.G
        return self.g * S + 1, (self.g + 1) * S

    def _tracks(self, level) -> bool:
        """Problem keeps SETTLS two-step history on `level` (optional protocol)."""
        f = getattr(self.problem, "tracks_history", None)
        return bool(f(level)) if f is not None else False

    def _step(self, level, x, prev=None, sharded=True):
        """One step of every point of x.  sharded: x is this rank's share of a sweep
        over G * len(x) points; the problem then picks its kernels for the global
        count (select_batch), so every rank count runs the same arithmetic per
        point.  Serial calls (coarsest sweep, initial guess) run on every rank
        alike and pass no hint."""
        if level == 0:
            self.fine_steps += x.shape[0]
        kw = {}
        if getattr(self.problem, "supports_select_batch", False):
            kw["select_batch"] = x.shape[0] * self.G if sharded else 0
        kw.update(self._deferred_kw())
        if prev is None:
            return self.problem.step_batch(level, x, **kw)
        return self.problem.step_batch(level, x, prev, **kw)

    def _step_into(self, level, u, src0, dst, count) -> bool:
        """step(u[src0 + i m]), i < count, written to u[dst + i m] (dst an int: in place
        on strided views of the level array) or to the tensor dst, where the problem
        supports it (no forcing on this path)."""
        f = getattr(self.problem, "step_into", None)
        if (f is None or count <= 0
                or not getattr(self.problem, "supports_deferred_check", False)):
            return False
        m = self.m
        if isinstance(u, LevelWindow):  # a rank's block of the level: local rows
            last = (count - 1) * m - u.base
            if (src0 < u.base or src0 + last >= u.data.shape[0]
                    or (isinstance(dst, int) and (dst < u.base or dst + last >= u.data.shape[0]))):
                return False
            src0 -= u.base
            if isinstance(dst, int):
                dst -= u.base
            u = u.data
        if not isinstance(u, torch.Tensor):
            return False
        src = u[src0:src0 + (count - 1) * m + 1:m]
        if isinstance(dst, int):
            dst = u[dst:dst + (count - 1) * m + 1:m]
        kw = {}
        if getattr(self.problem, "supports_select_batch", False):
            kw["select_batch"] = count * self.G
        if not f(level, src, dst, **kw):
            return False
        if level == 0:
            self.fine_steps += count
        return True

    def _deferred_kw(self):
        """Steps and sweeps queued without a host round trip where the problem
        supports it; their errors are raised once per cycle (_check_deferred)."""
        return {"deferred": True} if getattr(self.problem, "supports_deferred_check", False) else {}

    def _check_deferred(self):
        """Raise the problem's deferred step errors (ImplicitSolveError of a step
        queued without a host round trip) before the iteration's results are used."""
        f = getattr(self.problem, "check_deferred", None)
        if f is not None:
            f()

    def _exchange_halo(self, level, u):
        if self.G == 1:
            return
        n = (u.shape[0] - 1) // self.m
        lo, hi = self._own(level, n)
        self.comm.halo(u[self.m * hi], u[self.m * (lo - 1)])

    # -- relaxation sweeps (pint.py:223-263) ------------------------------------
    def _f_sweep(self, level, u, g):
        m = self.m
        n = (u.shape[0] - 1) // m
        lo, hi = self._own(level, n)
        self._exchange_halo(level, u)
        if g is None:
            # unforced level: each F-point stepped straight into its neighbour
            s = 1
            while s < m and self._step_into(level, u, m * (lo - 1) + s - 1, m * (lo - 1) + s,
                                            hi - lo + 1):
                s += 1
            if s == m:
                return
            assert s == 1  # (a problem either supports the level or does not)
        left = torch.arange(m * (lo - 1), m * hi, m, device=u.device)
        x = u[left]
        for s in range(1, m):
            x = self._step(level, x)
            if g is not None:
                x = x + g[left + s]
            u[left + s] = x

    def _c_sweep(self, level, u, g):
        m = self.m
        n = (u.shape[0] - 1) // m
        lo, hi = self._own(level, n)
        if g is None and self._step_into(level, u, m * lo - 1, m * lo, hi - lo + 1):
            return
        cp = torch.arange(m * lo, m * hi + 1, m, device=u.device)
        x = self._step(level, u[cp - 1])
        if g is not None:
            x = x + g[cp]
        u[cp] = x

    def relax_fcf(self, level, u, g, nrelax):
        self._f_sweep(level, u, g)
        for _ in range(nrelax):
            self._c_sweep(level, u, g)
            self._f_sweep(level, u, g)

    # -- FAS components (pint.py:267-304) ----------------------------------------
    def _residual(self, level, u, g, lo, hi):
        m = self.m
        cp = torch.arange(m * lo, m * hi + 1, m, device=u.device)
        prop = None
        if isinstance(u, (torch.Tensor, LevelWindow)):  # from the strided view, no gather / clone
            ref = u.data if isinstance(u, LevelWindow) else u
            prop = torch.empty((hi - lo + 1,) + tuple(ref.shape[1:]), dtype=ref.dtype, device=ref.device)
            if not self._step_into(level, u, m * lo - 1, prop, hi - lo + 1):
                prop = None
        if prop is None:
            prop = self._step(level, u[cp - 1])
        if g is not None:
            prop = prop + g[cp]
        return prop - u[cp]

    def _fas_restrict(self, level, u, g):
        """Returns ubar, gbar as full-length coarse arrays (valid on owned points + halo)."""
        m = self.m
        n = (u.shape[0] - 1) // m
        lo, hi = self._own(level, n)
        pr = self.problem
        cps = torch.arange(m * (lo - 1), m * hi + 1, m, device=u.device)   # halo + owned
        ub_local = pr.restrict_batch(level, u[cps])
        r = self._residual(level, u, g, lo, hi)
        prev = None
        if self._tracks(level + 1):
            # the coarse operator sees the coarse sweep's history pattern
            # (pint.py:287-299): slice i >= 2 in two-step mode uses ubar[i-2]
            modes = settls_boundary_policy(self.L, level + 1, n, m, self.cfg.chunk_size)
            prev = ub_local[:-1].clone()
            for i in range(lo, hi + 1):
                if i >= 2 and modes[i - 1] == TWO_STEP:
                    if i - 2 < lo - 1:
                        raise NotImplementedError(
                            "SETTLS history across rank blocks: set chunk_size to a "
                            "multiple of the slices per rank")
                    prev[i - lo] = ub_local[i - 2 - (lo - 1)]
        tau = ub_local[1:] - self._step(level + 1, ub_local[:-1], prev)
        gb_local = pr.restrict_batch(level, r) + tau
        ubar = pr.zeros(level + 1, n + 1)
        gbar = pr.zeros(level + 1, n + 1)
        ubar[lo - 1:hi + 1] = ub_local
        gbar[lo:hi + 1] = gb_local
        if lo > 1:
            # point 0 (the initial condition) is known everywhere; the serial
            # coarsest sweep of every rank starts from it
            ubar[0:1] = pr.restrict_batch(level, u[0:1])
        return ubar, gbar

    def _coarsest_solve(self, u, g):
        """Serial sweep on the coarsest level (pint.py:306-320); with ranks, every
        rank gathers the forcing and runs the identical sweep."""
        lv = self.L - 1
        n = u.shape[0] - 1
        if self.G > 1:
            lo, hi = self._own_points(lv, n)
            g = torch.cat([g[:1], self.comm.all_gather(g[lo:hi + 1])])
        modes = settls_boundary_policy(self.L, lv, n, self.m, self.cfg.chunk_size)
        track = self._tracks(lv)
        sweep = getattr(self.problem, "sweep_batch", None)
        if sweep is not None and sweep(lv, u, g, **self._deferred_kw()):  # chain on the device
            return
        prev = None
        for j in range(1, n + 1):
            hist = prev if track and modes[j - 1] == TWO_STEP else None
            new = self._step(lv, u[j - 1:j], hist, sharded=False)
            if g is not None:
                new = new + g[j:j + 1]
            prev = u[j - 1:j].clone()
            u[j:j + 1] = new

    def _own_points(self, level, npts):
        S = npts // self.G
        return self.g * S + 1, (self.g + 1) * S

    def _cycle(self, level, u, g, kind):
        if level == self.L - 1:
            self._coarsest_solve(u, g)
            return
        m = self.m
        n = (u.shape[0] - 1) // m
        lo, hi = self._own(level, n)
        self.relax_fcf(level, u, g, self.cfg.nrelax)
        ubar, gbar = self._fas_restrict(level, u, g)
        v = ubar.clone()
        self._cycle(level + 1, v, gbar, kind)
        own = torch.arange(lo, hi + 1, device=u.device)
        err = v[own] - ubar[own]
        u[m * own] = u[m * own] + self.problem.prolong_batch(level + 1, err)
        self._f_sweep(level, u, g)
        if kind == F_THEN_V and level + 1 < self.L - 1:
            self._cycle(level, u, g, V_CYCLE)

    # -- driver (pint.py:341-400) ----------------------------------------------------
    def _initial_guess(self, u0):
        """Serial level-1 run prolonged to level 0 (also when L = 3, pint.py:341-353)."""
        n1 = self.cfg.points_on(1)
        pr = self.problem
        v = pr.zeros(1, n1 + 1)
        v[0:1] = pr.restrict_batch(0, u0)
        track = self._tracks(1) and self.L == 2
        sweep = getattr(pr, "sweep_batch", None)
        if not track and sweep is not None and sweep(1, v, None, **self._deferred_kw()):
            # the whole serial run on the device (swe_imex_sweep: one step graph per
            # point, one host check), bitwise the per-step loop below
            return pr.prolong_batch(1, v)
        modes = settls_boundary_policy(self.L, 1, n1, self.m, self.cfg.chunk_size)
        for j in range(1, n1 + 1):
            hist = v[j - 2:j - 1] if track and j >= 2 and modes[j - 1] == TWO_STEP else None
            v[j:j + 1] = self._step(1, v[j - 1:j], hist, sharded=False)
        return pr.prolong_batch(1, v)

    def _cpoints(self, u):
        """All level-0 C-points (gathered across ranks)."""
        m = self.m
        n = (u.shape[0] - 1) // m
        if self.G == 1:
            return u[::m].clone()
        lo, hi = self._own(0, n)
        mine = u[m * lo: m * hi + 1: m]
        return torch.cat([u[0:1], self.comm.all_gather(mine)])

    def run(self, u0, fine_reference=None, initial_cpoints=None, keep_snapshots=True,
            sync=None, clock=None) -> IterationTrace:
        """u0: tensor [1, ...] on level 0.  sync(): device barrier for wall times.
        clock: optional object with start() / stop() -> seconds timing each
        iteration's cycle (default: host perf_counter between sync() calls, the
        reference's per-iteration wall time, pint.py:384-390)."""
        cfg = self.cfg
        m = self.m
        n0, n1 = cfg.N0, cfg.points_on(1)
        sync = sync or (lambda: None)
        times = np.arange(n1 + 1) * (m * cfg.levels[0].dt)
        sync()
        t0 = time.perf_counter()
        if initial_cpoints is None:
            guess = self._initial_guess(u0)
        else:
            if len(initial_cpoints) != n1 + 1:
                raise ValueError("initial_cpoints must cover every C-point")
            guess = initial_cpoints.clone()
        self._check_deferred()
        sync()
        trace = IterationTrace(times=times, snapshots=[SnapshotList(self.problem, guess)],
                               wall_times=[time.perf_counter() - t0], config=cfg,
                               fine_reference=fine_reference)
        _, mx0 = self.problem.stats_batch(0, u0)
        limit = 1e10 * max(float(mx0[0]), 1e-300)
        self._check_finite(trace, 0, guess, limit)
        if self.G == 1:
            u = self.problem.zeros(0, n0 + 1)
            u[0:1] = u0
            idx = torch.arange(1, n1 + 1, device=u.device)
        else:
            # this rank's slices lo..hi and the C-point before them (the halo)
            lo, hi = self._own(0, n1)
            base = m * (lo - 1)
            u = LevelWindow(self.problem.zeros(0, m * (hi - lo + 1) + 1), base, n0 + 1,
                            u0.clone())
            if base == 0:
                u[0:1] = u0
            else:
                u[base:base + 1] = guess[lo - 1:lo]
            idx = torch.arange(lo, hi + 1, device=u.device)
        u[m * idx] = guess[idx]
        for s in range(1, m):
            u[m * (idx - 1) + s] = guess[idx - 1]
        for k in range(1, cfg.max_iters + 1):
            f0 = self.fine_steps
            if clock is not None:
                clock.start()
                self._cycle(0, u, None, cfg.cycle)
                self._check_deferred()
                trace.wall_times.append(clock.stop())
            else:
                sync()
                t0 = time.perf_counter()
                self._cycle(0, u, None, cfg.cycle)
                self._check_deferred()
                sync()
                trace.wall_times.append(time.perf_counter() - t0)
            trace.fine_steps.append(self.fine_steps - f0)
            snap = self._cpoints(u)
            trace.snapshots.append(SnapshotList(self.problem, snap) if keep_snapshots else None)
            self._check_finite(trace, k, snap, limit)
        return trace

    def _check_finite(self, trace, iteration, snap, limit):
        fin, mx = self.problem.stats_batch(0, snap)
        bad = (~fin) | (mx > limit)
        first = int(torch.nonzero(bad)[0]) if bool(bad.any()) else 1 << 60
        if self.comm is not None:
            first = self.comm.min_int(first)
        if first < (1 << 60):
            trace.blowup = {"iteration": iteration, "slice": first}
            raise PintBlowUpError(iteration, first, trace)


def mgrit_run(problem, config: PintConfig, u0, workers: int = 1, fine_reference=None,
              initial_cpoints=None, comm: Optional[Comm] = None) -> IterationTrace:
    """Run MGRIT (pint.py:403-408); `workers` is accepted for API parity (the
    batch replaces the thread pool)."""
    x0 = problem.as_batch(0, u0)
    ic = None if initial_cpoints is None else problem.as_batch(0, initial_cpoints)
    return MgritEngine(problem, config, comm).run(x0, fine_reference, ic)


def parareal_run(problem, config: PintConfig, u0, workers: int = 1, fine_reference=None,
                 initial_cpoints=None, comm: Optional[Comm] = None) -> IterationTrace:
    """Parareal = two-level F-relaxation MGRIT (pint.py:411-418)."""
    if config.nlevels != 2 or config.nrelax != 0:
        raise ValueError("Parareal requires nlevels=2 and nrelax=0")
    return mgrit_run(problem, config, u0, workers, fine_reference, initial_cpoints, comm)


def fine_serial_cpoints(problem, config: PintConfig, u0):
    """Serial fine solution at the level-0 C-points (pint.py:421-430)."""
    x = problem.as_batch(0, u0)
    out = [x.clone()]
    for _ in range(config.points_on(1)):
        for _ in range(config.cfactor):
            x = problem.step_batch(0, x)
        out.append(x.clone())
    return SnapshotList(problem, torch.cat(out))


class SweProblem:
    """Shallow-water levels on the GPU (pint.py:157-194), batched and per-state.

    Batched protocol (used by MgritEngine): tensors [points, 3, K] complex128.
    Per-state protocol (drop-in for the reference engine): step/restrict/
    prolong/copy/max_abs/is_finite/tracks_history on PrognosticState objects.
    """

    def __init__(self, config: PintConfig, geometry=None, phibar: Optional[float] = None):
        from .spharm import SphereGeometry, get_grid
        from .steppers import IMEX
        self.config = config
        self.geometry = geometry or SphereGeometry()
        self.grids = [get_grid(spec.M, self.geometry) for spec in config.levels]
        # SETTLS below the coarsest level runs one-step (pint.py:164-170)
        L = config.nlevels
        self.level_cfgs = [dataclasses.replace(spec.stepper, settls_mode=ONE_STEP)
                           if spec.stepper.scheme == SL_SI_SETTLS and lv < L - 1 else spec.stepper
                           for lv, spec in enumerate(config.levels)]
        self.phibar = phibar
        self.step_calls = 0
        self._pending = set()  # levels with deferred (unchecked) steps

    # -- batched protocol --------------------------------------------------------
    def _pb(self, n, dev):
        return torch.full((n,), float(self.phibar), dtype=torch.float64, device=dev)

    def as_batch(self, level, value):
        from .dynamics import PrognosticState
        if isinstance(value, PrognosticState):
            if self.phibar is None:
                self.phibar = value.phibar
            return value.data
        if isinstance(value, (list, tuple)):
            return torch.cat([self.as_batch(level, v) for v in value])
        return value

    def wrap(self, level, x):
        from .dynamics import PrognosticState
        return PrognosticState(self.grids[level], x, self._pb(x.shape[0], x.device))

    def zeros(self, level, n):
        g = self.grids[level]
        return torch.zeros((n, 3, g.n_modes), dtype=torch.complex128, device=f"cuda:{g.device}")

    supports_select_batch = True
    supports_deferred_check = True

    def check_deferred(self):
        """ImplicitSolveError if a deferred step (step_batch(..., deferred=True))
        did not converge (steppers.py:113-118)."""
        from .steppers import check_async_steps
        pending, self._pending = self._pending, set()
        for level in sorted(pending):
            check_async_steps(self.grids[level])

    def step_batch(self, level, x, prev=None, select_batch=0, deferred=False):
        """One step of every point of x; prev (SETTLS two-step history, same shape)
        or None.  For SETTLS a point's own value as its prev means no history.
        select_batch: kernel-selection batch (steppers module docstring).
        deferred: queue an IMEX step without a host round trip; an unconverged
        solve is raised by check_deferred (the engine calls it once per cycle)."""
        from .steppers import IMEX, imex_steps_async, imex_steps_inplace, settls_step_inplace
        st = self.wrap(level, x.clone())
        self.step_calls += x.shape[0]
        cfg = self.level_cfgs[level]
        if cfg.scheme == IMEX and deferred:
            imex_steps_async(st, cfg, 1, select_batch=select_batch)
            self._pending.add(level)
        elif cfg.scheme == IMEX:
            imex_steps_inplace(st, cfg, 1, select_batch=select_batch)
        else:
            settls_step_inplace(st, cfg, None if prev is None else self.wrap(level, prev),
                                select_batch=select_batch)
        return st.data

    def step_into(self, level, src, dst, select_batch=0) -> bool:
        """dst[i] = step(src[i]) for strided views of a level array (every m-th point),
        queued like step_batch(..., deferred=True) but without the gather, clone and
        scatter copies (swe_imex_step_async_io); False when the level is not a plain
        IMEX level (the caller then uses step_batch)."""
        from .steppers import IMEX, imex_step_async_io
        cfg = self.level_cfgs[level]
        if cfg.scheme != IMEX or src.shape[0] == 0:
            return False
        self.step_calls += src.shape[0]
        imex_step_async_io(self.grids[level], src, dst, self._pb(src.shape[0], src.device), cfg, 1,
                           select_batch=select_batch)
        self._pending.add(level)
        return True

    def sweep_batch(self, level, u, g, deferred=False) -> bool:
        """u[j] = step(u[j-1]) + g[j], j = 1..n, in place on the device
        (swe_imex_sweep); False when the level is not a plain IMEX level.
        deferred: no host check at the end (swe_imex_sweep_async); an unconverged
        solve is raised by check_deferred."""
        import ctypes
        from .spharm import _ptr, _stream
        from .steppers import IMEX, ImplicitSolveError
        cfg = self.level_cfgs[level]
        if cfg.scheme != IMEX or u.shape[0] < 2:
            return False
        grid = self.grids[level]
        n = u.shape[0] - 1
        self.step_calls += n
        pb = self._pb(1, u.device)
        c = cfg.to_c()
        resid = np.zeros(1)
        if deferred:
            rc = grid._lib.swe_imex_sweep_async(grid.plan, _ptr(u), None if g is None else _ptr(g),
                                                n, _ptr(pb), ctypes.byref(c), _stream())
            self._pending.add(level)
        else:
            rc = grid._lib.swe_imex_sweep(grid.plan, _ptr(u), None if g is None else _ptr(g), n,
                                          _ptr(pb), ctypes.byref(c),
                                          resid.ctypes.data_as(ctypes.c_void_p), _stream())
        try:
            _lib_check(rc, "swe_imex_sweep")
        except _NoConv as exc:
            raise ImplicitSolveError(str(exc)) from None
        return True

    def restrict_batch(self, level, x):
        from .spharm import truncate_pad
        return truncate_pad(x, self.grids[level], self.grids[level + 1])

    def prolong_batch(self, level, x):
        from .spharm import truncate_pad
        return truncate_pad(x, self.grids[level], self.grids[level - 1])

    def stats_batch(self, level, x):
        st = self.wrap(level, x)
        mx = st.max_abs_each()
        return st._fin.bool(), mx

    # -- per-state protocol (pint.py:172-194) --------------------------------------
    def step(self, level, value, prev=None):
        from .steppers import StepperState, advance
        self.step_calls += value.batch
        return advance(StepperState(value, prev), self.level_cfgs[level]).current

    def restrict(self, level, value):
        return value.to_truncation(self.grids[level + 1])

    def prolong(self, level, value):
        return value.to_truncation(self.grids[level - 1])

    def copy(self, value):
        return value.copy()

    def max_abs(self, value) -> float:
        return value.max_abs()

    def is_finite(self, value) -> bool:
        return value.is_finite()

    def tracks_history(self, level) -> bool:
        """pint.py:192-194."""
        from .steppers import SL_SI_SETTLS, TWO_STEP as TS
        cfg = self.level_cfgs[level]
        return cfg.scheme == SL_SI_SETTLS and cfg.settls_mode == TS
