"""Batched / sharded MGRIT engine on a scalar fake problem (CPU only).

Mirrors the reference's engine tests (tests/test_pint.py with
tests/helpers.py:75-106 ScalarProblem): a step multiplies by a complex factor,
restriction/prolongation are the identity.  The batched engine must equal the
oracle restatement of MgritEngine iterate by iterate, Parareal must match the
textbook predictor-corrector recurrence, and a 2-rank gloo run must be bitwise
identical to the single-process run.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.mgrit import OracleMgrit, PintCfg, Level
from paper_2306_09497_b200 import pint


class Scalar:
    """Scalar 'state' for the oracle engine (copy/+/-/max_abs/is_finite)."""

    def __init__(self, v):
        self.v = complex(v)

    def copy(self):
        return Scalar(self.v)

    def __add__(self, o):
        return Scalar(self.v + o.v)

    def __sub__(self, o):
        return Scalar(self.v - o.v)

    def max_abs(self):
        return np.array([abs(self.v)])

    def is_finite(self):
        return np.array([np.isfinite(self.v)])


class OracleScalarProblem:
    def __init__(self, factors):
        self.f = factors
        self.step_calls = 0

    def step(self, level, value):
        self.step_calls += 1
        return Scalar(self.f[level] * value.v)

    def restrict(self, level, value):
        return value.copy()

    def prolong(self, level, value):
        return value.copy()


class BatchedScalarProblem:
    """Batched protocol of paper_2306_09497_b200.pint on CPU tensors [n]."""

    def __init__(self, factors):
        self.f = [complex(x) for x in factors]
        self.step_calls = 0

    def as_batch(self, level, v):
        return torch.as_tensor(np.atleast_1d(v), dtype=torch.complex128)

    def wrap(self, level, x):
        return complex(x[0])

    def zeros(self, level, n):
        return torch.zeros(n, dtype=torch.complex128)

    def step_batch(self, level, x):
        # explicit real arithmetic: torch's complex multiply rounds differently in
        # its SIMD body and scalar tail, which would make a slice's result depend
        # on its position in the batch
        self.step_calls += x.shape[0]
        f = self.f[level]
        re = x.real * f.real - x.imag * f.imag
        im = x.real * f.imag + x.imag * f.real
        return torch.complex(re, im)

    def restrict_batch(self, level, x):
        return x.clone()

    def prolong_batch(self, level, x):
        return x.clone()

    def stats_batch(self, level, x):
        return torch.isfinite(x), x.abs()


class _Cfg:
    def __init__(self, dt):
        self.dt = dt


def configs():
    """(name, factors, PintConfig) covering Parareal, MGRIT with relaxation, 3 levels."""
    out = []
    f2 = [0.9 + 0.3j, 0.8 + 0.5j]
    out.append(("parareal", f2, dict(L=2, cf=2, N0=16, nrelax=0, iters=5, cycle="F_then_V")))
    out.append(("mgrit2_fcf", f2, dict(L=2, cf=2, N0=16, nrelax=1, iters=4, cycle="F_then_V")))
    f3 = [0.97 + 0.1j, 0.9 + 0.25j, 0.75 + 0.45j]
    out.append(("mgrit3_fv", f3, dict(L=3, cf=2, N0=32, nrelax=1, iters=3, cycle="F_then_V")))
    out.append(("mgrit3_v_cf4", f3, dict(L=3, cf=4, N0=64, nrelax=2, iters=3, cycle="V")))
    return out


def engine_cfg(c):
    levels = tuple(pint.LevelSpec(i, 16, _Cfg(10.0 * c["cf"] ** i)) for i in range(c["L"]))
    return pint.PintConfig(levels=levels, T=10.0 * c["N0"], N0=c["N0"], cfactor=c["cf"],
                           nrelax=c["nrelax"], max_iters=c["iters"], cycle=c["cycle"])


def oracle_trace(factors, c):
    levels = tuple(Level(16, None) for _ in range(c["L"]))
    pc = PintCfg(levels=levels, T=10.0 * c["N0"], N0=c["N0"], cfactor=c["cf"],
                 nrelax=c["nrelax"], max_iters=c["iters"], cycle=c["cycle"])
    eng = OracleMgrit(OracleScalarProblem(factors), pc)
    eng.c = pc
    tr = eng.run(Scalar(1.0 + 0.0j))
    return [[s.v for s in snap] for snap in tr.snapshots]


@pytest.mark.parametrize("name,factors,c", configs())
def test_batched_engine_equals_oracle_engine(name, factors, c):
    prob = BatchedScalarProblem(factors)
    tr = pint.mgrit_run(prob, engine_cfg(c), 1.0 + 0.0j)
    ref = oracle_trace(factors, c)
    assert len(tr.snapshots) == len(ref)
    for k, (snap, rsnap) in enumerate(zip(tr.snapshots, ref)):
        got = snap.tensor.numpy()
        assert np.abs(got - np.array(rsnap)).max() <= 1e-14, (name, k)


def test_parareal_textbook_recurrence():
    """U_{k+1}[i] = G U_{k+1}[i-1] + F U_k[i-1] - G U_k[i-1] (test_pint.py:77-83)."""
    f, gco = 0.95 + 0.2j, 0.8 + 0.45j
    c = dict(L=2, cf=2, N0=12, nrelax=0, iters=4, cycle="F_then_V")
    tr = pint.parareal_run(BatchedScalarProblem([f, gco]), engine_cfg(c), 1.0 + 0.0j)
    n = 6
    Ff = f * f
    U = [gco ** i for i in range(n + 1)]
    for k in range(1, 5):
        new = [1.0 + 0.0j]
        for i in range(1, n + 1):
            new.append(gco * new[i - 1] + Ff * U[i - 1] - gco * U[i - 1])
        U = new
        assert np.abs(tr.snapshots[k].tensor.numpy() - np.array(U)).max() < 1e-13


def test_exact_convergence_bound():
    """Parareal reproduces the fine solution after N0/cfactor iterations."""
    f, gco = 0.95 + 0.2j, 0.8 + 0.45j
    c = dict(L=2, cf=2, N0=8, nrelax=0, iters=4, cycle="F_then_V")
    cfg = engine_cfg(c)
    tr = pint.parareal_run(BatchedScalarProblem([f, gco]), cfg, 1.0 + 0.0j)
    fine = np.array([(f * f) ** i for i in range(5)])
    assert np.abs(tr.snapshots[cfg.exact_convergence_bound].tensor.numpy() - fine).max() < 1e-14


def test_parareal_rejects_mgrit_config():
    c = dict(L=2, cf=2, N0=8, nrelax=1, iters=2, cycle="F_then_V")
    with pytest.raises(ValueError):
        pint.parareal_run(BatchedScalarProblem([0.9, 0.8]), engine_cfg(c), 1.0 + 0.0j)


def test_blowup_raises_with_trace():
    c = dict(L=2, cf=2, N0=8, nrelax=0, iters=6, cycle="F_then_V")
    with pytest.raises(pint.PintBlowUpError) as ei:
        pint.parareal_run(BatchedScalarProblem([1e4, 1e5]), engine_cfg(c), 1.0 + 0.0j)
    assert ei.value.trace.blowup is not None
    assert ei.value.trace.blowup["iteration"] == ei.value.iteration


def test_config_validation():
    with pytest.raises(ValueError):
        engine_cfg(dict(L=2, cf=2, N0=7, nrelax=0, iters=1, cycle="F_then_V"))
    with pytest.raises(ValueError):
        pint.PintConfig(levels=(pint.LevelSpec(0, 16, _Cfg(1.0)),), T=1.0, N0=1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class StridedScalarProblem(BatchedScalarProblem):
    """BatchedScalarProblem with the optional strided in-place step protocol
    (SweProblem.step_into: dst[i] = step(src[i]) on views of the level array)."""

    supports_deferred_check = True

    def __init__(self, factors):
        super().__init__(factors)
        self.into_calls = 0

    def check_deferred(self):
        pass

    def step_batch(self, level, x, deferred=False):
        return super().step_batch(level, x)

    def step_into(self, level, src, dst):
        assert src.shape == dst.shape and src.data_ptr() != dst.data_ptr()
        self.into_calls += 1
        dst.copy_(super().step_batch(level, src))
        return True


def _rank_main(rank, world, port, name, factors, c, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prob = (StridedScalarProblem if name.startswith("strided_") else BatchedScalarProblem)(factors)
        tr = pint.mgrit_run(prob, engine_cfg(c), 1.0 + 0.0j, comm=pint.Comm())
        snaps = np.stack([s.tensor.numpy() for s in tr.snapshots])
        out[rank] = (snaps, prob.step_calls, getattr(prob, "into_calls", None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,factors,c", configs())
def test_two_rank_gloo_bitwise(name, factors, c):
    single = pint.mgrit_run(BatchedScalarProblem(factors), engine_cfg(c), 1.0 + 0.0j)
    ref = np.stack([s.tensor.numpy() for s in single.snapshots])
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, name, factors, c, out))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for r in range(2):
        assert np.array_equal(out[r][0], ref), (name, r)


@pytest.mark.parametrize("name,factors,c", configs())
def test_strided_step_protocol_bitwise(name, factors, c):
    """A problem offering step_into has its unforced sweeps stepped on strided views
    of the level array (full array at one rank, LevelWindow blocks at two): same
    trace and step count as the gather / step_batch / scatter path."""
    plain = BatchedScalarProblem(factors)
    single = pint.mgrit_run(plain, engine_cfg(c), 1.0 + 0.0j)
    ref = np.stack([s.tensor.numpy() for s in single.snapshots])
    prob = StridedScalarProblem(factors)
    tr = pint.mgrit_run(prob, engine_cfg(c), 1.0 + 0.0j)
    assert np.array_equal(np.stack([s.tensor.numpy() for s in tr.snapshots]), ref)
    assert prob.into_calls > 0 and prob.step_calls == plain.step_calls
    assert tr.fine_steps == single.fine_steps
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, "strided_" + name, factors, c, out))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for r in range(2):
        assert np.array_equal(out[r][0], ref), (name, r)
        assert out[r][2] > 0, "the rank's LevelWindow sweeps did not take the strided path"


def test_stepper_config_implicit_solver():
    """StepperConfig keeps the reference fields and defaults; the GPU-only
    implicit_solver extension defaults to the reference fixed point and is
    validated and passed through the C struct."""
    from paper_2306_09497_b200 import steppers
    c = steppers.StepperConfig()
    assert c.implicit_solver == "fixed_point" and c.implicit_max_iter == 200
    assert c.to_c().implicit_solver == 0
    assert steppers.StepperConfig(implicit_solver="direct").to_c().implicit_solver == 1
    with pytest.raises(ValueError):
        steppers.StepperConfig(implicit_solver="lu")


def test_level_window_matches_full_array():
    """pint.LevelWindow (a rank's rows of the level-0 array, O(N0 / ranks)) reads and
    writes like the full array for every index form the engine uses."""
    import torch
    full = torch.arange(41, dtype=torch.float64).reshape(41, 1) * 1.5
    base, n = 16, 13   # rows 16..28: slices 9..14 of cfactor 2 plus their halo C-point
    w = pint.LevelWindow(full[base:base + n].clone(), base, 41, full[0:1].clone())
    assert w.shape == (41, 1)
    assert torch.equal(w[0:1], full[0:1]) and torch.equal(w[20], full[20])
    idx = torch.arange(base, base + n - 1, 2)
    assert torch.equal(w[idx], full[idx]) and torch.equal(w[idx + 1], full[idx + 1])
    assert torch.equal(w[base:base + n:2], full[base:base + n:2])
    w[idx + 1] = -w[idx]
    full[idx + 1] = -full[idx]
    assert torch.equal(w.data, full[base:base + n])
