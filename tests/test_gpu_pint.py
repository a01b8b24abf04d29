"""Batched GPU MGRIT / Parareal vs the reference engine's own traces.

Goldens (oracle/make_golden.py) are `pint.mgrit_run` traces of the reference:
every C-point of every iteration must match to 1e-10 relative sup-norm per
field (north star tolerance), plus the serial fine C-points.
"""

import numpy as np
import pytest

from conftest import load_golden, rel_diff

pytestmark = pytest.mark.gpu


def _setup(g):
    import torch
    from paper_2306_09497_b200 import dynamics, pint, spharm, steppers
    fine, coarse = int(g["fineM"]), int(g["coarseM"])
    dt0, nl, cf = float(g["dt0"]), int(g["nlevels"]), int(g["cfactor"])
    scheme = str(g["coarse_scheme"]) if "coarse_scheme" in g else "imex"
    levels = [pint.LevelSpec(0, fine, steppers.StepperConfig(
        dt=dt0, viscosity=dynamics.ViscositySpec(2, float(g["nu_f"]))))]
    for lv in range(1, nl):
        levels.append(pint.LevelSpec(lv, coarse, steppers.StepperConfig(
            scheme=scheme, dt=dt0 * cf ** lv,
            viscosity=dynamics.ViscositySpec(2, float(g["nu_c"])))))
    pc = pint.PintConfig(levels=tuple(levels), T=float(g["T"]),
                         N0=int(round(float(g["T"]) / dt0)), cfactor=cf,
                         nrelax=int(g["nrelax"]), max_iters=int(g["iters"]), cycle=str(g["cycle"]),
                         chunk_size=int(g["chunk_size"]) if "chunk_size" in g else 0)
    prob = pint.SweProblem(pc)
    u0 = g["u0"]
    st = dynamics.PrognosticState.from_fields(prob.grids[0], u0[0], u0[1], u0[2],
                                              [float(g["phibar"])])
    return pint, prob, pc, st


@pytest.mark.parametrize("name", ["pint_fixture_M16.npz", "pint_mgrit3_M24.npz",
                                  "pint_mgrit2_M32.npz", "pint_settls_M24.npz",
                                  "pint_settls_chunk_M24.npz"])
def test_gpu_engine_matches_reference_trace(name):
    g = load_golden(name)
    pint, prob, pc, u0 = _setup(g)
    fine = pint.fine_serial_cpoints(prob, pc, u0)
    ref_fine = g["fine"]
    for i in range(len(ref_fine)):
        assert rel_diff(fine.tensor[i].cpu().numpy(), ref_fine[i]) < 1e-10, ("fine", i)
    tr = pint.mgrit_run(prob, pc, u0)
    snaps = g["snapshots"]
    assert tr.iterations == snaps.shape[0] - 1
    worst = 0.0
    for k, snap in enumerate(tr.snapshots):
        got = snap.tensor.cpu().numpy()
        for i in range(got.shape[0]):
            d = rel_diff(got[i], snaps[k, i])
            worst = max(worst, d)
            assert d < 1e-10, (name, k, i, d)
    print(f"[PARITY] {name}: worst per-C-point relative sup-norm {worst:.2e}")


def test_gpu_engine_per_state_protocol():
    """SweProblem also serves the reference's per-state protocol (pint.py:172-194)."""
    g = load_golden("pint_mgrit3_M24.npz")
    pint, prob, pc, u0 = _setup(g)
    v = prob.step(0, u0)
    assert v is not u0 and rel_diff(u0.data[0].cpu().numpy(), g["u0"]) == 0.0  # pure step
    r = prob.restrict(0, v)
    assert r.grid is prob.grids[1]
    back = prob.prolong(1, r)
    assert back.grid is v.grid
    d = v - back                      # keeps only the modes n > M_coarse
    assert np.isfinite(d.max_abs())
    assert prob.is_finite(v) and prob.max_abs(v) > 0
    with pytest.raises(ValueError):
        _ = v + r                     # different grids (dynamics.py:87-89)
    assert prob.copy(v).grid is prob.grids[0] and not prob.tracks_history(0)


def test_gpu_blowup_raises():
    """A diverging run raises PintBlowUpError carrying the partial trace (pint.py:396-400)."""
    g = load_golden("pint_fixture_M16.npz")
    pint, prob, pc, u0 = _setup(g)
    bad = u0.copy()
    bad.data[0, 2, 5] = float("nan")
    with pytest.raises(pint.PintBlowUpError) as ei:
        pint.mgrit_run(prob, pc, bad)
    assert ei.value.trace.blowup is not None


def test_device_sweep_matches_stepwise():
    """swe_imex_sweep (the coarsest solve on the device) equals stepping point by
    point and adding the forcing, bitwise; an unconverged solve still raises."""
    import torch
    from paper_2306_09497_b200 import dynamics, pint, scenarios, steppers
    g = load_golden("pint_mgrit2_M32.npz")
    _, prob, pc, u0 = _setup(g)
    lv = 1
    grid = prob.grids[lv]
    n = 6
    u = prob.zeros(lv, n + 1)
    u[0:1] = prob.restrict_batch(0, prob.as_batch(0, u0))
    rng = np.random.default_rng(1)
    taper = (grid.n_of + 1.0) ** -2
    f = torch.zeros_like(u)
    f[:, 0] = torch.from_numpy(rng.standard_normal((n + 1, grid.n_modes)) * taper).to(u.device)
    f[:, 1] = torch.from_numpy(rng.standard_normal((n + 1, grid.n_modes)) * 1e-9 * taper).to(u.device)
    ref = u.clone()
    for j in range(1, n + 1):
        ref[j:j + 1] = prob.step_batch(lv, ref[j - 1:j]) + f[j:j + 1]
    assert prob.sweep_batch(lv, u, f)
    assert bool(torch.isfinite(ref).all()) and torch.equal(u, ref)
    bad = pint.SweProblem(pint.PintConfig(
        levels=(pc.levels[0], pint.LevelSpec(1, grid.M, steppers.StepperConfig(
            dt=pc.levels[1].stepper.dt, implicit_max_iter=1))),
        T=pc.T, N0=pc.N0, cfactor=pc.cfactor))
    bad.phibar = prob.phibar
    for _ in range(2):   # second call replays the captured graph
        w = u.clone()
        with pytest.raises(steppers.ImplicitSolveError, match="residual"):
            bad.sweep_batch(1, w, None)
