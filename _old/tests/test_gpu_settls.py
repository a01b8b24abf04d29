"""SL-SI-SETTLS on the GPU vs the reference (goldens from oracle/make_golden.py):
the stepper (cold start, two-step history, one-step mode), departure points and
the bicubic interpolation (steppers.py:171-212, semilag.py:25-179)."""

import numpy as np
import pytest

from conftest import load_golden, rel_diff

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    import torch
    assert torch.cuda.is_available()
    from paper_2306_09497_b200 import dynamics, semilag, spharm, steppers
    return spharm, dynamics, steppers, semilag


def _cfg(steppers, dynamics, g, mode="two_step"):
    return steppers.StepperConfig(scheme="sl_si_settls", dt=float(g["dt"]), settls_mode=mode,
                                  viscosity=dynamics.ViscositySpec(2, float(g["nu"])))


def test_settls_steps_match_reference(mods):
    spharm, dynamics, steppers, _ = mods
    g = load_golden("settls_M16.npz")
    grid = spharm.get_grid(int(g["M"]))
    s0 = dynamics.PrognosticState.from_fields(grid, *g["s0"], [float(g["phibar"])])
    cfg = _cfg(steppers, dynamics, g)
    s1 = steppers.settls_step(steppers.StepperState(s0), cfg)
    s2 = steppers.settls_step(steppers.StepperState(s1, s0), cfg)
    s2o = steppers.settls_step(steppers.StepperState(s1, s0), _cfg(steppers, dynamics, g, "one_step"))
    for st, key in ((s1, "s1"), (s2, "s2"), (s2o, "s2_one")):
        d = rel_diff(st.data[0].cpu().numpy(), g[key])
        assert d < 1e-10, (key, d)
        print(f"[PARITY] settls {key}: {d:.2e}")
    # advance() keeps the two-step history like the reference
    st = steppers.advance(steppers.advance(steppers.StepperState(s0), cfg), cfg)
    assert rel_diff(st.current.data[0].cpu().numpy(), g["s2"]) < 1e-10
    assert st.previous is not None


def test_semilag_pieces_match_reference(mods):
    spharm, _, _, semilag = mods
    g = load_golden("settls_M16.npz")
    grid = spharm.get_grid(int(g["M"]))
    lam, th = semilag.departure_points(grid, g["u"], g["v"], 1.1 * g["u"], 0.9 * g["v"],
                                       float(g["dep_dt"]))
    assert np.abs(lam - g["lam"]).max() < 1e-12 and np.abs(th - g["th"]).max() < 1e-12
    adv = semilag.advect_scalar(grid, g["vals"], g["lam"], g["th"])
    assert np.abs(adv - g["adv"]).max() < 1e-12 * np.abs(g["adv"]).max()
    bad = np.full_like(g["u"], np.nan)
    with pytest.raises(semilag.DeparturePointError, match="diverged"):
        semilag.departure_points(grid, bad, g["v"], bad, g["v"], 600.0)


def test_settls_batched_equals_single(mods):
    """Slices of a batch (each with its own history) step independently, bitwise."""
    import torch
    spharm, dynamics, steppers, _ = mods
    g = load_golden("settls_M16.npz")
    grid = spharm.get_grid(int(g["M"]))
    rng = np.random.default_rng(3)
    base = g["s0"]
    states, prevs = [], []
    for b in range(3):
        taper = (grid.n_of + 1.0) ** -2
        noise = (rng.standard_normal(grid.n_modes) + 1j * rng.standard_normal(grid.n_modes)) * taper
        noise[: grid.M + 1] = noise[: grid.M + 1].real
        s = base.copy()
        s[1] = s[1] + 1e-6 * noise
        states.append(s)
        prevs.append(base)
    pb = [float(g["phibar"])] * 3
    cfg = _cfg(steppers, dynamics, g)
    batch = dynamics.PrognosticState.from_fields(grid, *np.stack(states, 1), pb)
    prev = dynamics.PrognosticState.from_fields(grid, *np.stack(prevs, 1), pb)
    from paper_2306_09497_b200 import _lib
    _lib.set_option("gemv_max_b", 0)  # one Legendre kernel generation for B = 1 and 3
    try:
        out = steppers.settls_step(steppers.StepperState(batch, prev), cfg).data.cpu()
        for b in range(3):
            one = dynamics.PrognosticState.from_fields(grid, *states[b], pb[:1])
            po = dynamics.PrognosticState.from_fields(grid, *prevs[b], pb[:1])
            r = steppers.settls_step(steppers.StepperState(one, po), cfg).data.cpu()
            assert torch.equal(r[0], out[b]), b
    finally:
        _lib.set_option("gemv_max_b", 3)
