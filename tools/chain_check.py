"""Persistent serial chain (chain.cu) vs the per-step sweep: bitwise equality and
time per step, for the coarse truncations of the BASELINE configs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_09497_b200 import _lib, dynamics, pint, scenarios, steppers

for M, dt, n in [(51, 120.0, 64), (32, 480.0, 16), (16, 600.0, 8), (51, 960.0, 64)]:
    cfg = steppers.StepperConfig(dt=dt, viscosity=dynamics.ViscositySpec(2, 1e5))
    prob = pint.SweProblem(pint.PintConfig(levels=(pint.LevelSpec(0, M, steppers.StepperConfig(dt=dt / 2)),
                                                   pint.LevelSpec(1, M, cfg)), T=dt, N0=2, cfactor=2))
    g = prob.grids[1]
    s = scenarios.gaussian_bumps(g)
    prob.phibar = float(s.phibar_t[0])
    rng = np.random.default_rng(M)
    taper = (g.n_of + 1.0) ** -2
    f = torch.zeros((n + 1, 3, g.n_modes), dtype=torch.complex128, device="cuda")
    f[:, 0] = torch.from_numpy(rng.standard_normal((n + 1, g.n_modes)) * taper).cuda()
    f[:, 1] = torch.from_numpy(rng.standard_normal((n + 1, g.n_modes)) * 1e-9 * taper).cuda()
    f[:, :, : M + 1] = f[:, :, : M + 1].real
    res = {}
    for chain in (0, 1):
        _lib.set_option("chain", chain)
        for rep in range(3):
            u = prob.zeros(1, n + 1)
            u[0:1] = s.data
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            prob.sweep_batch(1, u, f)
            e1.record()
            e1.synchronize()
        res[chain] = (u.clone(), e0.elapsed_time(e1) / n)
    _lib.set_option("chain", 1)
    a, b = res[0][0], res[1][0]
    d = float(((a - b).abs().amax() / a.abs().amax()))
    print(f"M={M} dt={dt} n={n}: per-step {res[0][1]*1e3:.1f} us/step, chain {res[1][1]*1e3:.1f} us/step, "
          f"bitwise {torch.equal(a, b)} (max rel {d:.2e}), finite {bool(torch.isfinite(b).all())}", flush=True)
