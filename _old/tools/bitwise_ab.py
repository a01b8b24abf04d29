"""Bitwise A/B of the step results between two builds of libswe_b200.so:
    python tools/bitwise_ab.py <lib.so> <out.npz>   (one process per library)
    python tools/bitwise_ab.py --cmp a.npz b.npz"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in a.files:
        eq = np.array_equal(a[k], b[k])
        d = np.abs(a[k] - b[k]).max() / max(np.abs(a[k]).max(), 1e-300)
        print(f"{k}: {'bitwise' if eq else 'DIFF %.2e' % d}")
    sys.exit(0)
from paper_2306_09497_b200 import _lib
_lib.load.__defaults__ = (os.path.abspath(sys.argv[1]),)
import torch
from paper_2306_09497_b200 import dynamics, scenarios, spharm, steppers, pint
out = {}
for M, B, dt, n in [(51, 1, 120.0, 3), (32, 2, 480.0, 3), (51, 64, 120.0, 2), (256, 64, 60.0, 2), (256, 1, 60.0, 1), (64, 16, 240.0, 2)]:
    g = spharm.get_grid(M)
    s = scenarios.gaussian_bumps(g, batch=B)
    rng = np.random.default_rng(M * 7 + B)
    taper = torch.from_numpy((g.n_of + 1.0) ** -2).cuda()
    noise = torch.from_numpy(rng.standard_normal((B, g.n_modes))).cuda() * taper
    noise[:, : M + 1] = noise[:, : M + 1].real
    s.data[:, 1] += 1e-6 * noise
    s.data[:, 2] += 1e-7 * noise
    cfg = steppers.StepperConfig(dt=dt, viscosity=dynamics.ViscositySpec(2, 1e5))
    for graphs in (0, 1):
        _lib.set_option("graphs", graphs)
        x = s.copy()
        steppers.imex_steps_inplace(x, cfg, n)
        out[f"M{M}_B{B}_g{graphs}"] = x.data[:8].cpu().numpy()
    _lib.set_option("graphs", 1)
    # serial sweep (device chain) with forcing
    if B == 1:
        prob = pint.SweProblem(pint.PintConfig(levels=(pint.LevelSpec(0, M, cfg), pint.LevelSpec(1, M, steppers.StepperConfig(dt=2 * dt, viscosity=dynamics.ViscositySpec(2, 1e5)))), T=4 * dt, N0=4, cfactor=2))
        prob.phibar = float(s.phibar_t[0])
        u = prob.zeros(0, 6)
        u[0:1] = s.data
        f = torch.zeros_like(u)
        f[:, 2] = 1e-8 * noise[0]
        prob.sweep_batch(0, u, f)
        out[f"sweep_M{M}"] = u.cpu().numpy()
np.savez(sys.argv[2], **out)
print("saved", sys.argv[2])
