import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2306_09497_b200 import _lib, dynamics, spharm, steppers, scenarios
M = int(sys.argv[1]) if len(sys.argv) > 1 else 100
grid = spharm.get_grid(M)
cfg = steppers.StepperConfig(dt=240.0, viscosity=dynamics.ViscositySpec(2, 1e5))
base = scenarios.gaussian_bumps(grid, batch=1)
rng = np.random.default_rng(1)
taper = torch.from_numpy((grid.n_of + 1.0) ** -2).cuda()
noise = torch.from_numpy(rng.standard_normal((1, grid.n_modes))).cuda() * taper
noise[:, : M + 1] = noise[:, : M + 1].real
base.data[:, 1] += 1e-6 * noise
base.data[:, 2] += 1e-7 * noise
_lib.set_option("graphs", 0)
if len(sys.argv) > 2: _lib.set_option("cn_small", 0)
out = {}
for cl in (0, 1):
    _lib.set_option("cn_cluster", cl)
    s = base.copy()
    it = np.zeros((1, 1, 2), dtype=np.int32)
    steppers.imex_steps_inplace(s, cfg, 1, it)
    out[cl] = s.data.cpu().numpy()[0]
    print("iters", cl, it.ravel())
K = grid.n_modes
C = -(-K // 2380); chunk = -(-K // C)
print("K", K, "C", C, "chunk", chunk)
for f in range(3):
    d = np.abs(out[1][f] - out[0][f]); sc = np.abs(out[0][f]).max()
    idx = np.argsort(d)[::-1][:8]
    print(f, "maxrel", d.max() / sc, "worst k", idx.tolist(), "bad count", int((d > 1e-13 * sc).sum()))
