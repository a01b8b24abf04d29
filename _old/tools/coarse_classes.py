"""Warm per-class device time of one M=51 single-slice IMEX step (eager launches with
CUDA events per launch, swe_profile) next to the graph-replayed step time."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_09497_b200 import _lib, dynamics, spharm, steppers, scenarios
M = int(sys.argv[1]) if len(sys.argv) > 1 else 51
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = spharm.get_grid(M)
s = scenarios.gaussian_bumps(g, batch=B)
cfg = steppers.StepperConfig(dt=120.0, viscosity=dynamics.ViscositySpec(2, 1e5))
for _ in range(3):
    steppers.imex_steps_inplace(s, cfg, 1)
torch.cuda.synchronize()
n = 20
_lib.profile(True)
for _ in range(n):
    steppers.imex_steps_inplace(s, cfg, 1)
torch.cuda.synchronize()
_lib.profile(False)
p = _lib.profile_read()
print(json.dumps({k: {"us_per_step": round(1e3 * v[0] / n, 2), "launches_per_step": v[2] / n}
                  for k, v in p.items()}))
