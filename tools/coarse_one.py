"""One eager M=51 B=1 IMEX step (coarse level of cfg2) for an ncu launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_09497_b200 import _lib, dynamics, spharm, steppers, scenarios
_lib.set_option("graphs", 0)
g = spharm.get_grid(51)
s = scenarios.gaussian_bumps(g, batch=1)
cfg = steppers.StepperConfig(dt=120.0, viscosity=dynamics.ViscositySpec(2, 1e5))
steppers.imex_steps_inplace(s, cfg, 1)
torch.cuda.synchronize()
print("ok")
