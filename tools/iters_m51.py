import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2306_09497_b200 import _lib, dynamics, spharm, steppers, scenarios
g = spharm.get_grid(51)
s = scenarios.gaussian_bumps(g, batch=1)
cfg = steppers.StepperConfig(dt=120.0, viscosity=dynamics.ViscositySpec(2, 1e5))
it = np.zeros((10, 1, 2), dtype=np.int32)
steppers.imex_steps_inplace(s, cfg, 10, it)
print(it[:, 0, :].tolist())
