"""Minimal driver for ncu: one warm cfg2 fine step (M=256, 64 slices) with the direct solver."""
import sys, os, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_09497_b200 import dynamics, spharm, steppers
import bench
grid = spharm.get_grid(256)
cfg = steppers.StepperConfig(dt=60.0, viscosity=dynamics.ViscositySpec(2, 1e5), implicit_solver="direct")
st = bench.make_states(grid, 64, 0)
steppers.imex_steps_inplace(st, cfg, 1)
torch.cuda.synchronize()
print("ok")
