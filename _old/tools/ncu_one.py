"""Minimal driver for ncu: one cfg2 fine step (M=256, 64 slices) after a warm-up step
(steady-state iteration guess); run ncu with --profile-from-start off."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_09497_b200 import _lib, dynamics, spharm, steppers
import bench
for kv in sys.argv[1:]:
    k, v = kv.split("=")
    _lib.set_option(k, int(v))
grid = spharm.get_grid(256)
cfg = steppers.StepperConfig(dt=60.0, viscosity=dynamics.ViscositySpec(2, 1e5))
st = bench.make_states(grid, 64, 0)
steppers.imex_steps_inplace(st, cfg, 1)
torch.cuda.synchronize()
torch.cuda.profiler.start()
steppers.imex_steps_inplace(st, cfg, 1)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
