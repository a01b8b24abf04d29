"""Class breakdown of an M=1024 IMEX step (cfg5 shape: 64 intervals per GPU)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_09497_b200 import _lib, dynamics, spharm, steppers, scenarios
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
g = spharm.get_grid(1024)
s = scenarios.gaussian_bumps(g, batch=B)
cfg = steppers.StepperConfig(dt=2.0, viscosity=dynamics.ViscositySpec(2, 0.0))
steppers.imex_steps_inplace(s, cfg, 1)
torch.cuda.synchronize()
_lib.profile(True)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); steppers.imex_steps_inplace(s, cfg, 2); e1.record(); e1.synchronize()
_lib.profile(False)
p = _lib.profile_read()
ms = e0.elapsed_time(e1) / 2
out = {"B": B, "ms_per_step": ms, "slice_steps_per_s": B / (ms * 1e-3),
       "class_ms": {k: round(v[0] / 2, 2) for k, v in p.items()},
       "leg_tf": (p["legendre_synthesis"][1] + p["legendre_analysis"][1]) /
                 max(1e-9, (p["legendre_synthesis"][0] + p["legendre_analysis"][0])) / 1e9}
print(json.dumps(out))
