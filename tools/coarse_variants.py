"""M=51 coarse-step latency under the half-step variants (cn_small vs cluster kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_09497_b200 import _lib, dynamics, spharm, steppers, scenarios
for opts in ({"cn_small": 1, "cn_cluster": 0}, {"cn_small": 0, "cn_cluster": 1}):
    for k, v in opts.items():
        _lib.set_option(k, v)
    for M, B, dt in [(51, 1, 120.0), (51, 64, 120.0), (32, 1, 480.0)]:
        g = spharm.get_grid(M)
        s = scenarios.gaussian_bumps(g, batch=B)
        cfg = steppers.StepperConfig(dt=dt, viscosity=dynamics.ViscositySpec(2, 1e5))
        for _ in range(5):
            steppers.imex_steps_inplace(s, cfg, 1)
        torch.cuda.synchronize()
        n = 50
        e2 = torch.cuda.Event(enable_timing=True); e3 = torch.cuda.Event(enable_timing=True)
        e2.record(); steppers.imex_steps_inplace(s, cfg, n); e3.record(); e3.synchronize()
        print(opts, f"M={M} B={B}: {e2.elapsed_time(e3)/n:.4f} ms/step ({n} steps per call)")
