"""Step latency vs batch with / without the dot-product Legendre kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_09497_b200 import _lib, dynamics, spharm, steppers, scenarios
for M, dt in [(51, 120.0), (256, 60.0)]:
    g = spharm.get_grid(M)
    cfg = steppers.StepperConfig(dt=dt, viscosity=dynamics.ViscositySpec(2, 1e5))
    for B in (1, 2, 3, 4):
        row = []
        for mb in (0, 4):
            _lib.set_option("gemv_max_b", mb)
            s = scenarios.gaussian_bumps(g, batch=B)
            for _ in range(3):
                steppers.imex_steps_inplace(s, cfg, 1)
            torch.cuda.synchronize()
            n = 20
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); steppers.imex_steps_inplace(s, cfg, n); e1.record(); e1.synchronize()
            row.append(e0.elapsed_time(e1) / n)
        print(f"M={M} B={B}: tiles {row[0]:.4f} ms, gemv {row[1]:.4f} ms")
    _lib.set_option("gemv_max_b", 3)
