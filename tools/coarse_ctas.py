"""M=51 single-slice step latency vs CTAs per slice of the shared-memory half step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_09497_b200 import _lib, dynamics, spharm, steppers, scenarios
for M, B, dt in [(51, 1, 120.0), (32, 1, 480.0), (51, 8, 120.0)]:
    g = spharm.get_grid(M)
    cfg = steppers.StepperConfig(dt=dt, viscosity=dynamics.ViscositySpec(2, 1e5))
    ref = None
    for C in (0, 2, 4, 8, 16):
        _lib.set_option("cn_cluster_ctas", C)
        s = scenarios.gaussian_bumps(g, batch=B)
        for _ in range(3):
            steppers.imex_steps_inplace(s, cfg, 1)
        torch.cuda.synchronize()
        n = 50
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); steppers.imex_steps_inplace(s, cfg, n); e1.record(); e1.synchronize()
        out = s.data.cpu().numpy()
        d = 0.0 if ref is None else float(np.abs(out - ref).max() / np.abs(ref).max())
        ref = out if ref is None else ref
        print(f"M={M} B={B} ctas={C}: {e0.elapsed_time(e1)/n:.4f} ms/step, diff vs ctas=0 {d:.1e}")
    _lib.set_option("cn_cluster_ctas", 0)
