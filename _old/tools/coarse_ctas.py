"""Single-slice coarse step time vs CTAs per slice of the cluster CN half step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_09497_b200 import _lib, dynamics, scenarios, spharm, steppers
for M, dt in [(51, 120.0), (32, 480.0), (51, 960.0)]:
    g = spharm.get_grid(M)
    cfg = steppers.StepperConfig(dt=dt, viscosity=dynamics.ViscositySpec(2, 1e5))
    res = []
    for c in (0, 1, 2, 4, 8, 16):
        _lib.set_option("cn_cluster_ctas", c)
        s = scenarios.gaussian_bumps(g)
        for _ in range(3):
            steppers.imex_steps_inplace(s, cfg, 1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        steppers.imex_steps_inplace(s, cfg, 50)
        e1.record()
        e1.synchronize()
        res.append(f"{c}:{e0.elapsed_time(e1) / 50 * 1e3:.1f}")
    _lib.set_option("cn_cluster_ctas", 0)
    print(f"M={M} dt={dt}: us/step by CTAs per slice (0 = auto) " + " ".join(res), flush=True)
