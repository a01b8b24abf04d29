"""Per-step latency of small (coarse-level) IMEX steps: M, B -> ms/step."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_09497_b200 import dynamics, spharm, steppers, scenarios
for M, B, dt in [(51, 1, 120.0), (51, 64, 120.0), (32, 1, 480.0), (64, 1, 240.0), (256, 1, 60.0)]:
    g = spharm.get_grid(M)
    s = scenarios.gaussian_bumps(g, batch=B)
    cfg = steppers.StepperConfig(dt=dt, viscosity=dynamics.ViscositySpec(2, 1e5))
    for _ in range(5):
        steppers.imex_steps_inplace(s, cfg, 1)
    torch.cuda.synchronize()
    n = 50
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(n):
        steppers.imex_steps_inplace(s, cfg, 1)
    e1.record(); e1.synchronize(); t1 = time.perf_counter()
    e2 = torch.cuda.Event(enable_timing=True); e3 = torch.cuda.Event(enable_timing=True)
    e2.record(); steppers.imex_steps_inplace(s, cfg, n); e3.record(); e3.synchronize()
    print(f"M={M} B={B}: {e0.elapsed_time(e1)/n:.3f} ms/step (1 step per call, wall {1e3*(t1-t0)/n:.3f}), "
          f"{e2.elapsed_time(e3)/n:.3f} ms/step ({n} steps per call)")
