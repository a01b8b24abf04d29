"""M=1024 sanity: plan, SHT round trip (cfg4 shape) and IMEX steps (cfg5 shape)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_09497_b200 import dynamics, spharm, steppers, scenarios
t = time.perf_counter()
g = spharm.get_grid(1024)
torch.cuda.synchronize()
print("plan M=1024", g.nlat, g.nlon, g.n_modes, f"{time.perf_counter() - t:.1f}s", f"{g.device_bytes() / 1e9:.2f} GB")
rng = np.random.default_rng(230609497)
B = 24
c = (g.n_of + 1.0) ** -1.5 * np.exp(2j * np.pi * rng.uniform(size=(B, g.n_modes)))
c[:, : g.M + 1] = c[:, : g.M + 1].real
ct = torch.from_numpy(c).cuda()
for _ in range(2):
    gr = g.synthesis(ct); back = g.analysis(gr)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); gr = g.synthesis(ct); back = g.analysis(gr); e1.record(); e1.synchronize()
err = float((back - ct).abs().max() / ct.abs().max())
print(f"round trip B={B}: rel err {err:.2e}, {e0.elapsed_time(e1):.1f} ms "
      f"({B / (e0.elapsed_time(e1) * 1e-3):.0f} field-slices/s)")
s = scenarios.gaussian_bumps(g, batch=16)
cfg = steppers.StepperConfig(dt=2.0, viscosity=dynamics.ViscositySpec(2, 0.0))
steppers.imex_steps_inplace(s, cfg, 2)
torch.cuda.synchronize()
e0.record(); steppers.imex_steps_inplace(s, cfg, 3); e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"IMEX M=1024 B=16 dt=2: {ms:.1f} ms/step = {16 / (ms * 1e-3):.0f} slice-steps/s, finite={s.is_finite()}")
