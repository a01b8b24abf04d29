"""Device time per step of the serial coarsest sweep (swe_imex_sweep, M=51, one
slice, graph replay) - the cfg2/cfg3 Amdahl term; run under ncu for the per-kernel
launch list."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_09497_b200 import _lib, dynamics, spharm, steppers, scenarios
M = int(sys.argv[1]) if len(sys.argv) > 1 else 51
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
for kv in (sys.argv[3].split(",") if len(sys.argv) > 3 else []):
    _lib.set_option(kv.split("=")[0], int(kv.split("=")[1]))
g = spharm.get_grid(M)
s = scenarios.gaussian_bumps(g, batch=1)
cfg = steppers.StepperConfig(dt=120.0, viscosity=dynamics.ViscositySpec(2, 1e5))
u = torch.zeros((n + 1, 3, g.n_modes), dtype=torch.complex128, device="cuda")
u[0] = s.data[0]
import ctypes
from paper_2306_09497_b200.spharm import _ptr, _stream
c = cfg.to_c()
pb = s.phibar_t[:1].contiguous()
resid = np.zeros(1)
def sweep():
    _lib.check(g._lib.swe_imex_sweep(g.plan, _ptr(u), None, n, _ptr(pb), ctypes.byref(c),
                                     resid.ctypes.data_as(ctypes.c_void_p), _stream()), "sweep")
for _ in range(2):
    sweep()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    sweep()
e1.record()
e1.synchronize()
print(f"M={M} {sys.argv[3:]} sweep of {n} steps: {e0.elapsed_time(e1) / 5 / n * 1e3:.1f} us per step")
