"""Fine-step time at the per-rank batch of a sharded cfg2 (64 global slices over G ranks):
batch 64/G with select_batch 64 (the kernels a rank runs), M=256, dt=60, nu=1e5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_09497_b200 import _lib, dynamics, scenarios, spharm, steppers
import bench
g = spharm.get_grid(256)
cfg = steppers.StepperConfig(dt=60.0, viscosity=dynamics.ViscositySpec(2, 1e5))
out = []
for B in (64, 32, 16, 8):
    s = bench.make_states(g, B, 0)
    for _ in range(3):
        steppers.imex_steps_inplace(s, cfg, 1, select_batch=64)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        steppers.imex_steps_inplace(s, cfg, 1, select_batch=64)
    e1.record()
    e1.synchronize()
    out.append(f"B={B}: {e0.elapsed_time(e1) / 10:.3f} ms")
print("per-rank fine step, select_batch 64: " + ", ".join(out))

# per-class device time at 8 slices (the per-rank batch at 8 GPUs)
s = bench.make_states(g, 8, 0)
steppers.imex_steps_inplace(s, cfg, 1, select_batch=64)
_lib.profile(True)
for _ in range(5):
    steppers.imex_steps_inplace(s, cfg, 1, select_batch=64)
torch.cuda.synchronize()
_lib.profile(False)
p = _lib.profile_read()
print("B=8 classes (ms/step): " + ", ".join(f"{k} {v[0] / 5:.3f} ({v[2] // 5} launches)" for k, v in p.items()))
