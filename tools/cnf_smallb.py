"""Small batches at M=256: cluster half step (default below 32 slices) vs k_cn_fused."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_09497_b200 import _lib, dynamics, spharm, steppers
import bench
grid = spharm.get_grid(256)
cfg = steppers.StepperConfig(dt=60.0, viscosity=dynamics.ViscositySpec(2, 1e5))
for B in (1, 2, 4, 8, 16, 24):
    res = {}
    for name, cl in (("cluster", 1), ("fused", 0)):
        _lib.set_option("cn_cluster", cl)
        st = bench.make_states(grid, B, 0)
        steppers.imex_steps_inplace(st, cfg, 3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            steppers.imex_steps_inplace(st, cfg, 1)
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / 20
    print(f"B={B}: " + ", ".join(f"{k} {v:.3f} ms" for k, v in res.items()), flush=True)
_lib.set_option("cn_cluster", 1)
