"""Compare kernel paths on the cfg2 fine step (M=256, 64 slices): per-class device time."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_09497_b200 import _lib, dynamics, spharm, steppers
import bench

def run(steps, **opts):
    for k, v in opts.items():
        _lib.set_option(k, v)
    grid = spharm.get_grid(256)
    cfg = steppers.StepperConfig(dt=60.0, viscosity=dynamics.ViscositySpec(2, 1e5))
    st = bench.make_states(grid, 64, 0)
    steppers.imex_steps_inplace(st, cfg, 1)
    torch.cuda.synchronize()
    _lib.profile(True)
    t0 = time.perf_counter()
    steppers.imex_steps_inplace(st, cfg, steps)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    _lib.profile(False)
    p = _lib.profile_read()
    leg = (p["legendre_synthesis"][1] + p["legendre_analysis"][1]) / (p["legendre_synthesis"][0] + p["legendre_analysis"][0]) / 1e9
    out = {k: round(v[0] / steps, 3) for k, v in p.items()}
    print(json.dumps({"opts": opts, "ms_per_step": round(1e3 * el / steps, 3), "class_ms": out,
                      "synth_tf": round(p["legendre_synthesis"][1] / p["legendre_synthesis"][0] / 1e9, 2),
                      "anal_tf": round(p["legendre_analysis"][1] / p["legendre_analysis"][0] / 1e9, 2),
                      "fft_gbs": round(p["fft_grid"][1] / p["fft_grid"][0] / 1e6, 1)}), flush=True)

if __name__ == "__main__":
    for spec in sys.argv[1:]:
        opts = dict(kv.split("=") for kv in spec.split(","))
        run(3, **{k: int(v) for k, v in opts.items()})
