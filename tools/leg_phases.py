"""Consumer-warp time split of the v3 Legendre GEMMs (full-barrier waits, epilogue,
DMMA main loop) from a debug build with -DSWE_LEG_PHASES:
    bash tools/altlib.sh legph -DSWE_LEG_PHASES
    SWE_LIB=paper_2306_09497_b200/_build/legph/libswe_b200.so python tools/leg_phases.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_09497_b200 import _lib
_lib.load.__defaults__ = (os.path.abspath(os.environ["SWE_LIB"]),)
from paper_2306_09497_b200 import dynamics, spharm, steppers
import bench
for kv in sys.argv[1:]:
    k, v = kv.split("=")
    _lib.set_option(k, int(v))
lib = ctypes.CDLL(os.environ["SWE_LIB"])
grid = spharm.get_grid(256)
cfg = steppers.StepperConfig(dt=60.0, viscosity=dynamics.ViscositySpec(2, 1e5))
st = bench.make_states(grid, 64, 0)
_lib.set_option("graphs", 0)
steppers.imex_steps_inplace(st, cfg, 1)
torch.cuda.synchronize()
lib.swe_debug_leg_phases(None, 1)
steppers.imex_steps_inplace(st, cfg, 2)
torch.cuda.synchronize()
out = (ctypes.c_ulonglong * 8)()
lib.swe_debug_leg_phases(out, 0)
for i, name in enumerate(("synthesis", "analysis")):
    w, e, t, n = out[4 * i:4 * i + 4]
    print(f"{name}: full-barrier waits {100 * w / t:.1f}%, epilogue {100 * e / t:.1f}%, "
          f"rest (DMMA main loop) {100 * (t - w - e) / t:.1f}%; {n / 8:.0f} units per launch-pair x CTA-sum")
