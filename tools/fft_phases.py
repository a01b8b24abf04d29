"""Per-phase clock cycles of the nonlinear lane FFT pass (thread 0 of each CTA, summed
over CTAs), from a debug build with -DSWE_FFT_PHASES:
    bash tools/altlib.sh phases -DSWE_FFT_PHASES
    SWE_LIB=paper_2306_09497_b200/_build/phases/libswe_b200.so python tools/fft_phases.py"""
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
lib.swe_debug_fft_phases(None, 1)
steppers.imex_steps_inplace(st, cfg, 2)
torch.cuda.synchronize()
out = (ctypes.c_ulonglong * 16)()
lib.swe_debug_fft_phases(out, 0)
names = {0: "load E/O + put_z", 2: "inverse stage 1 (7)", 3: "inverse stage 2 (11)", 1: "inverse stage 0 (5)",
         8: "fused middle", 9: "forward stage 0", 10: "forward stage 1 (7)", 11: "forward stage 2 (11)",
         15: "extract + stores"}
tot = sum(out)
for i in range(16):
    if out[i]:
        print(f"{names.get(i, i):24s} {100.0 * out[i] / tot:5.1f}%  {out[i] / 4 / 12352:9.0f} cycles per CTA")
