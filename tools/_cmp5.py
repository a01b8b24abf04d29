import sys, os
sys.path.insert(0, os.getcwd())
import torch, bench, numpy as np
from paper_2306_09497_b200 import _lib, steppers, pint
orig = steppers.imex_steps_inplace
def wrapped(state, cfg, nsteps=1, iters=None, select_batch=0):
    if iters is None:
        iters = np.zeros((nsteps, state.batch, 2), dtype=np.int32)
    return orig(state, cfg, nsteps, iters, select_batch)
mode = sys.argv[1]
if "wrap" in mode:
    steppers.imex_steps_inplace = wrapped
if "nodefer" in mode:
    pint.SweProblem.supports_deferred_check = False
if "nograph" in mode:
    _lib.set_option("graphs", 0)
r = bench.pint_leg(torch, "cfg2", None, iters=6)
print(mode, round(r["ms_per_iteration"], 2))
