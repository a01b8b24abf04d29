"""cfg3 (3-level MGRIT, M=256/51/51, cfactor 4, nrelax 2) convergence probe: per
iteration, max|u| over C-points and the relative Phi' error at the last C-point
against the serial fine solution, for a few horizon lengths."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_09497_b200 import dynamics, pint, scenarios, steppers

def run(N0, nrelax=2, iters=6, Ms=(256, 51, 51), dt0=60.0, cf=4, nu=1e5, cycle="F_then_V"):
    lv = [pint.LevelSpec(l, Ml, steppers.StepperConfig(dt=dt0 * cf ** l, viscosity=dynamics.ViscositySpec(2, nu)))
          for l, Ml in enumerate(Ms)]
    pc = pint.PintConfig(levels=tuple(lv), T=N0 * dt0, N0=N0, cfactor=cf, nrelax=nrelax, max_iters=iters, cycle=cycle)
    prob = pint.SweProblem(pc)
    u0 = prob.as_batch(0, scenarios.gaussian_bumps(prob.grids[0]))
    fine = pint.fine_serial_cpoints(prob, pc, u0).tensor
    eng = pint.MgritEngine(prob, pc)
    try:
        tr = eng.run(u0)
        snaps = tr.snapshots
    except pint.PintBlowUpError as e:
        tr = e.trace
        snaps = tr.snapshots
    out = []
    for k, sn in enumerate(snaps):
        x = sn.tensor
        d = (x - fine).clone()
        d[:, 0, 0] = 0
        f = fine.clone(); f[:, 0, 0] = 0
        err = float(d[:, 0].abs().amax() / f[:, 0].abs().amax())
        out.append((k, float(x.abs().amax()), err))
    print(f"N0={N0} nrelax={nrelax} Ms={Ms} cycle={cycle}: blowup={tr.blowup}", flush=True)
    for r in out:
        print("   it %d max|u| %.3e  err(Phi') %.3e" % r, flush=True)

import json
cases = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [dict(N0=1024)]
for args in cases:
    if "Ms" in args:
        args["Ms"] = tuple(args["Ms"])
    t0 = time.time(); run(**args); print("  %.1fs" % (time.time() - t0), flush=True)
