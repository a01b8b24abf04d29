"""Where the time of a cfg2 MGRIT iteration goes (host wall with device syncs)."""
import os, sys, time, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_09497_b200 import dynamics, pint, scenarios, steppers
lv = [pint.LevelSpec(0, 256, steppers.StepperConfig(dt=60.0, viscosity=dynamics.ViscositySpec(2, 1e5))),
      pint.LevelSpec(1, 51, steppers.StepperConfig(dt=120.0, viscosity=dynamics.ViscositySpec(2, 1e5)))]
pc = pint.PintConfig(levels=tuple(lv), T=7680.0, N0=128, cfactor=2, nrelax=1, max_iters=3)
prob = pint.SweProblem(pc)
u0 = prob.as_batch(0, scenarios.gaussian_bumps(prob.grids[0]))
eng = pint.MgritEngine(prob, pc)
acc = collections.defaultdict(float)
def wrap(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize(); acc[name] += time.perf_counter() - t
        return r
    return w
for name in ("_f_sweep", "_c_sweep", "_residual", "_coarsest_solve", "_fas_restrict"):
    setattr(eng, name, wrap(name, getattr(eng, name)))
eng.run(u0, sync=torch.cuda.synchronize)
acc.clear()
t = time.perf_counter()
tr = eng.run(u0, sync=torch.cuda.synchronize)
tot = sum(tr.wall_times[1:])
print("per iteration ms:", 1e3 * tot / 3)
for k, v in sorted(acc.items(), key=lambda x: -x[1]):
    print(f"  {k:18s} {1e3 * v / 3:8.2f} ms")
