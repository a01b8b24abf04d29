"""Probe the host-pipeline overlap: copy times alone, compute alone, pipelined."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2306_09497_b200 import dynamics, spharm, steppers
import bench
grid = spharm.get_grid(256)
cfg = steppers.StepperConfig(dt=60.0, viscosity=dynamics.ViscositySpec(2, 1e5))
st = bench.make_states(grid, 64, 0)
host = st.data.cpu().pin_memory()
out = torch.empty_like(host).pin_memory()
pb = st.phibar_t.cpu().pin_memory()
dev = st.data
def ev():
    e = torch.cuda.Event(enable_timing=True); e.record(); return e
for name, fn in [("h2d", lambda: dev.copy_(host, non_blocking=True)),
                 ("d2h", lambda: out.copy_(dev, non_blocking=True)),
                 ("step", lambda: steppers.imex_steps_inplace(st, cfg, 1))]:
    fn(); torch.cuda.synchronize()
    a = ev()
    for _ in range(5): fn()
    b = ev(); b.synchronize()
    print(name, a.elapsed_time(b) / 5, "ms")
s2 = torch.cuda.Stream()
a = ev()
with torch.cuda.stream(s2):
    for _ in range(5): dev.copy_(host, non_blocking=True)
for _ in range(5): out.copy_(st.slots if False else dev, non_blocking=True)
torch.cuda.synchronize(); b = ev(); b.synchronize()
print("h2d||d2h x5", a.elapsed_time(b), "ms")
pipe = steppers.HostPipeline(grid, cfg, 64)
for depth in (2, 3):
    pipe = steppers.HostPipeline(grid, cfg, 64, depth=depth)
    for _ in range(3): pipe.submit(host, pb, out)
    pipe.flush()
    t0 = time.perf_counter()
    s = torch.cuda.Event(enable_timing=True); s.record(pipe.h2d)
    for _ in range(20): pipe.submit(host, pb, out)
    e = pipe.flush()
    print("pipeline depth", depth, s.elapsed_time(e) / 20, "ms/step", (time.perf_counter() - t0) * 50, "wall ms/step")
