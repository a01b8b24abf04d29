"""Device time of the nonlinear FFT pass alone (swe_tendency kind 'nonlinear', M=256,
64 slices) under library options given as k=v[,k=v] specs."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_09497_b200 import _lib
if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):  # optional library build to time
    _lib.load.__defaults__ = (os.path.abspath(sys.argv.pop(1)),)
import torch
from paper_2306_09497_b200 import dynamics, spharm
import bench

g = spharm.get_grid(256)
st = bench.make_states(g, 64, 0)
for spec in sys.argv[1:]:
    for kv in spec.split(","):
        k, v = kv.split("=")
        _lib.set_option(k, int(v))
    dynamics.nonlinear(st)
    torch.cuda.synchronize()
    _lib.profile(True)
    for _ in range(10):
        dynamics.nonlinear(st)
    torch.cuda.synchronize()
    _lib.profile(False)
    p = _lib.profile_read()
    print(json.dumps({"opts": spec, **{k: round(v[0] / max(v[2], 1), 4) for k, v in p.items()}}), flush=True)
