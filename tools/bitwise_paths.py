"""Are the Legendre kernel generations bitwise interchangeable? synthesis/analysis of
the same slices inside batches that select different kernels (M=256)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2306_09497_b200 import _lib, spharm
g = spharm.get_grid(256)
rng = np.random.default_rng(1)
c = (g.n_of + 1.0) ** -1.5 * np.exp(2j * np.pi * rng.uniform(size=(64, g.n_modes)))
c[:, :257] = c[:, :257].real
ct = torch.from_numpy(c).cuda()
full = g.synthesis(ct)          # B=64: v3
res = {}
for B in (1, 2, 7, 40):
    part = g.synthesis(ct[:B])
    res[B] = [bool(torch.equal(part[i], full[i])) for i in range(min(B, 3))]
print("synthesis bitwise vs B=64:", res)
gr = full
af = g.analysis(gr)
res = {}
for B in (1, 2, 7, 40):
    ap = g.analysis(gr[:B])
    res[B] = [bool(torch.equal(ap[i], af[i])) for i in range(min(B, 3))]
print("analysis bitwise vs B=64:", res)
