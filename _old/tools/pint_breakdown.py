"""Where a cfg2 MGRIT iteration spends its time: CUDA-event totals of the problem's
batched steps per level, the coarsest device sweep and the rest (engine arithmetic,
restriction/prolongation, snapshots, blow-up check)."""
import collections, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2306_09497_b200 import pint

acc = collections.defaultdict(float)
cnt = collections.Counter()
orig_step, orig_sweep = pint.SweProblem.step_batch, pint.SweProblem.sweep_batch


def timed(name, fn):
    def wrap(self, level, *a, **k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn(self, level, *a, **k)
        e1.record()
        e1.synchronize()
        key = f"{name}[L{level}, B={a[0].shape[0]}]" if name == "step" else f"{name}[L{level}]"
        acc[key] += e0.elapsed_time(e1)
        cnt[key] += 1
        return out
    return wrap


name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
pint.SweProblem.step_batch = timed("step", orig_step)
pint.SweProblem.sweep_batch = timed("sweep", orig_sweep)
rec = bench.pint_leg(torch, name, None, iters=3)
tot = rec["ms_per_iteration"] * 3 * 2  # warm-up run + timed run, 3 iterations each
print(f"{name}: {rec['ms_per_iteration']:.2f} ms per iteration (timed run)")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k}: {v / 6:.2f} ms per iteration over {cnt[k] / 6:.1f} calls")
