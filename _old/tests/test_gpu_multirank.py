"""Rank-count determinism of the sharded MGRIT engine on the SWE problem.

The reference promises worker-count-independent results (SPEC.md:330,
tests/test_pint.py:162-167, :322-332).  Here the workers are ranks holding
contiguous slice blocks; their sweeps are batches of n/G slices stepped with the
kernels chosen for the global count n (`select_batch`).  These tests check:

* a slice stepped inside any sub-batch with select_batch = n is bitwise equal to
  the same slice inside the full batch of n, at the coarse and fine truncations
  and on every kernel generation the batch size would otherwise pick;
* the real SweProblem engine at world size 2 (two processes sharing this GPU,
  gloo with host-staged buffers -- no kernel of one rank waits on the other)
  reproduces the one-rank trace bitwise, and the reference's trace to 1e-10.
"""

import os
import socket

import numpy as np
import pytest

from conftest import load_golden, rel_diff

pytestmark = pytest.mark.gpu


def _perturbed(grid, B, seed, scale=1e-6):
    import torch
    from paper_2306_09497_b200 import scenarios
    base = scenarios.gaussian_bumps(grid, batch=B)
    rng = np.random.default_rng(seed)
    taper = torch.from_numpy((grid.n_of + 1.0) ** -2).cuda()
    noise = torch.from_numpy(rng.standard_normal((B, grid.n_modes))).cuda() * taper
    noise[:, : grid.M + 1] = noise[:, : grid.M + 1].real
    base.data[:, 1] += scale * noise
    base.data[:, 2] += 0.1 * scale * noise
    return base


@pytest.mark.parametrize("M,dt,n", [(32, 480.0, 16), (51, 120.0, 64), (64, 240.0, 16),
                                    (256, 60.0, 64)])
def test_select_batch_makes_slices_bitwise_batch_invariant(M, dt, n):
    import torch
    from paper_2306_09497_b200 import dynamics, spharm, steppers
    grid = spharm.get_grid(M)
    cfg = steppers.StepperConfig(dt=dt, viscosity=dynamics.ViscositySpec(2, 1e5))
    base = _perturbed(grid, n, M)
    full = base.copy()
    steppers.imex_steps_inplace(full, cfg, 2)
    ref = full.data.clone()
    for B in sorted({1, 2, 3, 4, 8, n // 8, n // 4, n // 2}):
        for lo in (0, n - B):
            part = dynamics.PrognosticState(grid, base.data[lo:lo + B].clone(),
                                            base.phibar_t[lo:lo + B].clone())
            steppers.imex_steps_inplace(part, cfg, 2, select_batch=n)
            assert torch.equal(part.data, ref[lo:lo + B]), (M, B, lo)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, name, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch
    import torch.distributed as dist
    from test_gpu_pint import setup_from_golden
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = load_golden(name)
        pint, prob, pc, u0 = setup_from_golden(g)
        tr = pint.mgrit_run(prob, pc, u0, comm=pint.Comm())
        out[rank] = np.stack([s.tensor.cpu().numpy() for s in tr.snapshots])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["pint_cfg1_M64.npz", "pint_mgrit2_M32.npz"])
def test_two_ranks_on_one_gpu_bitwise_equal_one_rank(name):
    import multiprocessing as mp
    from test_gpu_pint import check_trace, setup_from_golden
    g = load_golden(name)
    pint, prob, pc, u0 = setup_from_golden(g)
    single = pint.mgrit_run(prob, pc, u0)
    ref = np.stack([s.tensor.cpu().numpy() for s in single.snapshots])
    check_trace(g, ref)
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, name, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    for r in range(2):
        assert np.array_equal(out[r], ref), (name, r)
    print(f"[MULTIRANK] {name}: world 2 trace bitwise equal to world 1 "
          f"({ref.shape[0]} snapshots x {ref.shape[1]} C-points)")
