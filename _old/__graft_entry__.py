"""Driver entry points: build() compiles, smoke() runs one tiny GPU step vs the oracle."""

from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def build() -> None:
    """Compile libswe_b200.so for sm_100a (nvcc, -lineinfo) and the oracle's
    reference-backed goldens stay as committed data; then import the package."""
    from paper_2306_09497_b200 import build as b
    lib = b.build()
    print("built", lib)
    import paper_2306_09497_b200  # noqa: F401
    from paper_2306_09497_b200 import _lib
    import ctypes
    handle = ctypes.CDLL(lib)
    for sym in _lib.EXPORTS:
        getattr(handle, sym)


def smoke() -> None:
    """One IMEX step of a 2-slice batch at M=32 on cuda:0, checked against the oracle."""
    import numpy as np
    import torch
    from oracle.sht import OracleSphere
    from oracle.swe import OracleState, StepCfg, gaussian_bumps as o_bumps, imex_step as o_step
    from paper_2306_09497_b200 import _lib, dynamics, spharm, steppers

    assert torch.cuda.is_available(), "smoke() needs cuda:0"
    torch.cuda.set_device(0)
    M = 32
    sph = OracleSphere(M)
    s0 = o_bumps(sph, batch=2)
    s0.xi[1] += 1e-7 * (sph.n_of + 1.0) ** -2
    ref = o_step(s0, StepCfg(dt=240.0, visc_nu=1e5))
    grid = spharm.get_grid(M)
    st = dynamics.PrognosticState.from_fields(grid, s0.phi, s0.xi, s0.delta, s0.phibar)
    n0 = _lib.kernel_launches()
    out = steppers.imex_step(st, steppers.StepperConfig(dt=240.0,
                                                        viscosity=dynamics.ViscositySpec(2, 1e5)))
    torch.cuda.synchronize()
    phi, xi, de, _ = out.to_numpy()
    err = 0.0
    for got, want in ((phi, ref.phi), (xi, ref.xi), (de, ref.delta)):
        err = max(err, float(np.abs(got - want).max() / np.abs(want).max()))
    launches = _lib.kernel_launches() - n0
    print(f"smoke: M={M} B=2 rel err {err:.3e}, {launches} kernel launches")
    assert err < 1e-10, err
    assert launches > 0


if __name__ == "__main__":
    build()
    if len(sys.argv) > 1 and sys.argv[1] == "smoke":
        smoke()
