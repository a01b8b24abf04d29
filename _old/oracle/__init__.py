"""CPU oracle for the fine SWE propagator -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's algorithm for the hot path
(`/root/reference/pkg/src/pintswe/{spharm,dynamics,steppers,pint,diagnostics}.py`),
batched over time slices.  Every function cites the reference file:line it
follows.  It exists to CHECK the CUDA path:

* only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
  `--impl reference` legs may import it;
* the product package `paper_2306_09497_b200` never imports it and has no CPU
  fallback.

Parity pin: `oracle/make_golden.py` imports the reference itself (in the
build container, where `/root/reference` exists) and writes seeded golden
vectors to `tests/golden/`; `tests/test_oracle.py` checks this restatement
against them and against the reference's frozen run outputs
(`pkg/frontend/fixtures/errors.csv`, `spectrum.csv`), which are copied
verbatim as data into `tests/golden/fixtures/`.
"""

from .sht import OracleSphere, grid_shape, gauss_nodes, legendre_tables  # noqa: F401
from .swe import OracleState, StepCfg, imex_step, ImplicitSolveError  # noqa: F401
