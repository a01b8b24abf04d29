"""On-device diagnostics and the run-pint outputs vs the reference's frozen
fixtures (pkg/frontend/fixtures errors.csv / spectrum.csv, manifest.json config)."""

import csv
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _read(path):
    with open(path) as fh:
        rows = list(csv.reader(fh))
    return rows[0], rows[1:]


def test_diagnostics_match_oracle():
    import torch
    from paper_2306_09497_b200 import diagnostics, dynamics, spharm
    from oracle import mgrit as om
    from oracle.sht import OracleSphere, random_bandlimited
    from oracle.swe import OracleState
    rng = np.random.default_rng(12)
    for M, Mt in ((16, 16), (24, 16), (16, 32)):
        g, gt = spharm.get_grid(M), spharm.get_grid(Mt)
        so, sto = OracleSphere(M), OracleSphere(Mt)
        c = [random_bandlimited(so, rng, batch=(1,)) for _ in range(3)]
        ct = [random_bandlimited(sto, rng, batch=(1,)) for _ in range(3)]
        s = dynamics.PrognosticState.from_fields(g, *c, [3e5])
        t = dynamics.PrognosticState.from_fields(gt, *ct, [3e5])
        os_ = OracleState(so, *c, np.array([3e5]))
        ot = OracleState(sto, *ct, np.array([3e5]))
        got = diagnostics.phi_error_records(3, s, "fine", t, [4, 8], include_l2=True)
        want = om.phi_error_records(3, os_, "fine", ot, [4, 8], include_l2=True)
        for a, b in zip(got, want):
            assert a.row()[:3] == tuple(b[:3])
            assert abs(a.value - b[3]) <= 1e-12 * abs(b[3])
        n, wl, en = om.ke_spectrum(os_)
        rec = diagnostics.ke_spectrum(s)
        assert np.array_equal(rec.n, n) and np.allclose(rec.wavelength, wl, rtol=1e-15, atol=0)
        assert np.abs(rec.energy - en).max() <= 1e-13 * np.abs(en).max()
    with pytest.raises(ValueError):
        diagnostics.spectral_error(c[0][0], g, c[0][0], g, g.M + 1)
    z = torch.zeros(g.n_modes, dtype=torch.complex128)
    with pytest.raises(ZeroDivisionError):
        diagnostics.spectral_error(c[0][0], g, z, g, 4)


def test_run_pint_outputs_match_frozen_fixtures(tmp_path):
    """The fixture run (gaussian_bumps, M=16, dt=600, Parareal, 4 iterations) on the
    GPU path reproduces errors.csv / spectrum.csv: the spectrum to 1e-10 relative,
    the errors (differences of nearly equal iterates, ~1e-7 and below) to 1e-6."""
    from paper_2306_09497_b200 import runner
    man = json.load(open(os.path.join(GOLDEN, "fixtures", "manifest.json")))
    code = runner.cmd_run_pint(man["config"], str(tmp_path))
    assert code == runner.EXIT_OK
    hdr, rows = _read(tmp_path / "errors.csv")
    rhdr, ref = _read(os.path.join(GOLDEN, "fixtures", "errors.csv"))
    assert hdr == rhdr and len(rows) == len(ref)
    for got, want in zip(rows, ref):
        assert got[:3] == want[:3]
        w = float(want[3])
        assert abs(float(got[3]) - w) <= max(1e-6 * w, 1e-12), (got, want)
    hdr, rows = _read(tmp_path / "spectrum.csv")
    rhdr, ref = _read(os.path.join(GOLDEN, "fixtures", "spectrum.csv"))
    assert hdr == rhdr and len(rows) == len(ref)
    for got, want in zip(rows, ref):
        assert got[:3] == want[:3]
        assert abs(float(got[3]) - float(want[3])) <= 1e-15 * float(want[3])
        assert abs(float(got[4]) - float(want[4])) <= 1e-10 * float(want[4]) + 1e-30
    m = json.load(open(tmp_path / "manifest.json"))
    assert m["engine"] == "parareal" and m["iterations_completed"] == 4 and m["status"] == "ok"
    assert os.path.exists(tmp_path / "speedup.csv")
