"""Pin the CPU oracle against the reference's own outputs (CPU only).

The golden .npz files were produced by `oracle/make_golden.py` from the
reference `pintswe` package; `golden/fixtures/*.csv` are the reference's frozen
`run-pint` outputs (pkg/frontend/fixtures, config in manifest.json).
"""

import csv
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, rel_diff
from oracle import mgrit as om
from oracle.sht import OracleSphere, gauss_nodes, grid_shape, random_bandlimited
from oracle.swe import (OracleState, StepCfg, full_rhs, imex_step, linear_coriolis,
                        linear_gravity, nonlinear_advection, nonlinear_rest,
                        gaussian_bumps)

_SPH = {}


def sphere(M):
    if M not in _SPH:
        _SPH[M] = OracleSphere(M)
    return _SPH[M]


def state_from(sph, arr, phibar):
    return OracleState(sph, arr[0][None].copy(), arr[1][None].copy(), arr[2][None].copy(),
                       np.array([float(phibar)]))


@pytest.mark.parametrize("M,shape", [(16, (25, 50)), (32, (49, 98)), (51, (77, 154)),
                                     (64, (97, 194)), (256, (385, 770)), (1024, (1537, 3074))])
def test_grid_shape(M, shape):
    assert grid_shape(M) == shape


@pytest.mark.parametrize("n", [1, 2, 7, 49, 97])
def test_nodes_match_leggauss(n):
    x, w = gauss_nodes(n)
    xr, wr = np.polynomial.legendre.leggauss(n)
    assert np.abs(np.sort(x) - xr).max() < 1e-14
    assert np.abs(w[np.argsort(x)] - wr).max() < 1e-13


@pytest.mark.parametrize("name", ["sht_M16.npz", "sht_M32.npz"])
def test_sht_matches_reference(name):
    g = load_golden(name)
    sph = sphere(int(g["M"]))
    assert np.abs(sph.mu - g["mu"]).max() == 0.0
    assert np.abs(sph.weights - g["weights"]).max() == 0.0
    c, gi = g["coeffs"], g["grid_in"]
    assert rel_diff(sph.synthesis(c), g["synthesis"]) < 1e-13
    assert rel_diff(sph.analysis(gi), g["analysis"]) < 1e-13
    assert rel_diff(sph.synthesis_pair(c[:1], c[1:2]), g["pair"]) < 1e-13
    u, v = sph.uv_from_vortdiv(c[0], c[1])
    assert rel_diff(u, g["u"]) < 1e-13 and rel_diff(v, g["v"]) < 1e-13
    xi, de = sph.vortdiv_from_uv(gi[0], gi[1])
    assert rel_diff(xi, g["vd_xi"]) < 1e-13 and rel_diff(de, g["vd_delta"]) < 1e-13
    gx, gy = sph.grad_grid(c[2])
    assert rel_diff(gx, g["gx"]) < 1e-13 and rel_diff(gy, g["gy"]) < 1e-13


def test_round_trip_and_batching():
    sph = sphere(32)
    rng = np.random.default_rng(3)
    c = random_bandlimited(sph, rng, batch=(2, 3))
    back = sph.analysis(sph.synthesis(c))
    assert back.shape == c.shape
    assert np.abs(back - c).max() <= 1e-12 * np.abs(c).max()


def test_tendencies_match_reference():
    g = load_golden("tend_M24.npz")
    sph = sphere(int(g["M"]))
    s = state_from(sph, g["state"], g["phibar"])
    for name, fn in (("linear_gravity", linear_gravity), ("linear_coriolis", linear_coriolis),
                     ("nonlinear_advection", nonlinear_advection),
                     ("nonlinear_rest", nonlinear_rest), ("full_rhs", full_rhs)):
        t = np.stack([x[0] for x in fn(s)])
        ref = g[name]
        scale = max(np.abs(ref).max(), 1e-300)
        assert np.abs(t - ref).max() <= 1e-12 * scale, name


@pytest.mark.parametrize("name", ["step_M16.npz", "step_M32.npz"])
def test_imex_steps_match_reference(name):
    g = load_golden(name)
    sph = sphere(int(g["M"]))
    keys = sorted(k[:-4] for k in g if k.endswith("_cfg"))
    assert keys
    for key in keys:
        dt, q, nu, implicit, n = g[key + "_cfg"]
        cfg = StepCfg(dt=float(dt), visc_order=int(q), visc_nu=float(nu),
                      coriolis_treatment="implicit" if implicit else "explicit")
        s = state_from(sph, g[key + "_in"], g["phibar"])
        for _ in range(int(n)):
            s = imex_step(s, cfg)
        out = np.stack([s.phi[0], s.xi[0], s.delta[0]])
        assert rel_diff(out, g[key + "_out"]) < 1e-11, key


def test_batched_step_equals_single():
    g = load_golden("step_M16.npz")
    sph = sphere(16)
    a = state_from(sph, g["bumps_dt600_nu1e5_in"], g["phibar"])
    b = state_from(sph, g["random_dt120_q4_in"], g["phibar"])
    cfg = StepCfg(dt=600.0, visc_nu=1e5)
    both = imex_step(OracleState.stack([a, b]), cfg)
    sa, sb = imex_step(a, cfg), imex_step(b, cfg)
    # BLAS blocking differs with the column count: equal to roundoff, not bitwise
    assert rel_diff(both.phi[0], sa.phi[0]) < 1e-13
    assert rel_diff(both.xi[1], sb.xi[0]) < 1e-13


@pytest.mark.slow
def test_m256_step_window_matches_reference():
    g = load_golden("step_window_M256.npz")
    sph = sphere(256)
    s = gaussian_bumps(sph)
    s1 = imex_step(s, StepCfg(dt=float(g["dt"]), visc_nu=float(g["nu"])))
    out = np.stack([s1.phi[0], s1.xi[0], s1.delta[0]])[:, g["sel"]]
    ref = g["out_window"]
    for f in range(3):
        assert np.abs(out[f] - ref[f]).max() <= 1e-11 * g["out_maxabs"][f]


def _run_pint(g):
    fine, coarse = int(g["fineM"]), int(g["coarseM"])
    dt0, nl, cf = float(g["dt0"]), int(g["nlevels"]), int(g["cfactor"])
    scheme = str(g["coarse_scheme"]) if "coarse_scheme" in g else "imex"
    levels = [om.Level(fine, StepCfg(dt=dt0, visc_nu=float(g["nu_f"])))]
    for l in range(1, nl):
        levels.append(om.Level(coarse, StepCfg(dt=dt0 * cf ** l, visc_nu=float(g["nu_c"]),
                                               scheme=scheme)))
    pc = om.PintCfg(levels=tuple(levels), T=float(g["T"]), N0=int(round(float(g["T"]) / dt0)),
                    cfactor=cf, nrelax=int(g["nrelax"]), max_iters=int(g["iters"]),
                    cycle=str(g["cycle"]),
                    chunk_size=int(g["chunk_size"]) if "chunk_size" in g else 0)
    prob = om.OracleProblem(pc, {fine: sphere(fine), coarse: sphere(coarse)})
    u0 = state_from(prob.spheres[0], g["u0"], g["phibar"])
    return prob, pc, u0


@pytest.mark.parametrize("name", ["pint_fixture_M16.npz", "pint_mgrit3_M24.npz",
                                  "pint_mgrit2_M32.npz", "pint_settls_M24.npz",
                                  "pint_settls_chunk_M24.npz"])
def test_pint_trace_matches_reference(name):
    g = load_golden(name)
    prob, pc, u0 = _run_pint(g)
    fine = om.fine_serial_cpoints(prob, pc, u0)
    for i, st in enumerate(fine):
        assert rel_diff(np.stack([st.phi[0], st.xi[0], st.delta[0]]), g["fine"][i]) < 1e-11
    tr = om.OracleMgrit(prob, pc).run(u0)
    snaps = g["snapshots"]
    assert len(tr.snapshots) == snaps.shape[0]
    for k, snap in enumerate(tr.snapshots):
        for i, st in enumerate(snap):
            got = np.stack([st.phi[0], st.xi[0], st.delta[0]])
            assert rel_diff(got, snaps[k, i]) < 1e-10, (k, i)


@pytest.mark.slow
def test_pint_cfg1_trace_matches_reference():
    """BASELINE cfg1 (bumps-pint-desk, M=64/32, Parareal, N0 32, 5 iterations): the
    oracle engine against the reference's compact golden (every C-point on n <= 32,
    max|.| per field, full states at the middle and last C-point)."""
    g = load_golden("pint_cfg1_M64.npz")
    prob, pc, u0 = _run_pint(g)
    tr = om.OracleMgrit(prob, pc).run(u0)
    sel, win, mx = g["sel"], g["snap_window"], g["snap_maxabs"]
    assert len(tr.snapshots) == win.shape[0]
    full = {int(i): j for j, i in enumerate(g["snap_full_idx"])}
    for k, snap in enumerate(tr.snapshots):
        for i, st in enumerate(snap):
            got = np.stack([st.phi[0], st.xi[0], st.delta[0]])
            assert (np.abs(np.abs(got).max(axis=-1) - mx[k, i]) <= 1e-10 * mx[k, i]).all()
            assert (np.abs(got[:, sel] - win[k, i]).max(axis=-1) <= 1e-10 * mx[k, i]).all()
            if i in full:
                assert rel_diff(got, g["snap_full"][k, full[i]]) < 1e-10, (k, i)


def _read_csv(path):
    with open(path) as fh:
        rows = list(csv.reader(fh))
    return rows[0], rows[1:]


def test_frozen_fixture_csvs_regenerate():
    """errors.csv / spectrum.csv of pkg/frontend/fixtures (manifest.json config)."""
    g = load_golden("pint_fixture_M16.npz")
    prob, pc, u0 = _run_pint(g)
    fine = om.fine_serial_cpoints(prob, pc, u0)
    tr = om.OracleMgrit(prob, pc).run(u0)
    rows = []
    for k, snap in enumerate(tr.snapshots):
        rows += om.phi_error_records(k, snap[-1], "fine", fine[-1], [4, 8], include_l2=True)
    _, ref_rows = _read_csv(os.path.join(GOLDEN, "fixtures", "errors.csv"))
    assert len(rows) == len(ref_rows)
    for got, ref in zip(rows, ref_rows):
        assert (str(got[0]), got[1], got[2]) == (ref[0], ref[1], ref[2])
        want = float(ref[3])
        assert abs(got[3] - want) <= max(1e-6 * want, 1e-12), (got, ref)
    _, spec_rows = _read_csv(os.path.join(GOLDEN, "fixtures", "spectrum.csv"))
    series = {("fine", ""): fine[-1]}
    for k in (0, 2, 4):
        series[("pint", str(k))] = tr.snapshots[k][-1]
    for ser, it, n, wl, en in spec_rows:
        nn, wav, ener = om.ke_spectrum(series[(ser, it)])
        i = int(n) - 1
        assert abs(wav[i] - float(wl)) <= 1e-15 * float(wl)
        assert abs(ener[i] - float(en)) <= 1e-10 * float(en) + 1e-30


def test_settls_matches_reference():
    """SL-SI-SETTLS step, departure points and bicubic interpolation vs the
    reference (steppers.py:171-212, semilag.py:25-179)."""
    from oracle import semilag as osl
    g = load_golden("settls_M16.npz")
    M = int(g["M"])
    sph = sphere(M)
    cfg = StepCfg(dt=float(g["dt"]), visc_nu=float(g["nu"]), scheme="sl_si_settls")
    s0 = state_from(sph, g["s0"], g["phibar"])
    s1 = osl.settls_step(s0, None, cfg)
    s2 = osl.settls_step(s1, s0, cfg)
    s2o = osl.settls_step(s1, None, cfg)
    for st, key in ((s1, "s1"), (s2, "s2"), (s2o, "s2_one")):
        got = np.stack([st.phi[0], st.xi[0], st.delta[0]])
        assert rel_diff(got, g[key]) < 1e-11, key
    lam, th = osl.departure_points(sph, g["u"], g["v"], 1.1 * g["u"], 0.9 * g["v"],
                                   float(g["dep_dt"]))
    assert np.abs(lam - g["lam"]).max() < 1e-12 and np.abs(th - g["th"]).max() < 1e-12
    gi = osl.GridInterp(sph)
    adv = gi.apply(g["vals"], gi.stencil(lam, th))
    assert np.abs(adv - g["adv"]).max() < 1e-12 * np.abs(g["adv"]).max()
