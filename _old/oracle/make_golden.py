"""Generate golden vectors from the REFERENCE implementation itself.

TEST INFRASTRUCTURE ONLY.  Run in the build container, where the read-only
reference exists:

    python oracle/make_golden.py            # writes tests/golden/*.npz

It imports `pintswe` from /root/reference/pkg/src (never copies its source)
and records, on seeded inputs, the outputs of the reference's own transforms
(spharm.py:238-343), tendencies (dynamics.py:121-165), IMEX step
(steppers.py:155-168) and Parareal/MGRIT engine (pint.py:355-430).  It also
copies the reference's frozen run outputs (pkg/frontend/fixtures/*.csv,
produced by `pintswe run-pint` on fixtures/manifest.json) as data.
The GPU box never runs this script; the committed .npz files travel instead.
"""

from __future__ import annotations

import json
import os
import shutil
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _state_arrays(s):
    return np.stack([s.phi, s.xi, s.delta])


def _random_state(grid, rng, phibar, scales=(1e3, 1e-5, 1e-6)):
    """Random valid state (test_dynamics.py:23-31 scales), m = 0 rows real."""
    from pintswe.dynamics import PrognosticState
    out = []
    for sc in scales:
        c = rng.standard_normal(grid.n_modes) + 1j * rng.standard_normal(grid.n_modes)
        c[: grid.M + 1] = c[: grid.M + 1].real
        # smooth spectrum so the nonlinear terms stay tame
        c *= sc * (grid.n_of + 1.0) ** -2.0
        out.append(c)
    out[1][0] = 0.0
    out[2][0] = 0.0
    out[0][0] += phibar * np.sqrt(2.0)
    return PrognosticState(grid, out[0], out[1], out[2], phibar)


def gen_sht(M, seed):
    from pintswe.spharm import get_grid
    g = get_grid(M)
    rng = np.random.default_rng(seed)
    nb = 3
    c = rng.standard_normal((nb, g.n_modes)) + 1j * rng.standard_normal((nb, g.n_modes))
    c[:, : M + 1] = c[:, : M + 1].real
    grid_in = rng.standard_normal((nb, g.nlat, g.nlon))
    out = dict(M=M, mu=g.mu, weights=g.weights, coeffs=c, grid_in=grid_in)
    out["synthesis"] = np.stack([g.synthesis(x) for x in c])
    out["analysis"] = np.stack([g.analysis(x) for x in grid_in])
    out["pair"] = np.stack([g._synthesis_pair(c[0], c[1])])
    u, v = g.uv_from_vortdiv(c[0], c[1])
    out["u"], out["v"] = u, v
    xi, de = g.vortdiv_from_uv(grid_in[0], grid_in[1])
    out["vd_xi"], out["vd_delta"] = xi, de
    gx, gy = g.grad_grid(c[2])
    out["gx"], out["gy"] = gx, gy
    return out


def gen_tendencies(M, seed):
    from pintswe import dynamics
    from pintswe.spharm import get_grid
    g = get_grid(M)
    rng = np.random.default_rng(seed)
    phibar = 9.80616 * 29400.0
    s = _random_state(g, rng, phibar)
    out = dict(M=M, phibar=phibar, state=_state_arrays(s))
    for name in ("linear_gravity", "linear_coriolis", "nonlinear_advection",
                 "nonlinear_rest", "full_rhs"):
        t = getattr(dynamics, name)(s)
        out[name] = np.stack([t.phi, t.xi, t.delta])
    return out


def gen_steps(M, seed):
    """One and several IMEX steps on bumps and on a random state."""
    from pintswe import scenarios, steppers
    from pintswe.dynamics import ViscositySpec
    from pintswe.spharm import get_grid
    from pintswe.steppers import StepperConfig, StepperState
    g = get_grid(M)
    rng = np.random.default_rng(seed)
    bumps = scenarios.gaussian_bumps(g)
    rnd = _random_state(g, rng, bumps.phibar)
    cases = {
        "bumps_dt600_nu1e5": (bumps, StepperConfig(dt=600.0, viscosity=ViscositySpec(2, 1e5)), 1),
        "bumps_dt240_nu0_x3": (bumps, StepperConfig(dt=240.0), 3),
        "random_dt120_q4": (rnd, StepperConfig(dt=120.0, viscosity=ViscositySpec(4, 1e16)), 1),
        "bumps_dt600_explicit": (bumps, StepperConfig(dt=600.0, coriolis_treatment="explicit"), 1),
    }
    out = dict(M=M, phibar=bumps.phibar)
    for key, (s0, cfg, n) in cases.items():
        s = StepperState(s0)
        for _ in range(n):
            s = steppers.advance(s, cfg)
        out[key + "_in"] = _state_arrays(s0)
        out[key + "_out"] = _state_arrays(s.current)
        out[key + "_cfg"] = np.array([cfg.dt, cfg.viscosity.order_q, cfg.viscosity.coeff_nu,
                                      1.0 if cfg.coriolis_treatment == "implicit" else 0.0, n])
    return out


def gen_window_step(M, dt, nu, window=32):
    """Big-M step on bumps, stored only on the n <= window modes."""
    from pintswe import scenarios, steppers
    from pintswe.dynamics import ViscositySpec
    from pintswe.spharm import get_grid
    from pintswe.steppers import StepperConfig
    g = get_grid(M)
    s0 = scenarios.gaussian_bumps(g)
    s1 = steppers.imex_step(s0, StepperConfig(dt=dt, viscosity=ViscositySpec(2, nu)))
    sel = (g.n_of <= window)
    return dict(M=M, dt=dt, nu=nu, window=window, sel=np.flatnonzero(sel),
                out_window=_state_arrays(s1)[:, sel],
                out_maxabs=np.array([np.abs(f).max() for f in (s1.phi, s1.xi, s1.delta)]))


def gen_pint(name, fineM, coarseM, dt0, T, nlevels, cfactor, nrelax, iters, nu_f, nu_c,
             cycle="F_then_V", coarse_scheme="imex", chunk_size=0):
    from pintswe import pint, scenarios
    from pintswe.dynamics import ViscositySpec
    from pintswe.pint import LevelSpec, PintConfig, SweProblem
    from pintswe.steppers import StepperConfig
    levels = [LevelSpec(0, fineM, StepperConfig(dt=dt0, viscosity=ViscositySpec(2, nu_f)))]
    for l in range(1, nlevels):
        levels.append(LevelSpec(l, coarseM, StepperConfig(scheme=coarse_scheme,
                                                          dt=dt0 * cfactor ** l,
                                                          viscosity=ViscositySpec(2, nu_c))))
    N0 = int(round(T / dt0))
    pc = PintConfig(levels=tuple(levels), T=T, N0=N0, cfactor=cfactor, nrelax=nrelax,
                    max_iters=iters, cycle=cycle, chunk_size=chunk_size)
    prob = SweProblem(pc)
    u0 = scenarios.gaussian_bumps(prob.grids[0])
    fine = pint.fine_serial_cpoints(prob, pc, u0)
    tr = pint.mgrit_run(prob, pc, u0)
    snaps = np.stack([np.stack([_state_arrays(x) for x in snap]) for snap in tr.snapshots])
    return dict(name=name, fineM=fineM, coarseM=coarseM, dt0=dt0, T=T, nlevels=nlevels,
                cfactor=cfactor, nrelax=nrelax, iters=iters, nu_f=nu_f, nu_c=nu_c,
                cycle=cycle, coarse_scheme=coarse_scheme, chunk_size=chunk_size,
                u0=_state_arrays(u0), phibar=u0.phibar,
                fine=np.stack([_state_arrays(x) for x in fine]), snapshots=snaps)


def gen_settls(M, seed):
    """SL-SI-SETTLS (steppers.py:171-212) and its semi-Lagrangian pieces
    (semilag.py:25-179) on seeded inputs."""
    from pintswe import semilag, steppers
    from pintswe.dynamics import ViscositySpec
    from pintswe.spharm import get_grid
    from pintswe.steppers import StepperConfig, StepperState
    grid = get_grid(M)
    rng = np.random.default_rng(seed)
    s0 = _random_state(grid, rng, 9.80616 * 29400.0, scales=(2e3, 2e-5, 2e-6))
    cfg2 = StepperConfig(scheme="sl_si_settls", dt=1200.0, viscosity=ViscositySpec(2, 1e5))
    cfg1 = StepperConfig(scheme="sl_si_settls", dt=1200.0, viscosity=ViscositySpec(2, 1e5),
                         settls_mode="one_step")
    s1 = steppers.settls_step(StepperState(s0), cfg2)          # cold start
    s2 = steppers.settls_step(StepperState(s1, s0), cfg2)      # two-step history
    s2o = steppers.settls_step(StepperState(s1, s0), cfg1)     # one-step ignores it
    u = 20.0 * rng.standard_normal((grid.nlat, grid.nlon))
    v = 10.0 * rng.standard_normal((grid.nlat, grid.nlon))
    lam, th = semilag.departure_points(grid, u, v, 1.1 * u, 0.9 * v, 900.0)
    vals = rng.standard_normal((grid.nlat, grid.nlon))
    adv = semilag.advect_scalar(grid, vals, lam, th)
    return dict(M=M, dt=1200.0, nu=1e5, phibar=s0.phibar, s0=_state_arrays(s0),
                s1=_state_arrays(s1), s2=_state_arrays(s2), s2_one=_state_arrays(s2o),
                u=u, v=v, dep_dt=900.0, lam=lam, th=th, vals=vals, adv=adv)


# --------------------------------------------------------------------------- round 2
# Compact PinT goldens for the BASELINE configs at their real parameters: every
# C-point of every iteration on the modes n <= window (the modes the coarse
# level corrects), full states at the middle and last C-point, per-field max|.|
# of every C-point, and the reference's own run-pint outputs (errors.csv /
# spectrum.csv written by runner._pint_outputs from the same trace).

# acceptance C10 configs (/root/reference/pkg/tests/test_acceptance.py:251-275)
AC10_CONFIG = {
    "scenario": "gaussian_bumps", "T": 6 * 3600.0,
    "fine": {"M": 64, "dt": 240.0, "scheme": "imex", "viscosity": {"order": 2, "coeff": 0.0}},
    "pint": {"nlevels": 2, "cfactor": 2, "nrelax": 0, "max_iters": 5, "chunk_size": 0,
             "coarse": {"M": 32, "scheme": "imex", "viscosity": {"order": 2, "coeff": 1.0e5}}},
    "diagnostics": {"rnorms": [8, 32], "spectrum_iterations": [0, 5], "l2": False},
}
AC10_AGGRESSIVE = {
    "scenario": "gaussian_bumps", "T": 48 * 240.0,
    "fine": {"M": 64, "dt": 240.0, "scheme": "imex", "viscosity": {"order": 2, "coeff": 0.0}},
    "pint": {"nlevels": 3, "cfactor": 4, "nrelax": 0, "max_iters": 5, "chunk_size": 0,
             "coarse": {"M": 32, "scheme": "imex", "viscosity": {"order": 2, "coeff": 1.0e5}}},
    "diagnostics": {"rnorms": [8, 32], "spectrum_iterations": [0], "l2": False},
}


def _with(cfg, **pint_over):
    import copy
    out = copy.deepcopy(cfg)
    for k, v in pint_over.items():
        if k in ("T",):
            out[k] = v
        else:
            out["pint"][k] = v
    return out


# cfg1 (BASELINE configs[0]): the bumps-pint-desk preset
# (config.py:113-124) on 8 intervals x 4 fine steps = N0 32 (T = 7680 s),
# Parareal (nrelax 0, cfactor 2), 5 iterations
CFG1 = _with(AC10_CONFIG, T=32 * 240.0)
# cfg3's level structure (3 levels, cfactor 4, nrelax 2, F_then_V) at M=64/32
CFG3_STRUCT = _with(AC10_AGGRESSIVE, nrelax=2, max_iters=4)


def gen_pint_run(name, cfg, window=32):
    """Reference trace of runner.cmd_run_pint's computation for `cfg`
    (runner.py:215-257), stored compactly, plus its errors.csv/spectrum.csv."""
    import tempfile
    from pintswe import pint, runner
    pcfg = runner.build_pint_config(cfg)
    geometry = runner.build_geometry(cfg)
    prob = pint.SweProblem(pcfg, geometry)
    u0 = runner.initial_state(cfg, pcfg.levels[0].M, geometry)
    fine = pint.fine_serial_cpoints(prob, pcfg, u0)
    tr = pint.mgrit_run(prob, pcfg, u0, fine_reference=fine)
    g0 = prob.grids[0]
    sel = np.flatnonzero(g0.n_of <= window)
    snaps = np.stack([np.stack([_state_arrays(x) for x in snap]) for snap in tr.snapshots])
    fine_a = np.stack([_state_arrays(x) for x in fine])
    n1 = snaps.shape[1] - 1
    full_idx = np.array(sorted({n1 // 2, n1}))
    with tempfile.TemporaryDirectory() as td:
        runner._pint_outputs(td, cfg, tr, fine[-1], None, 0.0, "ok", 1)
        errors = open(os.path.join(td, "errors.csv")).read()
        spectrum = open(os.path.join(td, "spectrum.csv")).read()
    lv = pcfg.levels
    return dict(name=name, config_json=json.dumps(cfg, sort_keys=True), window=window, sel=sel,
                fineM=lv[0].M, coarseM=lv[1].M, dt0=lv[0].dt, T=pcfg.T, N0=pcfg.N0,
                nlevels=pcfg.nlevels, cfactor=pcfg.cfactor, nrelax=pcfg.nrelax,
                iters=pcfg.max_iters, nu_f=lv[0].stepper.viscosity.coeff_nu,
                nu_c=lv[1].stepper.viscosity.coeff_nu, cycle=pcfg.cycle,
                u0=_state_arrays(u0), phibar=u0.phibar,
                snap_window=snaps[..., sel], snap_full_idx=full_idx,
                snap_full=snaps[:, full_idx], snap_maxabs=np.abs(snaps).max(axis=-1),
                fine_window=fine_a[..., sel], fine_final=fine_a[-1],
                errors_csv=np.array(errors), spectrum_csv=np.array(spectrum))


# cfg3's real horizon (N0 1024, dt0 60 s, 3 levels, cfactor 4, nrelax 2, coarse
# M=51) with the fine level at M=64 (the reference runs it in ~1 h): the engine
# diverges; the golden records the reference's blow-up iteration / slice and the
# trace up to it
CFG3_BLOWUP = {
    "scenario": "gaussian_bumps", "T": 1024 * 60.0,
    "fine": {"M": 64, "dt": 60.0, "scheme": "imex", "viscosity": {"order": 2, "coeff": 1.0e5}},
    "pint": {"nlevels": 3, "cfactor": 4, "nrelax": 2, "max_iters": 4, "chunk_size": 0,
             "coarse": {"M": 51, "scheme": "imex", "viscosity": {"order": 2, "coeff": 1.0e5}}},
    "diagnostics": {"rnorms": [8, 32], "spectrum_iterations": [0], "l2": False},
}


def gen_pint_blowup(name, cfg, window=32):
    """Reference mgrit_run until PintBlowUpError (pint.py:396-400): blow-up record
    plus the compact trace of the iterations before it."""
    from pintswe import pint, runner
    pcfg = runner.build_pint_config(cfg)
    geometry = runner.build_geometry(cfg)
    prob = pint.SweProblem(pcfg, geometry)
    u0 = runner.initial_state(cfg, pcfg.levels[0].M, geometry)
    try:
        tr = pint.mgrit_run(prob, pcfg, u0)
        blow = None
    except pint.PintBlowUpError as exc:
        tr = exc.trace
        blow = (exc.iteration, exc.slice_index)
    g0 = prob.grids[0]
    sel = np.flatnonzero(g0.n_of <= window)
    k_ok = len(tr.snapshots) if blow is None else blow[0]
    snaps = np.stack([np.stack([_state_arrays(x) for x in snap]) for snap in tr.snapshots[:k_ok]])
    lv = pcfg.levels
    # windowed states on every 16th C-point, the last one and those around slice 203
    n = snaps.shape[1]
    win_idx = np.array(sorted(set(range(0, n, 16)) | {n - 1} | set(range(200, 208))))
    return dict(name=name, config_json=json.dumps(cfg, sort_keys=True), window=window, sel=sel,
                fineM=lv[0].M, coarseM=lv[1].M, dt0=lv[0].dt, T=pcfg.T, N0=pcfg.N0,
                nlevels=pcfg.nlevels, cfactor=pcfg.cfactor, nrelax=pcfg.nrelax,
                iters=pcfg.max_iters, nu_f=lv[0].stepper.viscosity.coeff_nu,
                nu_c=lv[1].stepper.viscosity.coeff_nu, cycle=pcfg.cycle,
                u0=_state_arrays(u0), phibar=u0.phibar,
                blowup=np.array(blow if blow else (-1, -1)), win_idx=win_idx,
                snap_window=snaps[:, win_idx][..., sel], snap_maxabs=np.abs(snaps).max(axis=-1),
                snap_full_idx=np.array([snaps.shape[1] - 1]), snap_full=snaps[:, -1:])


# BASELINE cfg2 at its real parameters (M=256/51, dt 60/120 s, nu 1e5, cfactor 2,
# nrelax 1, N0 128), first 2 iterations (the reference needs ~15 min per iteration)
CFG2 = {
    "scenario": "gaussian_bumps", "T": 128 * 60.0,
    "fine": {"M": 256, "dt": 60.0, "scheme": "imex", "viscosity": {"order": 2, "coeff": 1.0e5}},
    "pint": {"nlevels": 2, "cfactor": 2, "nrelax": 1, "max_iters": 2, "chunk_size": 0,
             "coarse": {"M": 51, "scheme": "imex", "viscosity": {"order": 2, "coeff": 1.0e5}}},
    "diagnostics": {"rnorms": [8, 32], "spectrum_iterations": [0, 2], "l2": False},
}


# BASELINE cfg3 at its real parameters (M=256/51/51, dt 60/240/960 s, nu 1e5, cfactor 4,
# nrelax 2, F_then_V, N0 1024): the first iteration only (~4 h of reference time)
CFG3 = {
    "scenario": "gaussian_bumps", "T": 1024 * 60.0,
    "fine": {"M": 256, "dt": 60.0, "scheme": "imex", "viscosity": {"order": 2, "coeff": 1.0e5}},
    "pint": {"nlevels": 3, "cfactor": 4, "nrelax": 2, "max_iters": 1, "chunk_size": 0,
             "coarse": {"M": 51, "scheme": "imex", "viscosity": {"order": 2, "coeff": 1.0e5}}},
    "diagnostics": {"rnorms": [8, 32], "spectrum_iterations": [0, 1], "l2": False},
}


def gen_pint_big(name, cfg, window=24, workers=1):
    """Reference mgrit_run (no serial fine run) stored compactly: every C-point of
    every iteration on n <= window, max|.| per field, the full last C-point."""
    from pintswe import pint, runner
    pcfg = runner.build_pint_config(cfg)
    geometry = runner.build_geometry(cfg)
    prob = pint.SweProblem(pcfg, geometry)
    u0 = runner.initial_state(cfg, pcfg.levels[0].M, geometry)
    tr = pint.mgrit_run(prob, pcfg, u0, workers=workers)
    g0 = prob.grids[0]
    sel = np.flatnonzero(g0.n_of <= window)
    snaps = np.stack([np.stack([_state_arrays(x) for x in snap]) for snap in tr.snapshots])
    if snaps.shape[1] > 65:   # long horizons: every 8th C-point and the last few
        keep = np.array(sorted(set(range(0, snaps.shape[1], 8)) | {snaps.shape[1] - 1}))
    else:
        keep = np.arange(snaps.shape[1])
    lv = pcfg.levels
    return dict(name=name, config_json=json.dumps(cfg, sort_keys=True), window=window, sel=sel,
                fineM=lv[0].M, coarseM=lv[1].M, dt0=lv[0].dt, T=pcfg.T, N0=pcfg.N0,
                nlevels=pcfg.nlevels, cfactor=pcfg.cfactor, nrelax=pcfg.nrelax,
                iters=pcfg.max_iters, nu_f=lv[0].stepper.viscosity.coeff_nu,
                nu_c=lv[1].stepper.viscosity.coeff_nu, cycle=pcfg.cycle,
                u0=_state_arrays(u0), phibar=u0.phibar,
                win_idx=keep, snap_window=snaps[:, keep][..., sel],
                snap_maxabs=np.abs(snaps).max(axis=-1),
                snap_full_idx=np.array([snaps.shape[1] - 1]), snap_full=snaps[:, -1:])


def gen_m1024_step(window=64):
    """cfg5's step (M=1024, dt=2 s, nu=0, gaussian_bumps, steppers.py:155-168) on
    the modes n <= window, with per-field max|.| of the whole output."""
    out = gen_window_step(1024, 2.0, 0.0, window=window)
    return out


def gen_m1024_sht(seed=230609497, nfs=2, rows=(0, 1, 383, 768, 1536)):
    """cfg4's transforms at M=1024 on `nfs` field-slices drawn with cfg4's law
    (amplitude (n+1)^-1.5, random phase, m = 0 real): synthesis on a few latitude
    rows, analysis of a seeded random grid on n <= 64 plus max|.|."""
    from pintswe.spharm import get_grid
    M = 1024
    g = get_grid(M)
    rng = np.random.default_rng(seed)
    ph = rng.uniform(0.0, 2.0 * np.pi, size=(nfs, g.n_modes))
    amp = (g.n_of + 1.0) ** -1.5
    c = amp * np.exp(1j * ph)
    c[:, : M + 1] = amp[: M + 1] * np.cos(ph[:, : M + 1])
    rows = np.array(rows)
    syn = np.stack([g.synthesis(x)[rows] for x in c])
    rng2 = np.random.default_rng(seed + 1)
    gin = rng2.standard_normal((nfs, g.nlat, g.nlon))
    an = np.stack([g.analysis(x) for x in gin])
    sel = np.flatnonzero(g.n_of <= 64)
    # the coefficients are regenerated from `seed` by the tests (cfg4's law above)
    return dict(M=M, seed=seed, nfs=nfs, rows=rows, synthesis_rows=syn,
                synthesis_maxabs=np.array([np.abs(g.synthesis(x)).max() for x in c]),
                grid_seed=seed + 1, analysis_window=an[:, sel], sel=sel,
                analysis_maxabs=np.abs(an).max(axis=-1))


def main_r2(which):
    """Round-2 goldens: `python oracle/make_golden.py cfg1 ac10 cfg3s m1024 m1024sht`."""
    jobs = {
        "cfg1": ("pint_cfg1_M64.npz", lambda: gen_pint_run("cfg1", CFG1)),
        "ac10": ("pint_ac10_M64.npz", lambda: gen_pint_run("ac10", AC10_CONFIG)),
        "ac10agg": ("pint_ac10agg_M64.npz", lambda: gen_pint_run("ac10agg", AC10_AGGRESSIVE)),
        "cfg3s": ("pint_cfg3s_M64.npz", lambda: gen_pint_run("cfg3s", CFG3_STRUCT)),
        "m1024": ("step_window_M1024.npz", gen_m1024_step),
        "cfg2": ("pint_cfg2_M256.npz", lambda: gen_pint_big("cfg2", CFG2)),
        "cfg3": ("pint_cfg3_M256.npz", lambda: gen_pint_big("cfg3", CFG3, workers=6)),
        "cfg3blow": ("pint_cfg3blow_M64.npz", lambda: gen_pint_blowup("cfg3blow", CFG3_BLOWUP)),
        "m1024sht": ("sht_M1024.npz", gen_m1024_sht),
    }
    for w in which:
        fn, job = jobs[w]
        np.savez_compressed(os.path.join(OUT, fn), **job())
        print("wrote", fn, flush=True)


def main():
    sys.path.insert(0, REF)
    os.makedirs(OUT, exist_ok=True)
    if len(sys.argv) > 1:
        return main_r2(sys.argv[1:])
    np.savez_compressed(os.path.join(OUT, "sht_M16.npz"), **gen_sht(16, 230609497))
    np.savez_compressed(os.path.join(OUT, "sht_M32.npz"), **gen_sht(32, 230609498))
    np.savez_compressed(os.path.join(OUT, "tend_M24.npz"), **gen_tendencies(24, 7))
    np.savez_compressed(os.path.join(OUT, "step_M16.npz"), **gen_steps(16, 11))
    np.savez_compressed(os.path.join(OUT, "step_M32.npz"), **gen_steps(32, 12))
    np.savez_compressed(os.path.join(OUT, "step_window_M256.npz"),
                        **gen_window_step(256, 60.0, 1e5))
    # the frozen fixture run (manifest.json): Parareal, M16/M16, 4 iterations
    np.savez_compressed(os.path.join(OUT, "pint_fixture_M16.npz"),
                        **gen_pint("fixture", 16, 16, 600.0, 7200.0, 2, 2, 0, 4, 0.0, 1e5))
    # a 3-level F_then_V MGRIT with relaxation, spatial coarsening
    np.savez_compressed(os.path.join(OUT, "pint_mgrit3_M24.npz"),
                        **gen_pint("mgrit3", 24, 16, 300.0, 9600.0, 3, 2, 1, 3, 0.0, 1e5))
    # 2-level MGRIT with nrelax=1 (cfg2's level structure at small M)
    np.savez_compressed(os.path.join(OUT, "pint_mgrit2_M32.npz"),
                        **gen_pint("mgrit2", 32, 16, 240.0, 7680.0, 2, 2, 1, 3, 1e5, 1e5))
    # SL-SI-SETTLS: the stepper and a Parareal run with a SETTLS coarse level
    # (bumps-pint-settls structure at small M), one with chunk boundaries
    np.savez_compressed(os.path.join(OUT, "settls_M16.npz"), **gen_settls(16, 21))
    np.savez_compressed(os.path.join(OUT, "pint_settls_M24.npz"),
                        **gen_pint("settls", 24, 16, 300.0, 4800.0, 2, 2, 0, 3, 0.0, 1e6,
                                   coarse_scheme="sl_si_settls"))
    np.savez_compressed(os.path.join(OUT, "pint_settls_chunk_M24.npz"),
                        **gen_pint("settls_chunk", 24, 16, 300.0, 4800.0, 2, 2, 1, 3, 0.0, 1e6,
                                   coarse_scheme="sl_si_settls", chunk_size=2))
    fx = os.path.join(OUT, "fixtures")
    os.makedirs(fx, exist_ok=True)
    src = "/root/reference/pkg/frontend/fixtures"
    for name in ("errors.csv", "spectrum.csv", "manifest.json"):
        shutil.copyfile(os.path.join(src, name), os.path.join(fx, name))
    with open(os.path.join(OUT, "README.md"), "w") as fh:
        fh.write("Golden vectors generated by `python oracle/make_golden.py` from the "
                 "reference `pintswe` (imported read-only from /root/reference/pkg/src).\n"
                 "`fixtures/` holds the reference's frozen run-pint outputs "
                 "(pkg/frontend/fixtures) as data.\n")
    print(json.dumps(sorted(os.listdir(OUT))))


if __name__ == "__main__":
    main()
