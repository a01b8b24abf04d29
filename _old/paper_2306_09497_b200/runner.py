"""`run-pint` outputs from the GPU path (reference runner.py:171-257, ioutils.py).

The subset of the reference runner that drives the hot path end to end:
config sections `fine`, `pint`, `T`, `scenario` (gaussian_bumps),
`diagnostics` and optionally `reference`/`geometry`, exactly as
`runner.build_pint_config` reads them (runner.py:30-86); outputs errors.csv,
spectrum.csv, speedup.csv and manifest.json with the reference's 17-digit
formatting (ioutils.py:15-35), computed with the on-device diagnostics.
CLI parsing, presets and the other commands stay out of scope.
"""

from __future__ import annotations

import json
import os
import time

from . import __version__, diagnostics, pint, scenarios, steppers
from .dynamics import ViscositySpec
from .pint import LevelSpec, PintConfig, SweProblem
from .spharm import SphereGeometry, get_grid

EXIT_OK = 0
EXIT_CONFIG = 2
EXIT_BLOWUP = 3


class ConfigError(ValueError):
    """Invalid configuration (reference config.py ConfigError)."""


def fmt(value) -> str:
    if isinstance(value, bool):
        return "1" if value else "0"
    if isinstance(value, float):
        return format(value, ".17g")
    return str(value)


def write_csv(path, header, rows) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write(",".join(header) + "\n")
        for row in rows:
            fh.write(",".join(fmt(v) for v in row) + "\n")


def write_json(path, payload) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        json.dump(payload, fh, indent=2, sort_keys=True)


def build_geometry(cfg: dict) -> SphereGeometry:
    g = cfg.get("geometry", {})
    d = SphereGeometry()
    return SphereGeometry(radius_a=g.get("radius_a", d.radius_a), omega=g.get("omega", d.omega),
                          gravity_g=g.get("gravity_g", d.gravity_g))


def build_stepper(section: dict, dt=None) -> steppers.StepperConfig:
    try:
        v = section.get("viscosity", {})
        return steppers.StepperConfig(
            scheme=section.get("scheme", "imex"),
            dt=float(dt if dt is not None else section["dt"]),
            viscosity=ViscositySpec(order_q=int(v.get("order", 2)),
                                    coeff_nu=float(v.get("coeff", 0.0))),
            settls_mode=section.get("settls_mode", "two_step"),
            coriolis_treatment=section.get("coriolis_treatment", "implicit"))
    except (KeyError, ValueError) as exc:
        raise ConfigError(f"bad stepper section: {exc}") from exc


def build_pint_config(cfg: dict) -> PintConfig:
    fine, p = cfg["fine"], cfg["pint"]
    T, dt0 = float(cfg["T"]), float(fine["dt"])
    nlevels, cfactor = int(p.get("nlevels", 2)), int(p.get("cfactor", 2))
    coarse = p.get("coarse", {})
    levels = [LevelSpec(0, int(fine["M"]), build_stepper(fine))]
    for lv in range(1, nlevels):
        levels.append(LevelSpec(lv, int(coarse.get("M", fine["M"])),
                                build_stepper(coarse, dt=dt0 * cfactor ** lv)))
    try:
        return PintConfig(levels=tuple(levels), T=T, N0=int(round(T / dt0)), cfactor=cfactor,
                          nrelax=int(p.get("nrelax", 0)), max_iters=int(p.get("max_iters", 10)),
                          chunk_size=int(p.get("chunk_size", 0)),
                          cycle=p.get("cycle", pint.F_THEN_V))
    except ValueError as exc:
        raise ConfigError(str(exc)) from exc


def initial_state(cfg: dict, M: int, geometry: SphereGeometry):
    name = cfg.get("scenario")
    if name != "gaussian_bumps":
        raise ConfigError(f"scenario {name!r}: only gaussian_bumps is on the GPU path")
    return scenarios.gaussian_bumps(get_grid(M, geometry))


def serial_run(state, stepper_cfg, T: float, check_every: int = 32):
    """Serial propagation with periodic blow-up checks (runner.py:89-103)."""
    nsteps_f = T / stepper_cfg.dt
    nsteps = int(round(nsteps_f))
    if abs(nsteps_f - nsteps) > 1e-9:
        raise ConfigError("T must be an integral number of fine steps")
    s = state.copy()
    limit = 1e10 * max(state.max_abs(), 1e-300)
    done = 0
    while done < nsteps:
        k = min(check_every, nsteps - done)
        steppers.imex_steps_inplace(s, stepper_cfg, k)
        done += k
        if not s.is_finite() or s.max_abs() > limit:
            raise pint.PintBlowUpError(0, done, None)
    return s


def _manifest(out_dir, command, cfg, status, extra=None):
    payload = {"command": command, "config": cfg, "status": status, "version": __version__}
    if extra:
        payload.update(extra)
    write_json(os.path.join(out_dir, "manifest.json"), payload)


def _pint_outputs(out_dir, cfg, trace, fine_final, reference, t_ref, status, workers):
    """runner.py:171-211."""
    diag = cfg.get("diagnostics", {})
    rnorms = diag.get("rnorms", [8])
    include_l2 = diag.get("l2", False)
    error_rows = []
    for k, snap in enumerate(trace.snapshots):
        last = snap[-1]
        recs = diagnostics.phi_error_records(k, last, "fine", fine_final, rnorms,
                                             include_l2=include_l2)
        if reference is not None:
            recs += diagnostics.phi_error_records(k, last, "reference", reference, rnorms,
                                                  include_l2=include_l2)
        error_rows.extend(r.row() for r in recs)
    write_csv(os.path.join(out_dir, "errors.csv"), diagnostics.ERROR_HEADER, error_rows)

    spec_rows = diagnostics.spectrum_rows("fine", "", diagnostics.ke_spectrum(fine_final))
    if reference is not None:
        spec_rows += diagnostics.spectrum_rows("reference", "", diagnostics.ke_spectrum(reference))
    for k in diag.get("spectrum_iterations", []):
        if 0 <= k < len(trace.snapshots):
            spec_rows += diagnostics.spectrum_rows(
                "pint", k, diagnostics.ke_spectrum(trace.snapshots[k][-1]))
    write_csv(os.path.join(out_dir, "spectrum.csv"), diagnostics.SPECTRUM_HEADER, spec_rows)

    speed_rows = [(r.iteration, r.wall_time, r.cumulative_time, r.speedup)
                  for r in pint.speedup_report(trace, t_ref)]
    write_csv(os.path.join(out_dir, "speedup.csv"),
              ("iteration", "wall_seconds", "cumulative_seconds", "speedup"), speed_rows)
    pcfg = trace.config
    engine = "parareal" if pcfg.nlevels == 2 and pcfg.nrelax == 0 else "mgrit"
    extra = {"engine": engine, "workers": workers, "iterations_completed": trace.iterations,
             "t_ref_seconds": t_ref}
    if trace.blowup:
        extra["blowup"] = trace.blowup
    _manifest(out_dir, "run-pint", cfg, status, extra)


def cmd_run_pint(cfg: dict, out_dir: str, workers: int = 1) -> int:
    """runner.py:215-257 on the GPU path."""
    if "fine" not in cfg or "pint" not in cfg or "T" not in cfg:
        raise ConfigError("run-pint needs 'fine', 'pint' and 'T'")
    os.makedirs(out_dir, exist_ok=True)
    geometry = build_geometry(cfg)
    pcfg = build_pint_config(cfg)
    problem = SweProblem(pcfg, geometry)
    u0 = initial_state(cfg, pcfg.levels[0].M, geometry)

    t0 = time.perf_counter()
    fine_cpoints = pint.fine_serial_cpoints(problem, pcfg, u0)
    fine_final = fine_cpoints[-1]
    t_ref = time.perf_counter() - t0

    reference = None
    if "reference" in cfg:
        ref0 = initial_state(cfg, int(cfg["reference"]["M"]), geometry)
        reference = serial_run(ref0, build_stepper(cfg["reference"]), float(cfg["T"]))
    try:
        trace = pint.mgrit_run(problem, pcfg, u0, workers=workers, fine_reference=fine_cpoints)
        status, code = "ok", EXIT_OK
    except pint.PintBlowUpError as exc:
        trace = exc.trace
        failing = trace.snapshots[exc.iteration]
        keep = exc.iteration + 1 if all(problem.is_finite(v) for v in failing) else exc.iteration
        trace.snapshots = trace.snapshots[:keep]
        trace.wall_times = trace.wall_times[:keep]
        status, code = "blowup", EXIT_BLOWUP
        if not trace.snapshots:
            _manifest(out_dir, "run-pint", cfg, status, {"blowup": trace.blowup,
                                                         "workers": workers})
            return code
    _pint_outputs(out_dir, cfg, trace, fine_final, reference, t_ref, status, workers)
    return code
