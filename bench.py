"""Benchmark: batched fine IMEX propagator of cfg2 (M=256, dt=60 s, nu=1e5).

One bench step = one F-relaxation sweep step of cfg2's fine level: every one of
the 64 time slices owned by a GPU advances one IMEX step (steppers.py:155-168)
in a single batched call.  value = fine slice-steps/s over all ranks (weak
scaling: 64 slices per GPU, no data-path collective in that leg).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--gpus N` with N > 1 and no torchrun environment relaunches itself under
`torch.distributed.run` (one rank per GPU, NCCL).  Besides the headline leg,
every N runs the SHARDED MGRIT legs of BASELINE cfg2 and cfg3 (level-0
C-slices in contiguous blocks per rank, C-point halo send/recv and coarse
all-gather over NCCL inside the timed iterations; device-timed, max over
ranks; traces bitwise independent of N).

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port under oracle/, the reference being pure Python/numpy that cannot
travel to the GPU box) on all host cores: one process per core, the bench
step's 64 slices spread over them, on the same M/dt/nu.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fine SWE steps/s (fp64, M=256) at 1/2/4/8 B200; % FP64-TC / HBM roofline"
UNIT = "fine slice-steps/s"
M, DT, NU = 256, 60.0, 1.0e5
SLICES_PER_GPU = 64


def workload(slices):
    return {"workload": f"cfg2 fine level: gaussian_bumps M={M} dt={DT:g}s nu={NU:g} IMEX, "
                        f"{slices} time slices per GPU advanced one fine step per bench step",
            "M": M, "dt": DT, "nu": NU, "slices_per_gpu": slices, "parallelism": "slices"}


# --------------------------------------------------------------------------- CPU legs
_SPH = None
_STATES = None


def _cpu_worker_step(i):
    from oracle.swe import StepCfg, imex_step
    s = _STATES.slice(i)
    t0 = time.perf_counter()
    imex_step(s, StepCfg(dt=DT, visc_nu=NU))
    return time.perf_counter() - t0


def _cpu_setup(nslices):
    global _SPH, _STATES
    from oracle.sht import OracleSphere
    from oracle.swe import gaussian_bumps
    if _SPH is None:
        _SPH = OracleSphere(M)
    base = gaussian_bumps(_SPH, batch=nslices)
    rng = np.random.default_rng(0)
    for b in range(nslices):
        base.xi[b] += 1e-9 * rng.standard_normal(_SPH.n_modes) * (_SPH.n_of + 1.0) ** -2
    base.xi[:, : M + 1] = base.xi[:, : M + 1].real
    _STATES = base


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_steps(nsteps, nproc, nslices):
    """Oracle IMEX steps of `nslices` slices per bench step, one process per core
    (OPENBLAS_NUM_THREADS=1).  Returns (elapsed seconds of the timed steps,
    slice-steps done)."""
    import multiprocessing as mp
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    _cpu_setup(nslices)
    ctx = mp.get_context("fork")
    with ctx.Pool(nproc) as pool:
        pool.map(_cpu_worker_step, range(nproc))          # warm the workers
        t0 = time.perf_counter()
        for _ in range(nsteps):
            pool.map(_cpu_worker_step, range(nslices), chunksize=1)
        el = time.perf_counter() - t0
    return el, nsteps * nslices


def cpu_baseline_record(value, nproc, nslices, nsteps):
    return {"value": value, "unit": UNIT, "cores": nproc, "kind": "port",
            "cpu_model": cpu_model(), "host_cores_total": os.cpu_count(),
            "sample": f"{nsteps} bench step(s) x {nslices} slices x 1 IMEX step at M={M} "
                      f"(the GPU leg's per-GPU workload), numpy oracle port of "
                      f"steppers.imex_step, one process per core, OPENBLAS_NUM_THREADS=1"}


def cpu_cfg1_mgrit(iters=2):
    """The oracle port of the reference engine (oracle/mgrit.py, MgritEngine control
    flow, serial like the reference's GIL-bound thread pool) on
    BASELINE cfg1 (bumps-pint-desk: M=64/32, dt 240, Parareal, N0 32): reference-
    equivalent fine steps/s = 48 engine-accounted fine steps per iteration / mean
    iteration time (first `iters` iterations, after the initial guess)."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import mgrit as om
    from oracle.sht import OracleSphere
    from oracle.swe import StepCfg, gaussian_bumps
    levels = (om.Level(64, StepCfg(dt=240.0, visc_nu=0.0)),
              om.Level(32, StepCfg(dt=480.0, visc_nu=1e5)))
    pc = om.PintCfg(levels=levels, T=32 * 240.0, N0=32, cfactor=2, nrelax=0, max_iters=iters)
    prob = om.OracleProblem(pc, {64: OracleSphere(64), 32: OracleSphere(32)})
    u0 = gaussian_bumps(prob.spheres[0])
    eng = om.OracleMgrit(prob, pc)
    t0 = time.perf_counter()
    eng.run(u0, iters=0)
    t_guess = time.perf_counter() - t0
    t0 = time.perf_counter()
    eng.run(u0, iters=iters)
    el = time.perf_counter() - t0 - t_guess
    per_it = el / iters
    return {"value": 48 / per_it, "unit": "reference-equivalent fine steps/s",
            "s_per_iteration": per_it, "cores": 1, "kind": "port", "cpu_model": cpu_model(),
            "config": "cfg1: bumps-pint-desk M=64/32, dt 240/480 s, Parareal, N0 32, "
                      "48 fine steps per iteration",
            "sample": f"{iters} MGRIT iterations of the oracle engine (serial)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    nproc = cpu_cores()
    nslices = args.slices
    if args.warmup:
        cpu_steps(args.warmup, nproc, nslices)
    el, done = cpu_steps(args.steps, nproc, nslices)
    v = done / el
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (gaussian_bumps + per-slice perturbation)",
            "config": workload(nslices), "impl": "reference",
            "cpu_baseline": cpu_baseline_record(v, nproc, nslices, args.steps),
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU leg
class Clocks:
    """SM clock and throttle-reason sampling during the timed region
    (B200_PROFILING.md clocks line): NVML polled every 5 ms from a thread (the
    timed region is ~0.1 s, shorter than nvidia-smi's start-up), `nvidia-smi
    -lms` as the fallback."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event-reason bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40}

    def __init__(self, device):
        self.device = device
        self.p = self.f = self.thread = None
        self.rows = []       # NVML samples: (sm MHz, reasons bitmask)
        self.max_mhz = None
        try:
            import threading
            import pynvml
            import torch
            pynvml.nvmlInit()
            try:
                uuid = str(torch.cuda.get_device_properties(device).uuid)
                h = pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid).encode())
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            self.stop_flag = threading.Event()

            def poll():
                while not self.stop_flag.is_set():
                    try:
                        self.rows.append((float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                                          int(reasons(h))))
                    except Exception:
                        pass
                    self.stop_flag.wait(0.005)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={device}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "25"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.thread is not None:
            self.stop_flag.set()
            self.thread.join()
            if not self.rows:
                return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"]}
            reasons = sorted(n for n, bit in self.BITS.items() if any(r[1] & bit for r in self.rows))
            return {"sm_mhz": float(np.median([r[0] for r in self.rows])),
                    "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.rows),
                    "source": "nvml, 5 ms period"}
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for ln in fh:
                parts = [x.strip() for x in ln.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows), "source": "nvidia-smi -lms 25"}


def fp64_peak_tflops(torch, dev, sustain_s=0.0):
    """cuBLAS DGEMM 8192^3 (MEASURED_PEAKS.json has no fp64 entry): best of 5
    (burst), and with sustain_s > 0 also back to back for that long (sustained,
    the power-capped figure for kernels timed inside a long step)."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    burst = 2.0 * n ** 3 / (best * 1e-3) / 1e12
    sustained = None
    if sustain_s > 0:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(1, int(sustain_s / (best * 1e-3)))
        s.record()
        for _ in range(reps):
            torch.matmul(a, b)
        e.record()
        e.synchronize()
        sustained = 2.0 * n ** 3 * reps / (s.elapsed_time(e) * 1e-3) / 1e12
    del a, b
    return burst, sustained


class CudaClock:
    """Per-iteration device time of the MGRIT engine: CUDA events on the current
    stream around each cycle (MgritEngine.run(clock=...))."""

    def __init__(self, torch):
        self.torch = torch

    def start(self):
        self.e0 = self.torch.cuda.Event(enable_timing=True)
        self.e0.record()

    def stop(self):
        e1 = self.torch.cuda.Event(enable_timing=True)
        e1.record()
        e1.synchronize()
        return self.e0.elapsed_time(e1) * 1e-3


def make_states(grid, n, seed):
    """Gaussian bumps + a per-slice vorticity/divergence perturbation."""
    import torch
    from paper_2306_09497_b200 import scenarios
    s = scenarios.gaussian_bumps(grid, batch=n)
    rng = np.random.default_rng(seed)
    pert = rng.standard_normal((n, grid.n_modes)) + 1j * rng.standard_normal((n, grid.n_modes))
    pert[:, : M + 1] = pert[:, : M + 1].real
    pert *= (grid.n_of + 1.0) ** -2
    pt = torch.from_numpy(pert).to(s.data.device)
    s.data[:, 1] += 1e-9 * pt
    s.data[:, 2] += 1e-10 * pt
    return s


PINT_LEGS = {
    # BASELINE configs[0] (bumps-pint-desk preset, config.py:113-124): Parareal,
    # M=64/32, dt 240/480 s, nu 0 / 1e5, cfactor 2, 16 C-slices (N0 32), 5 iterations
    "cfg1": dict(Ms=(64, 32), nus=(0.0, 1e5), dt0=240.0, cfactor=2, nrelax=0, N0=32, iters=5,
                 fine_per_iter=48),
    # BASELINE configs[1]: MGRIT L=2, M=256/51, dt 60/120 s, nu 1e5, cfactor 2,
    # nrelax 1, 64 C-slices (N0 128, T 7680 s), 10 iterations
    "cfg2": dict(Ms=(256, 51), nus=(1e5, 1e5), dt0=60.0, cfactor=2, nrelax=1, N0=128, iters=10,
                 fine_per_iter=320),
    # BASELINE configs[2]: MGRIT L=3, M=256/51/51, dt 60/240/960 s, nu 1e5,
    # cfactor 4, nrelax 2, F_then_V, 256 C-slices (N0 1024, T 61440 s), 10 iterations
    "cfg3": dict(Ms=(256, 51, 51), nus=(1e5, 1e5, 1e5), dt0=60.0, cfactor=4, nrelax=2, N0=1024, iters=10,
                 fine_per_iter=7680),
}


def pint_leg(torch, name, comm=None, iters=None):
    """A BASELINE MGRIT config end to end through pint.mgrit's engine, slices
    sharded over the ranks of `comm` (halo send/recv + coarse all-gather on NCCL
    inside every timed iteration).  SURVEY.md §8d "steps/s accounting":
    reference-equivalent fine steps/s = engine-accounted level-0 steps per
    iteration (summed over ranks) / iteration time; iteration time = CUDA-event
    time of the cycle, max over ranks, median over the iterations (the initial
    guess and the serial fine reference excluded).  A warm-up run of the same
    iterations captures every step graph first."""
    from paper_2306_09497_b200 import dynamics, pint, scenarios, steppers
    spec = PINT_LEGS[name]
    iters = iters or spec["iters"]
    cf = spec["cfactor"]
    lv = [pint.LevelSpec(l, Ml, steppers.StepperConfig(
        dt=spec["dt0"] * cf ** l, viscosity=dynamics.ViscositySpec(2, spec["nus"][l])))
        for l, Ml in enumerate(spec["Ms"])]
    pc = pint.PintConfig(levels=tuple(lv), T=spec["N0"] * spec["dt0"], N0=spec["N0"], cfactor=cf,
                         nrelax=spec["nrelax"], max_iters=iters)
    prob = pint.SweProblem(pc)
    u0 = prob.as_batch(0, scenarios.gaussian_bumps(prob.grids[0]))

    def run():
        # cfg3 diverges (the reference's own engine raises PintBlowUpError at the
        # same iteration, tests/golden/pint_cfg3blow_M64.npz): time the iterations
        # completed before the blow-up iteration
        eng = pint.MgritEngine(prob, pc, comm)
        try:
            return eng.run(u0, keep_snapshots=False, clock=CudaClock(torch)), None
        except pint.PintBlowUpError as exc:
            return exc.trace, exc

    run()
    if comm is not None:
        comm.dist.barrier()
    tr, blow = run()
    n_ok = len(tr.wall_times) - 1 if blow is None else blow.iteration - 1
    dev = u0.device
    t = torch.tensor(tr.wall_times[1:1 + n_ok], dtype=torch.float64, device=dev)
    steps = torch.tensor([sum(tr.fine_steps[:n_ok])], dtype=torch.float64, device=dev)
    if comm is not None:
        comm.dist.all_reduce(t, op=comm.dist.ReduceOp.MAX)
        comm.dist.all_reduce(steps, op=comm.dist.ReduceOp.SUM)
    its = t.cpu().numpy()
    per_it = float(steps[0]) / max(n_ok, 1)
    med = float(np.median(its))
    G = comm.size if comm is not None else 1
    return {"value": per_it / med, "unit": "reference-equivalent fine steps/s",
            "config": f"{name}: MGRIT L={len(spec['Ms'])}, M={'/'.join(map(str, spec['Ms']))}, "
                      f"dt0={spec['dt0']:g} s, nu={'/'.join(f'{x:g}' for x in spec['nus'])}, "
                      f"cfactor {cf}, nrelax {spec['nrelax']}, "
                      f"N0={spec['N0']} ({spec['N0'] // cf} C-slices), gaussian_bumps",
            "ranks": G, "slices_per_rank": spec["N0"] // cf // G,
            "iterations": n_ok, "fine_steps_per_iteration": per_it,
            "blowup": None if blow is None else {
                "iteration": blow.iteration, "slice": blow.slice_index,
                "note": "PintBlowUpError (pint.py:396-400) as in the reference engine; the "
                        "iterations before it are timed"},
            "fine_steps_per_iteration_expected": spec["fine_per_iter"],
            "ms_per_iteration": 1e3 * med, "ms_per_iteration_mean": 1e3 * float(its.mean()),
            "value_from_mean": per_it / float(its.mean()),
            "timing": "CUDA events around each MGRIT cycle, max over ranks, median iteration",
            "collectives": (f"{comm.dist.get_backend().upper()} halo send/recv + all-gather "
                            "of the coarse forcing + all-reduced blow-up check per iteration")
            if G > 1 else "none"}


def coriolis_legs(torch, steppers, cfg, state, steps, flush):
    """The same workload on the reference's own (pseudospectral) Coriolis
    evaluation: fast_coriolis 0 = FFT round trip exactly as dynamics.py:129-135,
    1 = the FFT-free Legendre pair (identity rfft(irfft(X) s) = s X on the band).
    The headline uses the spectral three-term operator (fast_coriolis 2, identical
    to roundoff); these legs separate the algorithmic gain from the
    kernel gain."""
    from paper_2306_09497_b200 import _lib
    out = {}
    ref = state.copy()
    steppers.imex_steps_inplace(ref, cfg, 1)
    for mode, label in ((0, "pseudospectral_fft"), (1, "pseudospectral_fft_free")):
        _lib.set_option("fast_coriolis", mode)
        try:
            st = state.copy()
            steppers.imex_steps_inplace(st, cfg, 1)
            x, y = ref.data.clone(), st.data.clone()
            x[:, 0, 0] = 0.0
            y[:, 0, 0] = 0.0
            rel = float(((x - y).abs().amax(dim=-1) / x.abs().amax(dim=-1)).max())
            for _ in range(2):
                steppers.imex_steps_inplace(st, cfg, 1)
            torch.cuda.synchronize()
            total = 0.0
            for _ in range(steps):
                flush.zero_()
                s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s_ev.record()
                steppers.imex_steps_inplace(st, cfg, 1)
                e_ev.record()
                e_ev.synchronize()
                total += s_ev.elapsed_time(e_ev)
        finally:
            _lib.set_option("fast_coriolis", 2)
        out[label] = {"fast_coriolis": mode, "value": state.batch * steps / (total * 1e-3),
                      "unit": UNIT, "ms_per_step": total / steps,
                      "max_rel_diff_vs_headline": rel}
    out["note"] = ("same workload with the reference's pseudospectral Coriolis operator "
                   "(2 Legendre GEMM pairs + FFTs per fixed-point iteration)")
    return out


def sht_cfg4(torch, Ms=(256, 1024)):
    """cfg4: batched SHT round trip, 3 fields x 256 slices, c_mn =
    (n+1)^-1.5 e^{i phi}, phi ~ U[0, 2 pi) from default_rng(230609497) drawn as
    (3, 256, K), m = 0 entries real (cos phi).  One synthesis + one analysis per
    field-slice, one field (256 slices) per call, coefficients resident on the GPU;
    CUDA events around the 3 fields after a warm-up pass."""
    import numpy as np
    from paper_2306_09497_b200 import spharm
    out = {}
    for M in Ms:
        g = spharm.get_grid(M)
        rng = np.random.default_rng(230609497)
        ph = rng.uniform(0.0, 2.0 * np.pi, size=(3, 256, g.n_modes))
        amp = (g.n_of + 1.0) ** -1.5
        c = amp * np.exp(1j * ph)
        c[..., : M + 1] = amp[: M + 1] * np.cos(ph[..., : M + 1])
        ct = torch.from_numpy(c).cuda()
        del c, ph
        back = g.analysis(g.synthesis(ct[0]))  # warm-up (plans, workspaces)
        torch.cuda.synchronize()
        ms = None
        for _ in range(2):  # best of two passes: the first may still grow the allocator's pool
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            backs = [g.analysis(g.synthesis(ct[f])) for f in range(3)]
            e1.record()
            e1.synchronize()
            t = e0.elapsed_time(e1)
            ms = t if ms is None else min(ms, t)
            err = max(float((backs[f] - ct[f]).abs().max()) for f in range(3))
            del backs
        out[f"M{M}"] = {"field_slices_per_s": 768 / (ms * 1e-3), "ms": ms,
                        "round_trip_max_abs_err": err}
        del ct, back
        torch.cuda.empty_cache()
    out["note"] = "3 fields x 256 slices, synthesis + analysis per field-slice; best of 2 passes"
    return out


def fine_cfg5(torch, slices=64, steps=5):
    """cfg5: M=1024, dt=2 s, nu=0, gaussian_bumps, 64 independent
    intervals per GPU (512 over 8 GPUs) advanced by the fine IMEX step; CUDA
    events around `steps` steps after 2 warm-up steps."""
    from paper_2306_09497_b200 import dynamics, scenarios, spharm, steppers
    g = spharm.get_grid(1024)
    s = scenarios.gaussian_bumps(g, batch=slices)
    cfg = steppers.StepperConfig(dt=2.0, viscosity=dynamics.ViscositySpec(2, 0.0))
    for _ in range(2):  # the second call captures the step graph (outside the timing)
        steppers.imex_steps_inplace(s, cfg, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    steppers.imex_steps_inplace(s, cfg, steps)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    rate = slices / (ms * 1e-3)
    return {"value": rate, "unit": "fine slice-steps/s per GPU", "ms_per_step": ms,
            "slices_per_gpu": slices, "finite": bool(s.is_finite()),
            "cfg5_seconds_at_8_gpus": 15360 / (8 * rate),
            "config": "cfg5: gaussian_bumps M=1024, dt=2 s, nu=0, IMEX, 512 intervals x 30 steps "
                      "(64 per GPU at 8 GPUs)"}


def direct_leg(torch, steppers, cfg, state, steps, flush):
    """Same workload with StepperConfig.implicit_solver="direct" (per-m tridiagonal
    solve of the CN implicit system instead of the reference's fixed point,
    SURVEY.md §8f row 4): device-timed like the main leg, plus its max relative
    difference from the fixed-point step on the same input (Phi' and xi/delta)."""
    import dataclasses
    cfg_d = dataclasses.replace(cfg, implicit_solver="direct")
    st = state.copy()
    for _ in range(3):
        steppers.imex_steps_inplace(st, cfg_d, 1)
    torch.cuda.synchronize()
    total = 0.0
    for _ in range(steps):
        flush.zero_()
        s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_ev.record()
        steppers.imex_steps_inplace(st, cfg_d, 1)
        e_ev.record()
        e_ev.synchronize()
        total += s_ev.elapsed_time(e_ev)
    a, d = state.copy(), state.copy()
    steppers.imex_steps_inplace(a, cfg, 1)
    steppers.imex_steps_inplace(d, cfg_d, 1)
    x, y = a.data.clone(), d.data.clone()
    x[:, 0, 0] = 0.0   # Phi': the mean mode dominates Phi
    y[:, 0, 0] = 0.0
    rel = float(((x - y).abs().amax(dim=-1) / x.abs().amax(dim=-1)).max())
    B = state.batch
    return {"value": B * steps / (total * 1e-3), "unit": "fine slice-steps/s",
            "ms_per_step": total / steps, "max_rel_diff_vs_fixed_point": rel,
            "note": "opt-in solver (implicit_solver='direct'); the headline value uses the "
                    "reference's fixed point"}


def ncu_traffic():
    """DRAM bytes per launch of the dominant kernels from the newest committed
    `ncu --set full` capture (profiles/*_kernels.json, tools/ncu_summary.py)."""
    import glob
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                          "profiles", "r*_kernels.json")))  # round tags sort
    if not files:
        return {}
    try:
        recs = json.load(open(files[-1]))
    except (OSError, ValueError):
        return {}
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def dram(r):
        u = scale.get(r.get("dram__bytes_read.sum:unit", "byte"), 1.0)
        return ((r.get("dram__bytes_read.sum") or 0) + (r.get("dram__bytes_write.sum") or 0)) * u

    leg = [dram(r) for r in recs if r["kernel"].startswith(("leg_synth_v3", "leg_anal_v3"))]
    # the bench configuration's FFT kernel (16-row lanes; M=1024 captures use 8 rows)
    fft = [dram(r) for r in recs
           if "fft_lanes_kernel" in r["kernel"] and ", 8," not in r["kernel"]]
    out = {"source": "profiles/" + os.path.basename(files[-1])}
    if leg:
        out["legendre"] = sum(leg) / len(leg)
    if fft:
        out["fft"] = sum(fft) / len(fft)
    return out


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2306_09497_b200 import _lib, dynamics, pint, spharm, steppers

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        comm = pint.Comm()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    for kv in args.opt:
        k, v = kv.split("=")
        _lib.set_option(k, int(v))
    B = args.slices
    grid = spharm.get_grid(M)
    cfg = steppers.StepperConfig(dt=DT, viscosity=dynamics.ViscositySpec(2, NU))
    state = make_states(grid, B, seed=rank)
    peak64, peak64_sus = fp64_peak_tflops(torch, dev, sustain_s=0.0 if args.no_extra else 4.0)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MB > L2

    for _ in range(args.warmup):
        steppers.imex_steps_inplace(state, cfg, 1)
    barrier()

    # timed region: one API step per bench step (each replays the plan's captured
    # CUDA graph of one IMEX step), queued with imex_steps_async so no host round
    # trip sits between the events; every step's convergence is still checked
    # (check_async_steps, right after its end event); L2 flushed between steps
    clocks = Clocks(local)
    total_ms = 0.0
    barrier()
    for _ in range(args.steps):
        flush.zero_()
        s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_ev.record()
        steppers.imex_steps_async(state, cfg, 1)
        e_ev.record()
        e_ev.synchronize()
        steppers.check_async_steps(grid)
        total_ms += s_ev.elapsed_time(e_ev)
    barrier()
    clk = clocks.stop()

    # profiled pass (same steps, eager launches with CUDA events per kernel class,
    # fixed-point iteration counts read back): roofline, class shares, launch count
    iters = np.zeros((1, B, 2), dtype=np.int32)
    its = []
    n_launch0 = _lib.kernel_launches()
    _lib.profile(True)
    prof_ms = 0.0
    for _ in range(args.steps):
        flush.zero_()
        s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_ev.record()
        steppers.imex_steps_inplace(state, cfg, 1, iters)
        e_ev.record()
        e_ev.synchronize()
        prof_ms += s_ev.elapsed_time(e_ev)
        its.append(iters.copy())
    _lib.profile(False)
    prof = _lib.profile_read()
    launches = _lib.kernel_launches() - n_launch0
    total_ms = max_over_ranks(total_ms)
    value = world * B * args.steps / (total_ms * 1e-3)

    # BASELINE cfg2 / cfg3 end to end, sharded over the ranks (right after the main
    # leg, before the legs that add plans, graphs and pinned buffers)
    pint_legs = {}
    if not args.no_pint:
        for name in ("cfg1", "cfg2", "cfg3"):
            pint_legs[name] = pint_leg(torch, name, comm)
            barrier()
    direct = (direct_leg(torch, steppers, cfg, state, args.steps, flush)
              if not args.no_extra and world == 1 else None)
    cor = (coriolis_legs(torch, steppers, cfg, state, min(args.steps, 5), flush)
           if not args.no_extra and world == 1 else None)

    # e2e through the public API with pinned host buffers: every step copies its
    # batch in (H2D) and its result out (D2H); steppers.HostPipeline overlaps the
    # copies of neighbouring steps with the compute of the current one
    host_in = state.data.cpu().pin_memory()
    host_out = [torch.empty_like(host_in).pin_memory() for _ in range(2)]
    host_pb = state.phibar_t.cpu().pin_memory()
    pipe = steppers.HostPipeline(grid, cfg, B)
    for i in range(2):                      # warm the pipeline's streams and buffers
        pipe.submit(host_in, host_pb, host_out[i % 2])
    pipe.flush()
    barrier()
    s_ev = torch.cuda.Event(enable_timing=True)
    s_ev.record(pipe.h2d)
    for i in range(args.steps):
        pipe.submit(host_in, host_pb, host_out[i % 2])
    e_ev = pipe.flush()
    e2e_ms = max_over_ranks(s_ev.elapsed_time(e_ev))
    e2e_value = world * B * args.steps / (e2e_ms * 1e-3)
    nbytes = host_in.numel() * host_in.element_size()
    nbytes_in = nbytes + host_pb.numel() * host_pb.element_size()

    # roofline of the dominant kernel class (device time share inside the step)
    leg_ms = prof["legendre_synthesis"][0] + prof["legendre_analysis"][0]
    leg_flops = prof["legendre_synthesis"][1] + prof["legendre_analysis"][1]
    fft_ms, fft_bytes = prof["fft_grid"][0], prof["fft_grid"][1]
    peaks = load_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    share = {k: round(v[0] / max(prof_ms, 1e-9), 4) for k, v in prof.items()}
    traffic = ncu_traffic()
    ach_l = leg_flops / (leg_ms * 1e-3) / 1e12
    roof_leg = {"kernel": "leg_synth_v3 + leg_anal_v3 (FP64 DMMA.8x8x4, parity-folded)",
                "bound": "tensor", "achieved": ach_l, "peak": peak64, "unit": "TFLOP/s",
                "frac": ach_l / peak64, "traffic": traffic.get("legendre"),
                "traffic_unit": "DRAM bytes per launch (mean of synthesis and analysis)",
                "traffic_source": traffic.get("source"),
                "peak_source": "cuBLAS DGEMM 8192^3 measured live in bench.py (burst)",
                "peak_sustained": peak64_sus,
                "frac_of_sustained": ach_l / peak64_sus if peak64_sus else None,
                "work_per_unit": "2*J*K flops per slice per Legendre term (N/S folded): "
                                 "14 terms per nonlinear evaluation, 2 evaluations per step",
                "time_share": leg_ms / max(prof_ms, 1e-9)}
    ach_f = fft_bytes / (fft_ms * 1e-3) / 1e9
    # SURVEY.md §8(d)'s executed-work figure: the 12 longitude transforms one
    # reference nonlinear evaluation runs (9 for nonlinear_advection, 3 for
    # nonlinear_rest) at J*I*8 + J*(M+1)*16 bytes each, per slice and launch
    g = grid
    b8d = 12.0 * (g.nlat * g.nlon * 8 + g.nlat * (M + 1) * 16) * B * prof["fft_grid"][2]
    ach_8d = b8d / (fft_ms * 1e-3) / 1e9
    roof_fft = {"kernel": "fft_lanes_kernel<5,16,0,696> (5x7x11 prime-factor lanes: inverse FFT, fused middle with the grid products, forward FFT)",
                "bound": "hbm", "achieved": ach_f, "peak": hbm, "unit": "GB/s",
                "frac": ach_f / hbm, "traffic": traffic.get("fft"),
                "traffic_unit": "DRAM bytes per launch", "traffic_source": traffic.get("source"),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "work_per_unit": "(7 in + 4 out) (M+1) J 16 B per slice: 7 E/O half-spectrum "
                                 "fields read, 4 F+/F- fields written",
                "binding_unit": "shared-memory / L1 data pipe (ncu "
                                "l1tex__data_pipe_lsu_wavefronts), not HBM",
                "achieved_survey_8d": ach_8d, "frac_survey_8d": ach_8d / hbm,
                "survey_8d_work": "12 transforms x (J*I*8 + J*(M+1)*16) B per slice per launch "
                                  "(the reference's rfft/irfft count of one nonlinear "
                                  "evaluation; executed-work bytes, SURVEY.md 8d)",
                "time_share": fft_ms / max(prof_ms, 1e-9)}
    # the dominant single kernel is the FFT pass; the Legendre GEMM pair is the
    # dominant kernel family and is reported alongside
    roof = roof_fft if fft_ms >= max(prof["legendre_synthesis"][0],
                                     prof["legendre_analysis"][0]) else roof_leg
    it_arr = np.concatenate(its)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (gaussian_bumps + per-slice perturbation)",
            "config": dict(workload(B), l2="256 MB buffer written between timed steps",
                           avg_fixed_point_iters=float(it_arr.mean()),
                           parallelism=f"slices: {B} per GPU x {world} GPU(s); MGRIT legs "
                                       f"shard C-slices over the {world} rank(s)"),
            "roofline": roof,
            "roofline_legendre": roof_leg, "roofline_fft": roof_fft,
            "kernel_time_share": share,
            "legendre_tflops": leg_flops / max(leg_ms, 1e-9) / 1e9,
            "fft_stage_gbs": fft_bytes / max(fft_ms, 1e-9) / 1e6,
            "fp64_peak_tflops_measured": peak64, "fp64_peak_tflops_sustained": peak64_sus,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": nbytes_in,
                    "d2h_bytes_per_step": nbytes,
                    "api": "steppers.HostPipeline (pinned host batches; H2D/D2H of "
                           "neighbouring steps overlap the current step)"},
            "gpu_launches": launches,
            "gpu_launches_note": "counted over the profiled pass (eager launches of the same "
                                 "kernels the timed pass replays as one CUDA graph per step)",
            "ms_per_step_profiled_eager": prof_ms / args.steps, "clocks": clk}
    for name, rec in pint_legs.items():
        line[f"pint_{name}"] = rec
    if direct is not None:
        line["direct_solve"] = direct
    if cor is not None:
        line["coriolis_faithful"] = cor
    if rank == 0 and world == 1 and not args.no_extra:
        line["sht_cfg4"] = sht_cfg4(torch)
        line["fine_cfg5"] = fine_cfg5(torch)
    if rank == 0 and not args.no_cpu:
        nproc = cpu_cores()
        el, done = cpu_steps(1, nproc, B)
        line["cpu_baseline"] = cpu_baseline_record(done / el, nproc, B, 1)
        if not args.no_extra:
            line["cpu_cfg1_mgrit"] = cpu_cfg1_mgrit()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def launch_ranks(args):
    """--gpus N > 1 outside torchrun: relaunch this script with one rank per GPU
    (torch.distributed.run, 127.0.0.1 rendezvous); NCCL_DEBUG=INFO (init lines,
    on stderr) shows the communicator's rank count in the log."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    # NCCL's lines on stderr, so rank 0's JSON line stays alone on stdout
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    if os.environ.get("SWE_LIB"):  # A/B of another build of the library (tools only)
        from paper_2306_09497_b200 import _lib as _l
        _l.load.__defaults__ = (os.path.abspath(os.environ["SWE_LIB"]),)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--slices", type=int, default=SLICES_PER_GPU)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline legs")
    ap.add_argument("--no-pint", action="store_true", help="skip the cfg2 / cfg3 MGRIT legs")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the cfg4 / cfg5 (M=1024), direct-solve, Coriolis and CPU-MGRIT legs")
    ap.add_argument("--opt", action="append", default=[],
                    help="library tuning switch key=value (swe_set_option), for experiments")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return launch_ranks(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
