"""CUDA tendencies and IMEX propagator vs the oracle and reference goldens.

Tolerances (fp64): tendencies 1e-11 relative to the field's max; one or more
IMEX steps 1e-10 relative sup-norm per field (the north star's bound).
"""

import dataclasses

import numpy as np
import pytest

from conftest import load_golden, rel_diff

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    import torch
    assert torch.cuda.is_available()
    from paper_2306_09497_b200 import dynamics, scenarios, spharm, steppers
    return spharm, dynamics, steppers, scenarios


def _state(mods, M, arr, phibar):
    spharm, dynamics, _, _ = mods
    grid = spharm.get_grid(M)
    return dynamics.PrognosticState.from_fields(grid, arr[0], arr[1], arr[2], [float(phibar)])


def test_tendencies_match_reference(mods):
    _, dynamics, _, _ = mods
    g = load_golden("tend_M24.npz")
    s = _state(mods, int(g["M"]), g["state"], g["phibar"])

    def check(t, ref):
        got = np.stack([x[0].cpu().numpy() for x in t])
        scale = np.abs(ref).max()
        assert np.abs(got - ref).max() <= 1e-11 * scale

    check(dynamics.linear_gravity(s), g["linear_gravity"])
    check(dynamics.linear_coriolis(s), g["linear_coriolis"])
    check(dynamics.nonlinear(s), g["nonlinear_advection"] + g["nonlinear_rest"])
    check(dynamics.full_rhs(s), g["full_rhs"])


@pytest.mark.parametrize("name", ["step_M16.npz", "step_M32.npz"])
def test_imex_steps_match_reference(mods, name):
    _, dynamics, steppers, _ = mods
    g = load_golden(name)
    M = int(g["M"])
    keys = sorted(k[:-4] for k in g if k.endswith("_cfg"))
    for key in keys:
        dt, q, nu, implicit, n = g[key + "_cfg"]
        cfg = steppers.StepperConfig(dt=float(dt),
                                     viscosity=dynamics.ViscositySpec(int(q), float(nu)),
                                     coriolis_treatment="implicit" if implicit else "explicit")
        s = _state(mods, M, g[key + "_in"], g["phibar"])
        st = steppers.propagate(steppers.StepperState(s), 0.0, float(dt) * int(n), cfg)
        out = st.current.data[0].cpu().numpy()
        assert rel_diff(out, g[key + "_out"]) < 1e-10, key
        # input untouched (steps are pure, pint.py relies on it)
        assert np.array_equal(s.data[0].cpu().numpy(), g[key + "_in"])


@pytest.mark.parametrize("path,cor", [(1, 2), (2, 2), (2, 1), (2, 0)],
                         ids=["fft_rows", "fft_lanes", "cor_legendre", "cor_fft"])
def test_batched_step_matches_oracle_per_slice(mods, path, cor):
    """Per-slice states and Coriolis fixed-point iteration counts, on both FFT kernels
    and all three Coriolis evaluations (spectral / FFT-free Legendre / FFT)."""
    from paper_2306_09497_b200 import _lib
    _lib.set_option("fft_path", path)
    _lib.set_option("fast_coriolis", cor)
    try:
        _batched_step_check(mods)
    finally:
        _lib.set_option("fft_path", 0)
        _lib.set_option("fast_coriolis", 2)


def _batched_step_check(mods):
    """B slices with different states step in lockstep; each matches its own serial run."""
    spharm, dynamics, steppers, _ = mods
    from oracle.sht import OracleSphere
    from oracle.swe import OracleState, StepCfg, imex_step, gaussian_bumps
    M = 32
    sph = OracleSphere(M)
    rng = np.random.default_rng(5)
    base = gaussian_bumps(sph)
    B = 6
    states = []
    for b in range(B):
        s = base.copy()
        # different perturbations => different fixed-point iteration counts
        amp = 10.0 ** (b - 3)
        noise = (rng.standard_normal(sph.n_modes) + 1j * rng.standard_normal(sph.n_modes))
        noise[: M + 1] = noise[: M + 1].real
        noise *= (sph.n_of + 1.0) ** -3
        s.xi = s.xi + 1e-6 * amp * noise[None]
        s.delta = s.delta + 1e-7 * amp * noise[None]
        states.append(s)
    ob = OracleState.stack(states)
    cfg_o = StepCfg(dt=240.0, visc_nu=1e5)
    stats = []
    ref = imex_step(ob, cfg_o, stats)
    grid = spharm.get_grid(M)
    gs = dynamics.PrognosticState.from_fields(grid, ob.phi, ob.xi, ob.delta, ob.phibar)
    cfg = steppers.StepperConfig(dt=240.0, viscosity=dynamics.ViscositySpec(2, 1e5))
    iters = np.zeros((1, B, 2), dtype=np.int32)
    steppers.imex_steps_inplace(gs, cfg, 1, iters)
    phi, xi, de, _ = gs.to_numpy()
    for b in range(B):
        got = np.stack([phi[b], xi[b], de[b]])
        want = np.stack([ref.phi[b], ref.xi[b], ref.delta[b]])
        assert rel_diff(got, want) < 1e-10, b
    assert np.array_equal(iters[0, :, 0], stats[0]) and np.array_equal(iters[0, :, 1], stats[1])


def test_m256_step_window(mods):
    spharm, dynamics, steppers, scenarios = mods
    g = load_golden("step_window_M256.npz")
    grid = spharm.get_grid(256)
    s = scenarios.gaussian_bumps(grid)
    cfg = steppers.StepperConfig(dt=float(g["dt"]), viscosity=dynamics.ViscositySpec(2, float(g["nu"])))
    out = steppers.imex_step(s, cfg).data[0].cpu().numpy()[:, g["sel"]]
    for f in range(3):
        assert np.abs(out[f] - g["out_window"][f]).max() <= 1e-10 * g["out_maxabs"][f]


def test_nonconvergence_raises(mods):
    _, dynamics, steppers, _ = mods
    g = load_golden("step_M16.npz")
    s = _state(mods, 16, g["bumps_dt600_nu1e5_in"], g["phibar"])
    cfg = steppers.StepperConfig(dt=600.0, implicit_max_iter=1)
    with pytest.raises(steppers.ImplicitSolveError, match="residual"):
        steppers.imex_step(s, cfg)


@pytest.mark.parametrize("M", [16, 51, 64, 256])
def test_fft_free_coriolis_equals_pseudospectral(mods, M):
    """The FFT-free Coriolis (rfft(irfft(X) * s) = s X on the band) and the spectral
    three-term recurrence (plan.cu cor_cf, the default) agree with the FFT round
    trip to roundoff, batched, on every path."""
    spharm, dynamics, _, _ = mods
    from paper_2306_09497_b200 import _lib
    from oracle.sht import OracleSphere, random_bandlimited
    grid = spharm.get_grid(M)
    rng = np.random.default_rng(M)
    sph = OracleSphere(M) if M <= 64 else None
    B = 40
    c = [random_bandlimited(grid if sph is None else sph, rng, batch=(B,)) for _ in range(3)] \
        if sph is not None else None
    if c is None:
        K = grid.n_modes
        c = []
        for _ in range(3):
            x = rng.standard_normal((B, K)) + 1j * rng.standard_normal((B, K))
            x[:, : M + 1] = x[:, : M + 1].real
            c.append(x * (grid.n_of + 1.0) ** -2)
    s = dynamics.PrognosticState.from_fields(grid, 1e3 * c[0], 1e-5 * c[1], 1e-6 * c[2],
                                             [9.80616 * 29400.0] * B)
    try:
        outs = []
        for fast in (0, 1, 2):
            _lib.set_option("fast_coriolis", fast)
            t = dynamics.linear_coriolis(s)
            outs.append(np.stack([x.cpu().numpy() for x in t]))
    finally:
        _lib.set_option("fast_coriolis", 2)
    for f in (1, 2):
        # FFT-free: same arithmetic minus the FFT pair; spectral: exact recurrence, so
        # it differs by the pseudospectral path's own quadrature roundoff (~1e-13)
        for alt, tol in ((1, 1e-13), (2, 1e-12)):
            err = np.abs(outs[0][f] - outs[alt][f]).max() / np.abs(outs[0][f]).max()
            assert err <= tol, (f, alt, err)
    if sph is not None:
        from oracle.swe import OracleState, linear_coriolis
        o = linear_coriolis(OracleState(sph, 1e3 * c[0], 1e-5 * c[1], 1e-6 * c[2],
                                        np.full(B, 9.80616 * 29400.0)))
        for f in (1, 2):
            for alt in (1, 2):
                assert np.abs(outs[alt][f] - o[f]).max() <= 1e-12 * np.abs(o[f]).max()


def test_spectral_coriolis_edge_modes(mods):
    """Inputs the pseudospectral path drops (Im of m = 0, the n = 0 modes) are
    dropped by the spectral recurrence too; m = M and n = M rows included."""
    spharm, dynamics, _, _ = mods
    from paper_2306_09497_b200 import _lib
    from oracle.sht import OracleSphere
    from oracle.swe import OracleState, linear_coriolis
    M, B = 12, 3
    grid, sph = spharm.get_grid(M), OracleSphere(M)
    rng = np.random.default_rng(7)
    c = [rng.standard_normal((B, grid.n_modes)) + 1j * rng.standard_normal((B, grid.n_modes))
         for _ in range(3)]
    s = dynamics.PrognosticState.from_fields(grid, c[0], c[1], c[2], [3e4] * B)
    o = linear_coriolis(OracleState(sph, c[0], c[1], c[2], np.full(B, 3e4)))
    try:
        for fast in (0, 1, 2):
            _lib.set_option("fast_coriolis", fast)
            t = dynamics.linear_coriolis(s)
            for f in (1, 2):
                got = t[f].cpu().numpy()
                assert np.abs(got - o[f]).max() <= 1e-12 * np.abs(o[f]).max(), (fast, f)
    finally:
        _lib.set_option("fast_coriolis", 2)


def test_host_pipeline_matches_inplace(mods):
    """HostPipeline (copies overlapped with compute) returns exactly what the
    in-place device call computes, batch by batch."""
    import torch
    spharm, dynamics, steppers, scenarios = mods
    grid = spharm.get_grid(32)
    cfg = steppers.StepperConfig(dt=240.0, viscosity=dynamics.ViscositySpec(2, 1e5))
    base = scenarios.gaussian_bumps(grid)
    rng = np.random.default_rng(3)
    B, nb = 4, 5
    hosts, outs, want = [], [], []
    for i in range(nb):
        d = base.data.repeat(B, 1, 1).cpu()
        taper = torch.from_numpy((grid.n_of + 1.0) ** -2)
        noise = torch.from_numpy(rng.standard_normal((B, grid.n_modes))) * taper
        noise[:, : grid.M + 1] = noise[:, : grid.M + 1].real
        d[:, 0] += 10.0 * noise            # geopotential perturbation, m^2/s^2
        d[:, 1] += 1e-6 * noise            # vorticity perturbation, 1/s
        hosts.append(d.pin_memory())
        outs.append(torch.empty_like(d).pin_memory())
        s = dynamics.PrognosticState(grid, d.cuda(), base.phibar_t.expand(B).contiguous())
        want.append(steppers.imex_steps_inplace(s, cfg, 2).data.cpu())
    pb = base.phibar_t.expand(B).contiguous().cpu().pin_memory()
    pipe = steppers.HostPipeline(grid, cfg, B, nsteps=2, depth=2)
    for i in range(nb):
        pipe.submit(hosts[i], pb, outs[i])
    pipe.flush()
    for i in range(nb):
        assert torch.equal(outs[i], want[i]), i


@pytest.mark.parametrize("M,B", [(51, 3), (51, 40), (256, 3), (56, 3), (100, 3), (100, 40)])
@pytest.mark.parametrize("path", [1, 2], ids=["fft_rows", "fft_lanes"])
def test_nonlinear_prime_factor_sizes(mods, M, B, path):
    """Nonlinear tendency on prime-factor FFT lengths (N2 = 77 = 7*11 at M=51,
    385 = 5*7*11 at M=256, the benchmark size) on both FFT kernels, batched,
    against the oracle.  B = 40 takes the warp-specialised synthesis, which on
    the lane kernel hands over in the pair-major layout.  M = 56 (N2 = 85 = 5*17)
    runs a generic-radix lane stage; M = 100 (N2 = 151, prime) the 8-row lane
    kernel whose nonlinear pass splits the hemispheres over a two-CTA cluster."""
    spharm, dynamics, _, _ = mods
    from paper_2306_09497_b200 import _lib
    from oracle.sht import OracleSphere, random_bandlimited
    from oracle.swe import OracleState, nonlinear_advection, nonlinear_rest
    grid, sph = spharm.get_grid(M), OracleSphere(M)
    rng = np.random.default_rng(M + path)
    c = [random_bandlimited(sph, rng, batch=(B,)) for _ in range(3)]
    phi = 3e5 * c[0]
    phi[:, 0] += 9.80616 * 29400.0 * np.sqrt(2.0)
    xi, de = 1e-5 * c[1], 1e-6 * c[2]
    pb = np.full(B, 9.80616 * 29400.0)
    o = OracleState(sph, phi, xi, de, pb)
    want = [a + b for a, b in zip(nonlinear_advection(o), nonlinear_rest(o))]
    s = dynamics.PrognosticState.from_fields(grid, phi, xi, de, pb)
    _lib.set_option("fft_path", path)
    try:
        got = dynamics.nonlinear(s)
    finally:
        _lib.set_option("fft_path", 0)
    for f in range(3):
        g = got[f].cpu().numpy()
        assert np.abs(g - want[f]).max() <= 1e-11 * np.abs(want[f]).max(), f


def test_nonlinear_m1024_lanes_match_rows(mods):
    """M = 1024 (configs 4/5): the 8-row, cluster-split lane kernel with generic
    radices 29 and 53 gives the warp-per-row kernel's nonlinear tendency."""
    spharm, dynamics, _, _ = mods
    from paper_2306_09497_b200 import _lib
    grid = spharm.get_grid(1024)
    rng = np.random.default_rng(1024)
    B = 2
    c = []
    for _ in range(3):
        x = (grid.n_of + 1.0) ** -1.5 * np.exp(2j * np.pi * rng.uniform(size=(B, grid.n_modes)))
        x[:, : grid.M + 1] = x[:, : grid.M + 1].real
        c.append(x)
    phi = 3e5 * c[0]
    phi[:, 0] += 9.80616 * 29400.0 * np.sqrt(2.0)
    s = dynamics.PrognosticState.from_fields(grid, phi, 1e-5 * c[1], 1e-6 * c[2],
                                             np.full(B, 9.80616 * 29400.0))
    got = {}
    for path in (1, 2):
        _lib.set_option("fft_path", path)
        try:
            got[path] = [t.cpu().numpy() for t in dynamics.nonlinear(s)]
        finally:
            _lib.set_option("fft_path", 0)
    for f in range(3):
        a, b = got[1][f], got[2][f]
        assert np.isfinite(b).all()
        # north_star's 1e-10 relative L-inf: the two kernels run the prime-factor
        # stages in different orders (the lane kernel ends its inverse on stage 0 for
        # the fused middle), and the delta tendency is a small difference of flux terms
        assert np.abs(b - a).max() <= 1e-10 * np.abs(a).max(), f


@pytest.mark.parametrize("M,B", [(32, 3), (51, 40)])
def test_step_graph_matches_eager(mods, M, B):
    """Replayed CUDA step graphs (fixed point as a WHILE node) give bitwise the
    eager host-driven result; first call eager, second captures, later replay."""
    spharm, dynamics, steppers, scenarios = mods
    import torch
    from paper_2306_09497_b200 import _lib
    grid = spharm.get_grid(M)
    cfg = steppers.StepperConfig(dt=240.0, viscosity=dynamics.ViscositySpec(2, 1e5))
    base = scenarios.gaussian_bumps(grid, batch=B)
    rng = np.random.default_rng(M)
    taper = torch.from_numpy((grid.n_of + 1.0) ** -2).cuda()
    noise = torch.from_numpy(rng.standard_normal((B, grid.n_modes))).cuda() * taper
    noise[:, : M + 1] = noise[:, : M + 1].real
    base.data[:, 1] += 1e-6 * noise
    outs = {}
    for graphs in (0, 1):
        _lib.set_option("graphs", graphs)
        try:
            s = base.copy()
            for _ in range(4):
                steppers.imex_steps_inplace(s, cfg, 2)
            outs[graphs] = s.data.cpu()
        finally:
            _lib.set_option("graphs", 1)
    assert torch.equal(outs[0], outs[1])


def test_step_graph_nonconvergence_raises(mods):
    """An unconverged fixed point inside a replayed graph is caught on the device
    and re-run on the host path, raising ImplicitSolveError with the residual."""
    _, dynamics, steppers, _ = mods
    g = load_golden("step_M16.npz")
    s = _state(mods, 16, g["bumps_dt600_nu1e5_in"], g["phibar"])
    cfg = steppers.StepperConfig(dt=600.0, implicit_max_iter=1)
    for _ in range(3):
        with pytest.raises(steppers.ImplicitSolveError, match="residual"):
            steppers.imex_step(s, cfg)


def test_async_steps_match_inplace_and_report_nonconvergence(mods):
    """swe_imex_step_async (queued graph replays, no per-call host check) gives the
    synchronous call's states bitwise; an unconverged solve is reported by
    check_async_steps and leaves the queued states untouched."""
    spharm, dynamics, steppers, scenarios = mods
    import torch
    grid = spharm.get_grid(32)
    cfg = steppers.StepperConfig(dt=480.0, viscosity=dynamics.ViscositySpec(2, 1e5))
    s0 = scenarios.gaussian_bumps(grid, batch=3)
    want = s0.copy()
    for _ in range(3):
        steppers.imex_steps_inplace(want, cfg, 2)
    got = s0.copy()
    for _ in range(3):
        steppers.imex_steps_async(got, cfg, 2)
    steppers.check_async_steps(grid)
    assert torch.equal(got.data, want.data)
    bad = dataclasses.replace(cfg, implicit_max_iter=1)
    before = s0.data.clone()
    with pytest.raises(steppers.ImplicitSolveError):
        steppers.imex_steps_async(s0.copy(), bad, 1)  # first sight of the key: eager, raises
    x = s0.copy()
    y = s0.copy()
    steppers.imex_steps_async(x, bad, 1)   # graph replay: queued
    steppers.imex_steps_async(y, cfg, 1)   # queued after the failure: left untouched
    with pytest.raises(steppers.ImplicitSolveError):
        steppers.check_async_steps(grid)
    torch.cuda.synchronize()
    assert torch.equal(x.data, before) and torch.equal(y.data, before)
    steppers.check_async_steps(grid)       # the flag was reset


@pytest.mark.parametrize("M,B,dt", [(32, 3, 480.0), (64, 16, 240.0), (256, 32, 60.0)])
def test_strided_out_of_place_step_matches_inplace(mods, M, B, dt):
    """swe_imex_step_async_io: every 2nd point of a level array stepped into its
    neighbour (the MGRIT F-sweep without gather / scatter copies), in place, and into
    a separate tensor: bitwise the in-place step of the gathered slices; untouched
    points stay untouched; bad views are refused."""
    spharm, dynamics, steppers, scenarios = mods
    import torch
    grid = spharm.get_grid(M)
    cfg = steppers.StepperConfig(dt=dt, viscosity=dynamics.ViscositySpec(2, 1e5))
    s0 = scenarios.gaussian_bumps(grid, batch=B)
    rng = np.random.default_rng(5)
    s0.data[:, 1] *= torch.from_numpy(1.0 + 1e-3 * rng.standard_normal((B, 1))).cuda()
    want = s0.copy()
    steppers.imex_steps_inplace(want, cfg, 1)
    for _ in range(2):  # first sight runs eager, the second call replays the step graph
        u = torch.full((2 * B + 1, 3, grid.n_modes), 7.0 + 0j, dtype=torch.complex128, device="cuda")
        u[0:2 * B:2] = s0.data
        steppers.imex_step_async_io(grid, u[0:2 * B:2], u[1:2 * B + 1:2], s0.phibar_t, cfg)
        steppers.check_async_steps(grid)
        assert torch.equal(u[1:2 * B + 1:2], want.data)
        assert torch.equal(u[0:2 * B:2], s0.data) and bool((u[2 * B] == 7.0).all())
        out = torch.empty_like(s0.data)
        steppers.imex_step_async_io(grid, u[0:2 * B:2], out, s0.phibar_t, cfg)
        v = s0.data.clone()
        steppers.imex_step_async_io(grid, v, v, s0.phibar_t, cfg)  # in place, packed
        steppers.check_async_steps(grid)
        assert torch.equal(out, want.data) and torch.equal(v, want.data)
    with pytest.raises(ValueError):
        steppers.imex_step_async_io(grid, u[0:2 * B:2].transpose(1, 2), out, s0.phibar_t, cfg)
    with pytest.raises(ValueError):
        steppers.imex_step_async_io(grid, u[0:2 * B:2], out[:-1], s0.phibar_t, cfg)


def test_step_graph_nonconvergence_keeps_input(mods):
    """In place: a replayed step graph whose fixed point does not converge leaves the
    caller's state untouched (the layout kernel is skipped on the device flag) so the
    host-driven rerun starts from the true input and raises like the reference."""
    _, dynamics, steppers, _ = mods
    import torch
    g = load_golden("step_M16.npz")
    cfg = steppers.StepperConfig(dt=600.0, implicit_max_iter=1)
    for call in range(3):  # eager, capture, replay
        s = _state(mods, 16, g["bumps_dt600_nu1e5_in"], g["phibar"])
        before = s.data.clone()
        with pytest.raises(steppers.ImplicitSolveError, match="residual"):
            steppers.imex_steps_inplace(s, cfg, 1)
        torch.cuda.synchronize()
        assert torch.equal(s.data, before), f"call {call}: input modified by a failed step"


@pytest.mark.parametrize("M", [32, 51, 256])
def test_fft_kernel_variants_bitwise(mods, M):
    """The radix-specialised nonlinear lane kernels (49 = 7x7, 77 = 7x11, 385 = 5x7x11),
    their fused middle (inverse and forward stage 0 with the grid products on
    registers, fft_rm=2) and the L2 prefetch of the E/O blocks give bitwise the
    generic kernel's step."""
    spharm, dynamics, steppers, scenarios = mods
    import torch
    from paper_2306_09497_b200 import _lib
    grid = spharm.get_grid(M)
    cfg = steppers.StepperConfig(dt=120.0, viscosity=dynamics.ViscositySpec(2, 1e5))
    outs = {}
    try:
        for rm, pf in ((0, 0), (1, 0), (1, 2), (2, 0), (2, 2)):
            _lib.set_option("fft_rm", rm)
            _lib.set_option("fft_pf", pf)
            s = scenarios.gaussian_bumps(grid, batch=4)
            steppers.imex_steps_inplace(s, cfg, 2)
            outs[(rm, pf)] = s.data.cpu()
    finally:
        _lib.set_option("fft_rm", 2)
        _lib.set_option("fft_pf", 2)
    for key in ((1, 0), (1, 2), (2, 0), (2, 2)):
        assert torch.equal(outs[(0, 0)], outs[key]), key


def test_tiled_fixed_point_matches_untiled(mods):
    """The shared-memory-tiled fixed-point kernel (batches >= 32) matches the
    gather kernel: same iteration counts, states to roundoff."""
    spharm, dynamics, steppers, scenarios = mods
    import torch
    from paper_2306_09497_b200 import _lib
    M, B = 51, 40
    grid = spharm.get_grid(M)
    cfg = steppers.StepperConfig(dt=240.0, viscosity=dynamics.ViscositySpec(2, 1e5))
    base = scenarios.gaussian_bumps(grid, batch=B)
    rng = np.random.default_rng(4)
    taper = torch.from_numpy((grid.n_of + 1.0) ** -2).cuda()
    noise = torch.from_numpy(rng.standard_normal((B, grid.n_modes))).cuda() * taper
    noise[:, : M + 1] = noise[:, : M + 1].real
    base.data[:, 1] += 1e-6 * noise
    base.data[:, 2] += 1e-7 * noise
    outs, its = {}, {}
    for tiled in (0, 1):
        _lib.set_option("helm_tiled", tiled)
        try:
            s = base.copy()
            it = np.zeros((3, B, 2), dtype=np.int32)
            steppers.imex_steps_inplace(s, cfg, 3, it)
            outs[tiled], its[tiled] = s.data.cpu().numpy(), it
        finally:
            _lib.set_option("helm_tiled", 1)
    assert np.array_equal(its[0], its[1])
    for b in range(B):
        assert rel_diff(outs[1][b], outs[0][b]) < 1e-13, b


@pytest.mark.parametrize("M,B", [(100, 3), (256, 3), (256, 40)])
@pytest.mark.parametrize("graphs", [0, 1])
def test_cluster_half_step_matches_multikernel(mods, M, B, graphs):
    """The one-cluster-per-slice Crank-Nicolson half step (whole fixed point in
    distributed shared memory) gives the multi-kernel path's iteration counts and
    states (M = 100: 3-CTA clusters, M = 256: 16-CTA clusters)."""
    spharm, dynamics, steppers, scenarios = mods
    import torch
    from paper_2306_09497_b200 import _lib
    grid = spharm.get_grid(M)
    cfg = steppers.StepperConfig(dt=240.0, viscosity=dynamics.ViscositySpec(2, 1e5))
    base = scenarios.gaussian_bumps(grid, batch=B)
    rng = np.random.default_rng(M + B)
    taper = torch.from_numpy((grid.n_of + 1.0) ** -2).cuda()
    noise = torch.from_numpy(rng.standard_normal((B, grid.n_modes))).cuda() * taper
    noise[:, : M + 1] = noise[:, : M + 1].real
    base.data[:, 1] += 1e-6 * noise
    base.data[:, 2] += 1e-7 * noise
    outs, its = {}, {}
    _lib.set_option("graphs", graphs)
    try:
        for cl in (0, 2):
            _lib.set_option("cn_cluster", cl)
            s = base.copy()
            it = np.zeros((3, B, 2), dtype=np.int32)
            steppers.imex_steps_inplace(s, cfg, 3, None if graphs else it)
            outs[cl], its[cl] = s.data.cpu().numpy(), it
    finally:
        _lib.set_option("cn_cluster", 1)
        _lib.set_option("graphs", 1)
    assert np.array_equal(its[0], its[2])
    for b in range(B):
        assert rel_diff(outs[2][b], outs[0][b]) < 1e-13, b


@pytest.mark.parametrize("M,B", [(16, 1), (51, 1), (51, 40)])
@pytest.mark.parametrize("graphs", [0, 1])
def test_coarse_half_step_variants_agree(mods, M, B, graphs):
    """Coarse levels: the shared-memory-resident half step (one CTA per slice, rhs in
    shared memory; the default), the one-CTA k_cn_small and the multi-kernel path
    give the same iteration counts and states."""
    spharm, dynamics, steppers, scenarios = mods
    import torch
    from paper_2306_09497_b200 import _lib
    grid = spharm.get_grid(M)
    cfg = steppers.StepperConfig(dt=480.0, viscosity=dynamics.ViscositySpec(2, 1e5))
    base = scenarios.gaussian_bumps(grid, batch=B)
    rng = np.random.default_rng(M * B)
    taper = torch.from_numpy((grid.n_of + 1.0) ** -2).cuda()
    noise = torch.from_numpy(rng.standard_normal((B, grid.n_modes))).cuda() * taper
    noise[:, : M + 1] = noise[:, : M + 1].real
    base.data[:, 1] += 1e-6 * noise
    base.data[:, 2] += 1e-7 * noise
    outs, its = {}, {}
    _lib.set_option("graphs", graphs)
    try:
        for name, cl, sm in (("cluster", 1, 1), ("small", 0, 1), ("multi", 0, 0)):
            _lib.set_option("cn_cluster", cl)
            _lib.set_option("cn_small", sm)
            s = base.copy()
            it = np.zeros((3, B, 2), dtype=np.int32)
            steppers.imex_steps_inplace(s, cfg, 3, None if graphs else it)
            outs[name], its[name] = s.data.cpu().numpy(), it
    finally:
        _lib.set_option("cn_cluster", 1)
        _lib.set_option("cn_small", 1)
        _lib.set_option("graphs", 1)
    for name in ("small", "multi"):
        assert np.array_equal(its[name], its["cluster"]), name
        for b in range(B):
            assert rel_diff(outs[name][b], outs["cluster"][b]) < 1e-13, (name, b)


@pytest.mark.parametrize("M,B", [(256, 40), (101, 6), (64, 33)])
@pytest.mark.parametrize("graphs", [0, 1])
def test_fused_fixed_point_matches_multikernel(mods, M, B, graphs):
    """The speculative shared-memory fixed point (k_cn_fused: guessed iteration count,
    per-iteration maxima, recompute of early-converged slices, k_helm_tiled loop for
    late ones) gives the multi-kernel path's iteration counts and bitwise states.
    The dt sequence moves the guess above and below the true count (5 <-> 9)."""
    spharm, dynamics, steppers, scenarios = mods
    import torch
    from paper_2306_09497_b200 import _lib
    grid = spharm.get_grid(M)
    base = scenarios.gaussian_bumps(grid, batch=B)
    rng = np.random.default_rng(M + 7 * B)
    taper = torch.from_numpy((grid.n_of + 1.0) ** -2).cuda()
    noise = torch.from_numpy(rng.standard_normal((B, grid.n_modes))).cuda() * taper
    noise[:, : M + 1] = noise[:, : M + 1].real
    base.data[:, 1] += 1e-6 * noise
    base.data[:, 2] += 1e-7 * noise
    outs, its = {}, {}
    _lib.set_option("graphs", graphs)
    _lib.set_option("cn_cluster", 0)
    try:
        for fused in (0, 1):
            _lib.set_option("cn_fused", fused)
            s = base.copy()
            seq = []
            for dt in (60.0, 960.0, 60.0, 240.0):
                cfg = steppers.StepperConfig(dt=dt, viscosity=dynamics.ViscositySpec(2, 1e5))
                it = np.zeros((2, B, 2), dtype=np.int32)
                steppers.imex_steps_inplace(s, cfg, 2, None if graphs else it)
                seq.append(it)
            outs[fused], its[fused] = s.data.cpu().numpy(), np.stack(seq)
    finally:
        _lib.set_option("cn_fused", 1)
        _lib.set_option("cn_cluster", 1)
        _lib.set_option("graphs", 1)
    assert np.array_equal(its[0], its[1])
    assert np.array_equal(outs[0], outs[1])


def test_fused_fixed_point_nonconvergence_raises(mods):
    """max_iter below the needed count on the fused path raises ImplicitSolveError
    with the residual, eager and under graphs."""
    spharm, dynamics, steppers, scenarios = mods
    from paper_2306_09497_b200 import _lib
    grid = spharm.get_grid(256)
    s = scenarios.gaussian_bumps(grid, batch=36)
    _lib.set_option("cn_cluster", 0)
    try:
        for mi in (1, 2):
            cfg = steppers.StepperConfig(dt=600.0, implicit_max_iter=mi)
            for _ in range(3):
                with pytest.raises(steppers.ImplicitSolveError, match="residual"):
                    steppers.imex_step(s, cfg)
    finally:
        _lib.set_option("cn_cluster", 1)


def test_cluster_half_step_nonconvergence_raises(mods):
    """An unconverged fixed point on the cluster path raises ImplicitSolveError
    with the residual (eager and under graphs)."""
    spharm, dynamics, steppers, scenarios = mods
    from paper_2306_09497_b200 import _lib
    grid = spharm.get_grid(256)
    s = scenarios.gaussian_bumps(grid, batch=2)
    cfg = steppers.StepperConfig(dt=600.0, implicit_max_iter=1)
    _lib.set_option("cn_cluster", 2)
    try:
        for _ in range(3):
            with pytest.raises(steppers.ImplicitSolveError, match="residual"):
                steppers.imex_step(s, cfg)
    finally:
        _lib.set_option("cn_cluster", 1)


@pytest.mark.parametrize("M,B,dt", [(32, 6, 240.0), (51, 40, 960.0), (256, 3, 60.0), (256, 64, 60.0)])
def test_direct_implicit_solve_matches_fixed_point(mods, M, B, dt):
    """implicit_solver="direct" (per-m tridiagonal solve of (I - a L) U = R, SURVEY.md
    §8f row 4) agrees with the reference fixed point converged to tol = 1e-12."""
    spharm, dynamics, steppers, scenarios = mods
    import dataclasses
    import torch
    grid = spharm.get_grid(M)
    cfg = steppers.StepperConfig(dt=dt, viscosity=dynamics.ViscositySpec(2, 1e5))
    base = scenarios.gaussian_bumps(grid, batch=B)
    rng = np.random.default_rng(M + B)
    taper = torch.from_numpy((grid.n_of + 1.0) ** -2).cuda()
    noise = torch.from_numpy(rng.standard_normal((B, grid.n_modes))
                             + 1j * rng.standard_normal((B, grid.n_modes))).cuda() * taper
    noise[:, : M + 1] = noise[:, : M + 1].real
    base.data[:, 1] += 1e-6 * noise
    base.data[:, 2] += 1e-7 * noise
    out = {}
    for solver in ("fixed_point", "direct"):
        s = base.copy()
        it = np.zeros((4, B, 2), dtype=np.int32)
        steppers.imex_steps_inplace(s, dataclasses.replace(cfg, implicit_solver=solver), 4, it)
        out[solver] = (s.data.cpu().numpy(), it)
    a, ia = out["fixed_point"]
    d, idd = out["direct"]
    assert (ia > 0).all() and (idd == 0).all()
    for b in range(B):
        for f in range(3):
            ref = a[b, f] - (a[b, f, 0] if f == 0 else 0.0)   # Phi': the mean mode dominates Phi
            got = d[b, f] - (d[b, f, 0] if f == 0 else 0.0)
            assert np.abs(got - ref).max() <= 1e-11 * np.abs(ref).max(), (b, f)


def test_direct_implicit_solve_matches_oracle(mods):
    """The direct solve against the oracle's fixed-point step (6 slices at different
    perturbation levels, the per-slice oracle check of the batched step)."""
    spharm, dynamics, steppers, _ = mods
    from oracle.sht import OracleSphere
    from oracle.swe import StepCfg, imex_step, gaussian_bumps, OracleState
    M = 32
    sph = OracleSphere(M)
    rng = np.random.default_rng(5)
    base = gaussian_bumps(sph)
    states = []
    for b in range(6):
        s = base.copy()
        noise = (rng.standard_normal(sph.n_modes) + 1j * rng.standard_normal(sph.n_modes))
        noise[: M + 1] = noise[: M + 1].real
        noise *= (sph.n_of + 1.0) ** -3
        s.xi = s.xi + 1e-6 * 10.0 ** (b - 3) * noise[None]
        s.delta = s.delta + 1e-7 * 10.0 ** (b - 3) * noise[None]
        states.append(s)
    ob = OracleState.stack(states)
    ref = imex_step(ob, StepCfg(dt=240.0, visc_nu=1e5), [])
    grid = spharm.get_grid(M)
    gs = dynamics.PrognosticState.from_fields(grid, ob.phi, ob.xi, ob.delta, ob.phibar)
    cfg = steppers.StepperConfig(dt=240.0, viscosity=dynamics.ViscositySpec(2, 1e5),
                                 implicit_solver="direct")
    steppers.imex_steps_inplace(gs, cfg, 1)
    phi, xi, de, _ = gs.to_numpy()
    for b in range(6):
        got = np.stack([phi[b], xi[b], de[b]])
        want = np.stack([ref.phi[b], ref.xi[b], ref.delta[b]])
        assert rel_diff(got, want) < 1e-10, b


def test_direct_implicit_solve_settls(mods):
    """The SETTLS implicit solve (given right-hand side) through the direct solver."""
    spharm, dynamics, steppers, scenarios = mods
    import dataclasses
    grid = spharm.get_grid(51)
    cfg = steppers.StepperConfig(scheme=steppers.SL_SI_SETTLS, dt=960.0,
                                 viscosity=dynamics.ViscositySpec(2, 1e5))
    s0 = scenarios.gaussian_bumps(grid, batch=2)
    out = {}
    for solver in ("fixed_point", "direct"):
        st = steppers.StepperState(s0.copy())
        for _ in range(3):
            st = steppers.advance(st, dataclasses.replace(cfg, implicit_solver=solver))
        out[solver] = st.current.data.cpu().numpy()
    a, d = out["fixed_point"], out["direct"]
    for f in range(3):
        ref = a[:, f] - (a[:, f, :1] if f == 0 else 0.0)
        got = d[:, f] - (d[:, f, :1] if f == 0 else 0.0)
        assert np.abs(got - ref).max() <= 1e-11 * np.abs(ref).max(), f


@pytest.mark.parametrize("B", [65, 130])
def test_odd_and_wide_batches_match_single_slice(mods, B):
    """M=256 batches past the 64/128-column GEMM tiles and the 32-slice CN tiles
    (odd remainders): selected slices equal their own single-slice steps (which
    take the small-batch kernels and the per-slice cluster half step) with the
    same fixed-point iteration counts."""
    spharm, dynamics, steppers, scenarios = mods
    import torch
    M = 256
    grid = spharm.get_grid(M)
    cfg = steppers.StepperConfig(dt=60.0, viscosity=dynamics.ViscositySpec(2, 1e5))
    base = scenarios.gaussian_bumps(grid, batch=B)
    rng = np.random.default_rng(B)
    taper = torch.from_numpy((grid.n_of + 1.0) ** -2).cuda()
    noise = torch.from_numpy(rng.standard_normal((B, grid.n_modes))).cuda() * taper
    noise[:, : M + 1] = noise[:, : M + 1].real
    base.data[:, 1] += 1e-6 * noise
    base.data[:, 2] += 1e-7 * noise
    s = base.copy()
    it = np.zeros((2, B, 2), dtype=np.int32)
    steppers.imex_steps_inplace(s, cfg, 2, it)
    got = s.data.cpu().numpy()
    for b in (0, 31, 32, B // 2, B - 1):
        one = dynamics.PrognosticState(grid, base.data[b:b + 1].clone(), base.phibar_t[b:b + 1].clone())
        it1 = np.zeros((2, 1, 2), dtype=np.int32)
        steppers.imex_steps_inplace(one, cfg, 2, it1)
        assert np.array_equal(it1[:, 0], it[:, b]), b
        assert rel_diff(one.data[0].cpu().numpy(), got[b]) < 1e-12, b


@pytest.mark.parametrize("implicit,nonlin", [(True, False), (False, False)])
def test_linear_only_steps_match_oracle(mods, implicit, nonlin):
    """include_nonlinear=False (linear dynamics only, steppers.py:121-140), with the
    Coriolis term implicit or explicit, against the oracle step."""
    spharm, dynamics, steppers, _ = mods
    from oracle.sht import OracleSphere
    from oracle.swe import StepCfg, imex_step, gaussian_bumps
    M, B = 32, 2
    sph = OracleSphere(M)
    s0 = gaussian_bumps(sph, batch=B)
    s0.xi[1] += 1e-6 * (sph.n_of + 1.0) ** -2
    tr = "implicit" if implicit else "explicit"
    ref = imex_step(s0, StepCfg(dt=240.0, visc_nu=1e5, coriolis_treatment=tr,
                                include_nonlinear=nonlin), [])
    grid = spharm.get_grid(M)
    st = dynamics.PrognosticState.from_fields(grid, s0.phi, s0.xi, s0.delta, s0.phibar)
    cfg = steppers.StepperConfig(dt=240.0, viscosity=dynamics.ViscositySpec(2, 1e5),
                                 coriolis_treatment=tr, include_nonlinear=nonlin)
    out = steppers.imex_step(st, cfg)
    phi, xi, de, _ = out.to_numpy()
    for b in range(B):
        got = np.stack([phi[b], xi[b], de[b]])
        want = np.stack([ref.phi[b], ref.xi[b], ref.delta[b]])
        assert rel_diff(got, want) < 1e-10, b


@pytest.mark.parametrize("M,dt,B,nsteps", [(256, 60.0, 64, 2), (51, 120.0, 64, 2)])
def test_headline_path_full_state_matches_oracle(mods, M, dt, B, nsteps):
    """The bench's default path (M=256 x 64 slices: v3 DMMA GEMMs, the 16-row lane
    FFT, k_cn_fused + its WHILE-node graph; M=51 x 64: the coarse-level path) against
    the oracle's imex_step on full states: 4 slices spread over the batch, every
    field and Phi' to 1e-10 relative sup-norm, identical fixed-point iteration
    counts, and the graph replay bitwise equal to the eager launches."""
    spharm, dynamics, steppers, scenarios = mods
    import torch
    from oracle.sht import OracleSphere
    from oracle.swe import OracleState, StepCfg, imex_step as o_step
    grid = spharm.get_grid(M)
    cfg = steppers.StepperConfig(dt=dt, viscosity=dynamics.ViscositySpec(2, 1e5))
    base = scenarios.gaussian_bumps(grid, batch=B)
    rng = np.random.default_rng(M)
    taper = torch.from_numpy((grid.n_of + 1.0) ** -2).cuda()
    noise = torch.from_numpy(rng.standard_normal((B, grid.n_modes))
                             + 1j * rng.standard_normal((B, grid.n_modes))).cuda() * taper
    noise[:, : M + 1] = noise[:, : M + 1].real
    amp = torch.logspace(-9, -5, B, dtype=torch.float64).cuda()[:, None]
    base.data[:, 1] += amp * noise
    base.data[:, 2] += 0.1 * amp * noise
    # eager launches with iteration counts, then the graph path (the second call with
    # the same key captures, the third replays)
    eager = base.copy()
    its = np.zeros((nsteps, B, 2), dtype=np.int32)
    steppers.imex_steps_inplace(eager, cfg, nsteps, its)
    for _ in range(2):
        graph = base.copy()
        steppers.imex_steps_inplace(graph, cfg, nsteps)
    assert torch.equal(graph.data, eager.data)
    got = graph.data.cpu().numpy()
    pick = [0, B // 3, 2 * B // 3, B - 1]
    sph = OracleSphere(M)
    x = base.data[pick].cpu().numpy()
    s = OracleState(sph, x[:, 0].copy(), x[:, 1].copy(), x[:, 2].copy(),
                    base.phibar_t[pick].cpu().numpy())
    o_its = []
    for k in range(nsteps):
        stats = []
        s = o_step(s, StepCfg(dt=dt, visc_nu=1e5), stats)
        o_its.append(np.stack(stats, axis=-1))
    assert np.array_equal(its[:, pick], np.stack(o_its)), (its[:, pick], o_its)
    worst = 0.0
    for j, b in enumerate(pick):
        want = np.stack([s.phi[j], s.xi[j], s.delta[j]])
        d = rel_diff(got[b], want)
        pa, pw = got[b][0].copy(), want[0].copy()
        pa[0] = pw[0] = 0.0
        dp = float(np.abs(pa - pw).max() / np.abs(pw).max())
        worst = max(worst, d, dp)
        assert d < 1e-10 and dp < 1e-10, (b, d, dp)
    print(f"[PARITY] M={M} B={B} default path vs oracle: worst {worst:.2e}, "
          f"iterations {sorted(set(its.ravel().tolist()))}")


def test_m1024_step_window_matches_reference(mods):
    """cfg5's fine step (M=1024, dt=2 s, nu=0, gaussian_bumps) on the
    default path against the REFERENCE's own step (oracle/make_golden.py m1024) on
    the modes n <= 64, per field relative to the field's max."""
    spharm, dynamics, steppers, scenarios = mods
    g = load_golden("step_window_M1024.npz")
    grid = spharm.get_grid(1024)
    s = scenarios.gaussian_bumps(grid, batch=2)
    cfg = steppers.StepperConfig(dt=float(g["dt"]),
                                 viscosity=dynamics.ViscositySpec(2, float(g["nu"])))
    steppers.imex_steps_inplace(s, cfg, 1)
    full = s.data[0].cpu().numpy()
    out = full[:, g["sel"]]
    worst = 0.0
    for f in range(3):
        mx = float(np.abs(full[f]).max())
        assert abs(mx - g["out_maxabs"][f]) <= 1e-10 * g["out_maxabs"][f], f
        e = np.abs(out[f] - g["out_window"][f]).max() / g["out_maxabs"][f]
        worst = max(worst, e)
        assert e <= 1e-10, (f, e)
    print(f"[PARITY] M=1024 cfg5 step vs reference (n <= 64): worst {worst:.2e}")
