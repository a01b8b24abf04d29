/* swe_b200.h -- C ABI of the B200 fine-propagator library (libswe_b200.so).
 *
 * Drop-in boundary for the hot path of the reference `pintswe` package
 * (/root/reference/pkg/src/pintswe).  The reference has no FFI: its engine
 * talks to a duck-typed Python problem object (pint.py:10-13, SweProblem
 * pint.py:157-194) backed by SphereGrid (spharm.py:146-343) and the IMEX
 * stepper (steppers.py:155-168).  Every entry point below replaces one of
 * those Python calls; the Python mirror in paper_2306_09497_b200/ binds them
 * with ctypes (INTEGRATION.md shows the binding).
 *
 * Conventions
 *  - All array arguments are DEVICE pointers owned by the caller.
 *  - Spectral data: complex128 interleaved (re, im), packed m-major layout of
 *    spharm.py:149-173 (block m holds n = m..M), shape [batch][K] or, for
 *    prognostic states, [batch][3][K] with fields (Phi total, xi, delta).
 *  - Grid data: float64 [batch][nlat][nlon], latitudes north to south.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream); calls are
 *    stream-ordered and use the plan's workspace, so one plan must not be used
 *    from two streams concurrently.
 *  - Return codes: SWE_OK 0; SWE_ESHAPE 1 (ValueError in the reference);
 *    SWE_ENOCONV 2 (ImplicitSolveError, steppers.py:113-118); SWE_ENONFINITE 3;
 *    SWE_ECUDA 4; SWE_ENCCL 5.  swe_last_error() returns the message.
 */
#ifndef SWE_B200_H
#define SWE_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define SWE_OK 0
#define SWE_ESHAPE 1
#define SWE_ENOCONV 2
#define SWE_ENONFINITE 3
#define SWE_ECUDA 4
#define SWE_ENCCL 5

typedef struct swe_plan swe_plan;

/* Mirror of StepperConfig (steppers.py:31-50) for scheme="imex". */
typedef struct {
  double dt;               /* > 0 */
  int visc_order;          /* ViscositySpec.order_q (even >= 2), dynamics.py:107-118 */
  double visc_nu;          /* ViscositySpec.coeff_nu (>= 0) */
  int coriolis_implicit;   /* 1: "implicit" (default), 0: "explicit" */
  int include_nonlinear;   /* 1 (default) */
  double implicit_tol;     /* 1e-12 */
  int implicit_max_iter;   /* 200 */
  int implicit_solver;     /* 0: the reference fixed point (default); 1: direct per-m
                              tridiagonal solve of the same system,
                              no iterations (iters_out = 0), never SWE_ENOCONV */
  int select_batch;        /* 0 (default): kernels chosen for `batch`; n > 0: chosen as for
                              a batch of n slices, whatever `batch` is.  A slice's result
                              is bitwise a function of (its input, select_batch) only, so a
                              sharded engine that passes the GLOBAL slice count reproduces
                              the one-rank trace bitwise (SPEC.md:330 worker invariance) */
} swe_stepper_cfg;

/* sizeof(swe_stepper_cfg) as compiled into the library: bindings check it
 * against their own struct before the first call (the struct is passed by
 * pointer, so a short binding struct would be read past its end). */
int swe_stepper_cfg_size(void);

/* SphereGrid(Truncation.for_wavenumber(M), SphereGeometry(a, omega, g))
 * -- spharm.py:154-202, get_grid spharm.py:346-349. */
int swe_plan_create(int M, double radius_a, double omega, double gravity_g, int device,
                    swe_plan **out);
void swe_plan_destroy(swe_plan *plan);
/* nlat, nlon, n_modes (spharm.py:61-72); all outputs nullable */
int swe_plan_info(const swe_plan *plan, int *nlat, int *nlon, int *nmodes);
/* Gaussian nodes mu (decreasing) and weights, HOST arrays of nlat (spharm.py:75-108) */
int swe_plan_grid(const swe_plan *plan, double *mu, double *weights);
/* bytes of device memory held by tables (+ current workspace) */
long long swe_plan_bytes(const swe_plan *plan);

/* SphereGrid.synthesis (spharm.py:249-257): spec [batch][K] -> grid [batch][nlat][nlon] */
int swe_synthesis(swe_plan *plan, const double *spec, double *grid, int batch, void *stream);
/* SphereGrid.analysis (spharm.py:238-247): grid -> spec */
int swe_analysis(swe_plan *plan, const double *grid, double *spec, int batch, void *stream);
/* SphereGrid._synthesis_pair (spharm.py:259-267): sum_m (P cp_m + H ch_m) e^{i m lambda};
 * cp, ch [batch][K] -> grid [batch][nlat][nlon] */
int swe_synthesis_pair(swe_plan *plan, const double *cp, const double *ch, double *grid,
                       int batch, void *stream);
/* SphereGrid.grad_grid (spharm.py:282-294): gx = d/dlambda / (a cos), gy = d/dtheta / a */
int swe_grad_grid(swe_plan *plan, const double *spec, double *gx, double *gy, int batch,
                  void *stream);
/* SphereGrid.uv_from_vortdiv (spharm.py:296-313) */
int swe_uv_from_vortdiv(swe_plan *plan, const double *xi, const double *delta, double *u,
                        double *v, int batch, void *stream);
/* SphereGrid.vortdiv_from_uv (spharm.py:315-343) */
int swe_vortdiv_from_uv(swe_plan *plan, const double *u, const double *v, double *xi,
                        double *delta, int batch, void *stream);

/* Tendencies of a state batch (dynamics.py:121-165).  kind:
 *   0 linear_gravity, 1 linear_coriolis, 2 nonlinear_advection + nonlinear_rest,
 *   3 full_rhs, 4 nonlinear_advection, 5 nonlinear_rest.
 *   state/out: [batch][3][K]; phibar: [batch] (device). */
int swe_tendency(swe_plan *plan, int kind, const double *state, const double *phibar,
                 double *out, int batch, void *stream);

/* `nsteps` IMEX steps (steppers.py:155-168, advance :215-222) of every slice,
 * in place on state [batch][3][K]; phibar [batch] (device).
 * iters_out (HOST, nullable): [nsteps][batch][2] fixed-point iterations of the
 * two Crank-Nicolson solves.  resid_out (HOST, nullable): [batch] residual of
 * slices that hit implicit_max_iter (SWE_ENOCONV). */
int swe_imex_step(swe_plan *plan, double *state, const double *phibar, int batch,
                  const swe_stepper_cfg *cfg, int nsteps, int *iters_out, double *resid_out,
                  void *stream);

/* swe_imex_step without the per-call host check (graph replay path): enqueues
 * the layout conversion, nsteps step-graph launches and the result on `stream` and
 * returns at once, so back-to-back calls keep the device busy (the pipelined
 * host-batch API, steppers.HostPipeline).  An unconverged Coriolis solve raises a
 * per-plan device flag instead of returning SWE_ENOCONV; while it is up, queued
 * calls leave their state untouched.  Read (and optionally reset) it with
 * swe_plan_status.  Configurations without a step graph run swe_imex_step. */
int swe_imex_step_async(swe_plan *plan, double *state, const double *phibar, int batch,
                        const swe_stepper_cfg *cfg, int nsteps, void *stream);
/* swe_imex_step_async out of place on strided slices: slice b is read at
 * in + 2 * b * in_stride doubles and its result written at out + 2 * b * out_stride
 * (strides in complex elements, >= 3 K; every slice [3][K] contiguous).  The MGRIT
 * sweeps (pint.py:223-263) step every m-th point of the level array into its
 * neighbour: with this entry they need no gather / scatter copies.  `out` may
 * equal `in`; otherwise the output slices must not overlap the input slices. */
int swe_imex_step_async_io(swe_plan *plan, const double *in, long long in_stride, double *out,
                           long long out_stride, const double *phibar, int batch,
                           const swe_stepper_cfg *cfg, int nsteps, void *stream);
/* Synchronizes `stream` and returns in *failed whether any swe_imex_step_async call
 * since the last reset hit an unconverged solve; reset != 0 clears the flag. */
int swe_plan_status(swe_plan *plan, int *failed, int reset, void *stream);

/* truncate_pad (spharm.py:352-368) of `nfields` packed arrays between plans
 * (PrognosticState.to_truncation, dynamics.py:73-83). */
int swe_truncate_pad(const swe_plan *src, const swe_plan *dst, const double *in, double *out,
                     int nfields, void *stream);

/* PrognosticState.max_abs / is_finite (dynamics.py:65-71) per state of
 * [batch][3][K]; outputs are DEVICE arrays [batch]. */
int swe_state_stats(const swe_plan *plan, const double *state, int batch, double *max_abs_out,
                    int *finite_out, void *stream);

/* Serial IMEX sweep (the coarsest-level solve, pint.py:306-320): u [n+1][3][K]
 * device states, u[j] = step(u[j-1]) + g[j] for j = 1..n with g [n+1][3][K]
 * (nullable; g[0] unused); one CUDA-graph step per point and one host check. */
int swe_imex_sweep(swe_plan *plan, double *u, const double *g, int n, const double *phibar,
                   const swe_stepper_cfg *cfg, double *resid_out, void *stream);
/* swe_imex_sweep without the final host check (like swe_imex_step_async: an
 * unconverged solve raises the plan's flag, read by swe_plan_status). */
int swe_imex_sweep_async(swe_plan *plan, double *u, const double *g, int n, const double *phibar,
                         const swe_stepper_cfg *cfg, void *stream);
/* One SL-SI-SETTLS step (steppers.py:171-212) of every slice: state [batch][3][K]
 * advanced in place; prev [batch][3][K] is U_{n-1} (pass `state` itself for the
 * one-step variant or a cold start); the implicit solve always includes the
 * Coriolis term.  Returns SWE_ENOCONV (resid_out filled) like swe_imex_step and
 * SWE_ENONFINITE when a departure point is not finite. */
int swe_settls_step(swe_plan *plan, double *state, const double *prev, const double *phibar,
                    int batch, const swe_stepper_cfg *cfg, double *resid_out, void *stream);
/* Departure points (semilag.py:140-170) of every grid point for arrival winds
 * (u_arr, v_arr) and extrapolated winds (u_ext, v_ext), grids [batch][nlat][nlon];
 * outputs lam, th (same shape).  SWE_ENONFINITE if any is not finite. */
int swe_departure_points(swe_plan *plan, const double *u_arr, const double *v_arr,
                         const double *u_ext, const double *v_ext, int batch, double dt,
                         int iterations, double *lam, double *th, void *stream);
/* Bicubic interpolation of grids [batch][nlat][nlon] at (lam, th) of the same
 * shape (semilag.py:82-88, advect_scalar :173-179). */
int swe_interpolate(swe_plan *plan, const double *values, const double *lam, const double *th,
                    int batch, double *out, void *stream);

/* On-device diagnostics (diagnostics.py:46-118), deterministic reductions.
 * Kinetic-energy spectrum of states [batch][3][K]: energy[b][n-1], n = 1..M
 * (DEVICE output [batch][M]). */
int swe_ke_spectrum(const swe_plan *plan, const double *state, int batch, double *energy,
                    void *stream);
/* Windowed spectral error terms for fields x, y ([K] complex on this plan) and
 * rnorms[i] (HOST, 1..M, nr <= 64): out[2i] = max|x - y|, out[2i+1] = max|y| over
 * m, n <= rnorms[i] (DEVICE output [2 nr]). */
int swe_window_maxdiff(const swe_plan *plan, const double *x, const double *y,
                       const int *rnorms, int nr, double *out, void *stream);
/* out[0] = sum (x - y)^2, out[1] = sum y^2 over n doubles (DEVICE output [2]). */
int swe_grid_sqdiff(const double *x, const double *y, long long n, double *out, void *stream);

/* Number of this library's kernels launched since load (evidence counter). */
long long swe_kernel_launches(void);
/* Live per-launch profiling with CUDA events on the launching stream.
 * swe_profile(1) clears and starts recording, swe_profile(0) stops.
 * swe_profile_read fills, per kernel class [4] = {Legendre synthesis GEMM,
 * Legendre analysis GEMM, FFT + grid products, spectral elementwise}, the summed
 * device milliseconds, algorithmic work (flops for the GEMMs, bytes for the
 * FFT stage) and launch counts (all outputs HOST, nullable). */
int swe_profile(int enable);
/* Tuning switches.  "fft_path": 0 auto, 1 warp-per-row FFT kernel, 2 lane=row
 * FFT kernel (falls back to 1 where its radix/size limits do not hold).
 * "leg_path": 0 auto, 1 small-batch Legendre kernels, 2 / 3 wide-tile kernels
 * with 128 / 64 columns per CTA, 4 warp-specialised persistent kernels, 5 the
 * 8-lane dot-product kernels for 1..4 slices ("gemv_max_b": the auto path's
 * largest batch for them, default 3).
 * "fast_coriolis": 2 (default) spectral three-term recurrence, 1 FFT-free
 * Legendre pair, 0 pseudospectral FFT round trip.  "graphs": 1 (default)
 * replay one CUDA graph per IMEX step.  "helm_tiled", "cn_small", "cn_cluster":
 * 1 / 0 enable / disable the tiled fixed-point kernel and the one-CTA-per-slice
 * half step (K <= 2800); "cn_cluster" 1 (default) runs the shared-memory-resident
 * half step when its cluster of CTAs per slice is no larger than the batch asks
 * for (one CTA per slice from 32 slices, up to 16 for one slice; K up to ~38k
 * modes), 2 at any cluster size, 0 never; "cn_cluster_ctas" forces the CTAs per
 * slice (0 = by batch size). 
 * "cn_fused": 1 (default) speculative shared-memory fixed point for M <= 262 (the
 * guessed iteration count runs in one pass per m-block pair; slices converging
 * earlier are recomputed, later ones continue in the tiled loop), 0 off.  Results
 * agree to roundoff on every path (bitwise between the half-step paths; within
 * 1e-12 relative between the fast_coriolis modes). */
int swe_set_option(const char *key, int value);
int swe_profile_read(double *ms_out, double *work_out, long long *count_out);
const char *swe_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
