// Transform plan: grid, Legendre tables, FFT factorisation, workspaces.
//
// Mirrors SphereGrid.__init__ (spharm.py:154-202): Gauss-Legendre nodes,
// orthonormal P_mn and H_mn = (1-mu^2) dP/dmu tables, Laplacian eigenvalues,
// w/(1-mu^2), f = 2 Omega mu.  HBM layout (doubles):
//   P, H          [K rows][Jp]   row = offset[m] + (n-m even ? (n-m)/2 : ne(m) + (n-m-1)/2),
//                                column = latitude pair p (north row), zero for p >= Jh
//   spectral      [K][ld]        mode row in the same parity-split order as the tables
//                                x column 2*slice + re/im (boundary: reference packing)
//   half / F      [M+1][J][ld]   order m x latitude row x column
#pragma once

#include <vector>

#include "fft.cuh"
#include "legendre.cuh"

namespace swe {

struct Work {
  int cap = 0;         // slices the buffers were sized for
  double *spec = nullptr;   // NSPEC spectral arrays [K][2*cap]
  double *half = nullptr;   // NHALF half-spectrum arrays [M+1][J][2*cap]
  double *fspec = nullptr;  // NF analysis-input arrays  [M+1][J][2*cap]
  double *stats = nullptr;  // [cap][8]
  unsigned long long *fstats = nullptr;  // [cap][cn_fused_kmax()][6] (k_cn_fused)
  int *target2 = nullptr;   // [cap] k_cn_fused recompute targets
  int *flags = nullptr;     // [cap] active / converged flags, iteration counts
  int *iters = nullptr;     // [cap]
  int *counter = nullptr;   // device counter (active slices)
  int *h_counter = nullptr; // pinned host mirror
  int *h_iters = nullptr;   // [cap] pinned host mirror of iters
  // mapped (zero-copy) host words [1 + cap]: active count, then iters; written by
  // k_publish so the per-half-step check does not queue behind bulk D2H copies
  int *h_pub = nullptr, *d_pub = nullptr;
  unsigned long long *sched = nullptr;  // Legendre v3 work-unit scheduler [2] (device)
  int *loop = nullptr;                  // graph mode: fixed-point iteration counter (device)
  unsigned *hdone = nullptr;            // k_helm last-block detection (device, zero between launches)
  int *h_bad = nullptr, *d_bad = nullptr;  // SETTLS: non-finite departure point seen (mapped)
  double *grids = nullptr;              // SETTLS grid workspace: 12 x [gcap][J][I]
  double *sweep_g = nullptr;            // serial-sweep forcing, internal layout 3 x [K][2 scap]
  int scap = 0;
  int gcap = 0;
  int *h_fail = nullptr, *d_fail = nullptr;
  // an asynchronous call (swe_imex_step_async / swe_imex_sweep_async) may have raised
  // d_fail since the last swe_plan_status reset: synchronous calls then keep it up
  int async_pending = 0;
  // graph replays: the fused fixed point's iteration guess on the device (k_cn_decide
  // updates it, so a replayed graph adapts to the states as the host path does)
  int *gguess = nullptr;  // graph mode: unconverged-solve flag (device) and its host copy
  double *phi0 = nullptr;   // [cap] phibar*sqrt(2)*P_00: synthesis of the phi_prime shift
  double *phibar = nullptr; // [cap]
};

constexpr int NSPEC = 30;  // 21-23: input backup of a graph-mode call
constexpr int NHALF = 7;
constexpr int NF = 4;

}  // namespace swe

struct swe_plan {
  int M, J, I, Jh, Jp, K, N2, device;
  double a, omega, gravity;
  std::vector<double> mu, w;  // host copies (decreasing mu)
  // device tables
  double *P = nullptr, *H = nullptr;
  int *offsets = nullptr;
  int *perm = nullptr;  // [K] reference packed index -> internal (parity-split) row
  double *lap_eig = nullptr, *inv_lap = nullptr, *eps = nullptr;
  double *coslat = nullptr, *inv_acos = nullptr, *fcor = nullptr, *wq = nullptr, *wsin2 = nullptr;
  double *cor_scale = nullptr;  // [Jp] 2 w f / ((1 - mu^2) a^2) per pair (FFT-free Coriolis)
  int2 *cor_nb = nullptr;       // [K] internal rows of modes n-1, n+1 (-1: none) (spectral Coriolis)
  double4 *cor_cf = nullptr;    // [K] (c_lo, c_hi, c_im, m == 0) of the spectral Coriolis operator
  double *zeros = nullptr;      // 1024 zero doubles (padding rows of the v3 GEMMs)
  double *mu_dev = nullptr;     // [J] Gauss nodes (north -> south)
  double *sl_nodes = nullptr;   // [J+4] ascending latitudes + 2 pole ghosts each side (SETTLS)
  int2 *helm_tiles = nullptr;   // (m, chunk of 64 n) tiles of the tiled fixed-point kernel
  int n_helm_tiles = 0;
  double2 *tw = nullptr, *twh = nullptr;
  int *fft_pos_z = nullptr, *fft_pos_g = nullptr;
  int pfa = 0;
  int rgen = 0;
  int2 *synth_items = nullptr, *anal_items = nullptr;
  int n_synth_items = 0, n_anal_items = 0;
  int2 *synth_items_v3 = nullptr;  // last latitude tile absorbs a remainder of <= 8 pairs
  int n_synth_items_v3 = 0;
  int2 *anal_items_v2 = nullptr, *anal_items_v3 = nullptr;
  int n_anal_items_v2 = 0, n_anal_items_v3 = 0;
  int nst = 0;
  int radix[swe::FFT_MAXST], ns[swe::FFT_MAXST];
  std::vector<int> h_offsets;
  swe::Work ws;
  // CUDA graphs of one IMEX step (stepper.cu), keyed by batch, stepper config and
  // tuning switches; invalidated when the workspace is reallocated
  struct StepGraph {
    int B, Bsel;
    double dt, nu, tol;
    int order, cor_impl, nonlin, max_iter, solver;
    long long opts;
    cudaGraph_t graph;
    cudaGraphExec_t exec;
  };
  std::vector<StepGraph> graphs;
  cudaStream_t cap[2] = {nullptr, nullptr};  // capture streams (step, fixed-point body)
  int iter_guess = 1;  // fixed-point iterations launched before the first host check
  size_t table_bytes = 0;
  CUtensorMap tmap[2];  // TMA descriptors of P and H (legendre_v3.cu analysis tiles)
};
