// Longitude FFT stage with fused grid-space products.
//
// Reference: np.fft.irfft / rfft calls of SphereGrid (spharm.py:241, :257,
// :267, :325-326) and the grid products of dynamics.py:129-160.  One CTA owns
// one latitude pair (north row p, south row J-1-p) and a block of slices;
// every field of both rows is inverse-transformed into shared memory (north =
// E + O, south = E - O of the parity-split Legendre output), combined
// pointwise, forward-transformed and folded into F+- = w (f_N +- f_S) for the
// analysis GEMM, so grid values never touch HBM.  The real transforms of even
// length I are complex transforms of length N2 = I/2 (in-place mixed-radix
// Cooley-Tukey or prime-factor).
#pragma once

#include "common.cuh"

namespace swe {

constexpr int FFT_MAXST = 12;
constexpr int FFT_MAXF = 8;

enum FftOpKind {
  FOP_SYNTH_GRID = 0,    // 1 half-spectrum  -> grid (scale: none | 1/(a cos))
  FOP_SYNTH2_GRID = 1,   // 2 half-spectra   -> 2 grids (scale 1/(a cos)): winds
  FOP_ANALYSIS = 2,      // grid             -> F (w/I)
  FOP_VORTDIV = 3,       // 2 grids (u, v)   -> 2 F (u cos, v cos; w/((1-mu^2) I a))
  FOP_CORIOLIS = 4,      // half(u), half(v) -> F(f u cos), F(f v cos)
  FOP_NONLINEAR = 5,     // 7 half-spectra   -> F(tphi), F(ke), F(xi u cos), F(xi v cos)
};

struct FftArgs {
  int M, J, I, N2, nst;
  int radix[FFT_MAXST];
  int ns[FFT_MAXST];
  const double2 *tw;   // [N2]  e^{2 pi i e / N2}
  const double2 *twh;  // [N2]  e^{2 pi i k / I}
  const int *pos_z;    // [N2]  slot of spectral index k (c2r input / r2c output order)
  const int *pos_g;    // [N2]  slot of grid pair r (g[2r], g[2r+1]) (c2r output / r2c input)
  int pfa;             // 1: prime-factor (coprime radices, no twiddles), 0: Cooley-Tukey
  int rgen;            // largest non-unrolled radix (per-warp scratch, complex), 0 if none
  int nslices, ld, spb, nwarps;
  int scale_mode;      // FOP_SYNTH_GRID: 0 none, 1 times 1/(a cos)
  const double *coslat, *inv_acos, *fcor, *wq, *wsin2;  // per latitude row [J]
  double inv_I, inv_a;
  int Jh, Jp;                   // latitude pairs (incl. equator), padded pair count
  const double *phisub;         // [slice] phibar*sqrt2*P_00, subtracted from field 5 (FOP_NONLINEAR)
  int in_pm;                    // FOP_NONLINEAR, lane kernel: inputs in the pair-major layout
                                // [Jh][M+1][ld/2][E,O] (LegOut::layout 1)
  int dlam;                     // FOP_NONLINEAR: field 2 (d_lambda Phi) is i m times field 5's
                                // half spectrum (in[2] unused): saves one synthesis term
  int no_rest;                  // FOP_NONLINEAR: omit -Phi' delta (nonlinear_advection alone)
  int out_il;                   // FOP_NONLINEAR, lane kernel: F+ and F- of one (m, pair, slice)
                                // adjacent ([m][Jp][slice][F+, F-] complex), one 32-byte store
  int v4ld;                     // lane kernel, pair-major input: E and O of one (m, slice) in
                                // one 256-bit load (LDG.E.256)
  int pf_pairs;                 // FOP_NONLINEAR, lane kernel, pair-major input: each CTA
                                // prefetches into L2 its share of the E/O block of the pair
                                // this many pairs ahead (0: off)
  const double *in[FFT_MAXF];   // E/O half spectra      [m][2][Jp][ld]
  double *out[FFT_MAXF];        // F+/F- analysis inputs [m][2][Jp][ld]
  const double *gin[2];         // grids [slice][J][I]
  double *gout[2];
};

int fft_launch(int op, const FftArgs &a, int smem_bytes, cudaStream_t st);
__host__ __device__ constexpr int fft_rows_per_slice(int op) {
  return op == FOP_NONLINEAR ? 6 : ((op == FOP_SYNTH2_GRID || op == FOP_VORTDIV || op == FOP_CORIOLIS) ? 2 : 1);
}
bool fft_small_radix(int R);

// "lane = row" variant (fft_lanes.cu): slices per CTA for each op
// (16 rows = fields x 2 hemispheres x slices)
__host__ __device__ constexpr int fft_lane_slices(int op) {
  return op == FOP_NONLINEAR ? 1 : ((op == FOP_SYNTH_GRID || op == FOP_ANALYSIS) ? 8 : 4);
}
int fft_lanes_launch(int op, const FftArgs &a, cudaStream_t st);
extern int g_fft_rm;  // 1: radix-specialised nonlinear lane kernels for the hot lengths
// rows per CTA of the lane kernel for this length (0: does not apply); *rgen: the
// largest radix that runs as a generic stage (0: all unrolled)
int fft_lanes_width(const FftArgs &a, int *rgen);
bool fft_lanes_ok(const FftArgs &a);

}  // namespace swe
