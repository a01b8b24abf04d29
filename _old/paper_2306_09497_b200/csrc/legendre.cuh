// Legendre-stage kernels: grouped, parity-folded FP64 DMMA GEMMs over order m.
//
// Reference: SphereGrid.synthesis / _synthesis_pair / analysis / vortdiv_from_uv
// (/root/reference/pkg/src/pintswe/spharm.py:238-267, :315-343) loop over m and
// run one skinny BLAS GEMM per order.  Here every order m is a group of one
// batched launch, and the north/south symmetry P_mn(-mu) = (-1)^(n-m) P_mn(mu)
// (H flips the other way) halves the flops: tables hold only the latitude
// pairs p = 0..Jh-1 (north rows), with the modes of each m-block reordered as
// [even n-m | odd n-m].
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace swe {

// One additive term of a Legendre contraction.
//  synthesis: out[E/O] += T(p, n) * f(src[mode][col])
//  analysis : out[mode][col] += sum_p T(p, n) * f(F±[p][col])
// with f(x) = sign * scale[mode] * (times_im ? i*m : 1) * x and, for the
// (0,0) mode only, x.re -= phi0[slice] (phi_prime, dynamics.py:52-56).
struct LegTerm {
  const double *tab;    // P or H table, row stride Jp
  const double *src;    // synthesis: spectral [K][ld]; analysis: F+/F- planes [m][2][Jp][ld]
  const double *scale;  // per packed mode (synthesis only), nullable
  const double *phi0;   // per slice, nullable (synthesis only)
  const double *pscale; // analysis only, nullable: per latitude pair factor on F+-
  double sign;
  int times_im;
  int flip;     // 0: P-like parity, 1: H-like (odd in mu for even n-m)
  int swap_pm;  // analysis only: read plane 1 as F+ and plane 0 as F- (E/O input)
  int f_il;     // analysis (v3) only: F+- interleaved per slice, [m][Jp][slice][F+, F-]
                // complex (the lane FFT's 32-byte stores), instead of planes [m][2][Jp][ld]
};

struct LegOut {
  LegTerm t[2];
  int nterms;
  // synthesis output layout: 0 = planes [m][E,O][Jp][ld]; 1 = pair-major
  // [Jh][ld/2 slices][M+1][E,O] complex, so one (pair, slice) of a field is one
  // contiguous 16(M+1)-double block for the FFT loader (legendre_v3.cu only)
  int layout;
  double *dst;  // synthesis: [m][J][ld] (north/south rows); analysis: [K][ld]
};

constexpr int LEG_MAXOUT = 8;

struct LegArgs {
  LegOut out[LEG_MAXOUT];
  int nout;
  int M, J, Jh, Jp, ld;
  const int *offsets;  // [M+2] packed-mode block offsets
  const int2 *items;   // (m, tile) work items, heaviest first
  int nitems;
  // v3 dynamic scheduling: device [ticket counter, CTAs done] (per plan / stream;
  // zero between launches)
  unsigned long long *sched;
  const double *zeros;  // >= 1024 zero doubles (v3: source of padding rows)
  // v3 analysis: TMA tensor maps of the P (0) and H (1) tables, [K][Jp] fp64, box
  // 16 pairs x 32 modes, 128-byte swizzle (plan.cu)
  CUtensorMap tmap[2];
};

// Launch helpers (legendre.cu).  items/tiles are prepared by the plan.
int leg_synth_launch(const LegArgs &a, int ncoltiles, cudaStream_t st);
int leg_anal_launch(const LegArgs &a, int ncoltiles, cudaStream_t st);
// few-slice variants (8-lane dot products) over the first nslice complex columns
int leg_synth_gemv_launch(const LegArgs &a, int nslice, cudaStream_t st);
int leg_anal_gemv_launch(const LegArgs &a, int nslice, int K, cudaStream_t st);
// wide-tile variants (legendre_v2.cu): column tile bn = 64 (4 warps) or 128 (8 warps)
int leg_synth_v2_launch(const LegArgs &a, int bn, cudaStream_t st);
int leg_anal_v2_launch(const LegArgs &a, int bn, cudaStream_t st);
constexpr int V2_ABR = 32;  // analysis modes per parity per CTA
// warp-specialised persistent variants (legendre_v3.cu): TMA bulk-copy producer warp,
// 8 DMMA consumer warps, 128-column tiles, one CTA per SM
constexpr int V3_ABR = 32;  // v3 analysis modes per parity per work unit
int leg_synth_v3_launch(const LegArgs &a, cudaStream_t st);
int leg_anal_v3_launch(const LegArgs &a, cudaStream_t st);

constexpr int SY_BM = 64;   // latitude pairs per CTA
constexpr int SY_BN = 64;   // real columns per CTA
constexpr int AN_BR = 16;   // modes per parity per CTA
constexpr int AN_BN = 64;   // real columns per CTA
constexpr int AN_KP = 16;   // latitude pairs per k-chunk (Jp is a multiple of this)

}  // namespace swe
