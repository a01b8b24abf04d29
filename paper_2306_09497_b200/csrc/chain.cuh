// Persistent serial IMEX chain (the coarsest-level sweep, pint.py:306-320, and the
// level-1 initial guess, :341-353): u[j] = step(u[j-1]) + g[j], j = 1..n, for ONE
// slice of a coarse truncation, all n steps inside one thread-block-cluster kernel
// (chain.cu).  The per-step path launches ~12 kernels per step (M = 51: ~100 us,
// latency-bound); here the phases of a step are separated by cluster barriers and
// every phase runs the per-step path's device code (legendre_gemv.cuh,
// fft_lanes_dev.cuh, cn_cluster.cuh), so the chain is bitwise the per-step sweep.
#pragma once

#include "cn_cluster.cuh"
#include "fft.cuh"
#include "legendre.cuh"

namespace swe {

struct ChainArgs {
  LegArgs syn[2], an[2];  // nonlinear evaluation on U* (-> K1) and on U* + dt K1 (-> K2)
  FftArgs fft;
  CcRanges rg;
  int C, cap, K, M, n;
  double *U[3], *US[3], *K1[3], *K2[3], *MID[3], *TMP;  // internal layout, one slice
  const double *lap, *eps, *phibar;
  const int2 *nbt;
  const double4 *cft;
  double dt, alpha, dtnu, halfq, tol;
  int max_iter;
  int *iters, *flags, *counter, *fail;
  double *resid;
  const double *g;   // forcing, internal layout [3][K][n] (column j-1 for step j), nullable
  double *u;         // boundary layout [n+1][3][K] complex: u[j] written after step j
  const int *iperm;  // internal row -> reference packed index
};

// smem bytes of the kernel for a plan (0: the chain does not apply)
int chain_smem(int N2, int cap);
int chain_launch(const ChainArgs *dev_args, int C, int smem, cudaStream_t st);
// the cluster kernel can be scheduled with C CTAs and smem bytes each
bool chain_ok(int C, int smem);

}  // namespace swe
