// SL-SI-SETTLS kernels (settls.cu); see stepper.cu settls_internal for the step.
#pragma once

#include "common.cuh"

namespace swe {

struct SetArgs {
  int B, J, I;
  const double *mu, *coslat;  // [J] north -> south
  const double *nodes;        // [J+4] ascending latitudes with two pole ghosts each side
  double radius;
  // winds at t_n (arrival) and t_{n-1} (history), grids [B][J][I]
  const double *un, *vn, *up, *vp;
  int ext_given;  // 1: (up, vp) already hold the extrapolated wind, not t_{n-1}
};

struct GridPtrs {
  const double *in[4];
  double *out[4];
};

// departure points of every grid point (semilag.py:140-170); *bad = 1 when any
// is non-finite
int departure_points(const SetArgs &a, int iterations, double dt, double *lam, double *th,
                     int *bad, cudaStream_t st);
// bicubic interpolation of nf <= 4 grid fields at (lam, th) (semilag.py:82-88, :173-179)
int interp_fields(const SetArgs &a, const double *lam, const double *th, int nf,
                  const GridPtrs &p, cudaStream_t st);
// (phi - phibar[b]) * delta on the grid (nonlinear_rest's product)
int phiprime_mul(int B, size_t per, const double *phi, const double *de, const double *phibar,
                 double *out, cudaStream_t st);

// G = U + h (L U + 2 N_R(U) - N_R(prev)) (Phi), U + h L U (xi, delta)
int settls_g(int K, int B, double *const u[3], double *const l[3], const double *nru,
             const double *nrp, double h, double *const g[3], cudaStream_t st);
// y += s x over K*B complex values
int spec_axpy(int K, int B, double *y, const double *x, double s, cudaStream_t st);

}  // namespace swe
