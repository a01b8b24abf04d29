// On-device diagnostics (reference diagnostics.py:46-118): kinetic-energy
// spectrum, windowed spectral error and grid RMS sums.  Every reduction runs in
// a fixed order (no atomics), so results are bitwise reproducible run to run.
#include <cuda_runtime.h>

#include "common.cuh"
#include "plan.cuh"
#include "swe_b200.h"

namespace swe {

namespace {

struct Rnorms {
  int r[64];
};

// energy[b][n-1] = 0.25 a^2/(n(n+1)) sum_{m<=n} mult(m) (|xi_mn|^2 + |delta_mn|^2),
// m ascending like np.bincount over the packed order (diagnostics.py:78-87)
__global__ void k_ke_spectrum(const double2 *__restrict__ state, int B, int M, int K,
                              const int *__restrict__ offsets, double a, double *energy) {
  const int b = blockIdx.y;
  const int n = blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (n > M || b >= B) return;
  const double2 *xi = state + ((size_t)b * 3 + 1) * K, *de = state + ((size_t)b * 3 + 2) * K;
  double acc = 0.0;
  for (int m = 0; m <= n; ++m) {
    const int k = offsets[m] + (n - m);
    const double ax = hypot(xi[k].x, xi[k].y), ad = hypot(de[k].x, de[k].y);
    acc += (m == 0 ? 1.0 : 2.0) * (ax * ax + ad * ad);
  }
  energy[(size_t)b * M + (n - 1)] = 0.25 * a * a / (n * (n + 1.0)) * acc;
}

// out[2i] = max |x - y|, out[2i+1] = max |y| over the window m, n <= rnorm[i]
// (field x, y: [K] complex on one plan; diagnostics.py:46-65).  One block per rnorm.
__global__ void k_window_max(const double2 *__restrict__ x, const double2 *__restrict__ y,
                             int M, const int *__restrict__ offsets, Rnorms rn, double *out) {
  __shared__ double sd[256], sr[256];
  const int R = rn.r[blockIdx.x];
  double md = 0.0, mr = 0.0;
  for (int m = 0; m <= R && m <= M; ++m)
    for (int n = m + threadIdx.x; n <= R && n <= M; n += blockDim.x) {
      const int k = offsets[m] + (n - m);
      const double d = hypot(x[k].x - y[k].x, x[k].y - y[k].y), r = hypot(y[k].x, y[k].y);
      md = (isnan(d) || isnan(md)) ? nan("") : fmax(md, d);
      mr = (isnan(r) || isnan(mr)) ? nan("") : fmax(mr, r);
    }
  sd[threadIdx.x] = md;
  sr[threadIdx.x] = mr;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double a = sd[threadIdx.x], b = sd[threadIdx.x + s];
      sd[threadIdx.x] = (isnan(a) || isnan(b)) ? nan("") : fmax(a, b);
      const double c = sr[threadIdx.x], e = sr[threadIdx.x + s];
      sr[threadIdx.x] = (isnan(c) || isnan(e)) ? nan("") : fmax(c, e);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = sd[0];
    out[2 * blockIdx.x + 1] = sr[0];
  }
}

// out[0] = sum (x - y)^2, out[1] = sum y^2 (diagnostics.py:68-75), one block,
// fixed strided order + tree
__global__ void k_grid_sqdiff(const double *__restrict__ x, const double *__restrict__ y,
                              long long n, double *out) {
  __shared__ double s0[1024], s1[1024];
  double a = 0.0, c = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = x[i] - y[i];
    a += d * d;
    c += y[i] * y[i];
  }
  s0[threadIdx.x] = a;
  s1[threadIdx.x] = c;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      s0[threadIdx.x] += s0[threadIdx.x + s];
      s1[threadIdx.x] += s1[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = s0[0];
    out[1] = s1[0];
  }
}

}  // namespace
}  // namespace swe

using namespace swe;

extern "C" int swe_ke_spectrum(const swe_plan *pl, const double *state, int batch,
                               double *energy, void *stream) {
  if (!pl || !state || !energy || batch < 1) {
    set_error("swe_ke_spectrum: null argument or batch < 1");
    return E_SHAPE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid((pl->M + 127) / 128, batch);
  k_ke_spectrum<<<grid, 128, 0, st>>>(reinterpret_cast<const double2 *>(state), batch, pl->M,
                                      pl->K, pl->offsets, pl->a, energy);
  SWE_LAUNCH_CHECK();
  return OK;
}

extern "C" int swe_window_maxdiff(const swe_plan *pl, const double *x, const double *y,
                                  const int *rnorms, int nr, double *out, void *stream) {
  if (!pl || !x || !y || !rnorms || !out || nr < 1 || nr > 64) {
    set_error("swe_window_maxdiff: null argument or nr outside 1..64");
    return E_SHAPE;
  }
  for (int i = 0; i < nr; ++i)
    if (rnorms[i] < 1 || rnorms[i] > pl->M) {
      set_error("rnorm %d outside 1..%d", rnorms[i], pl->M);
      return E_SHAPE;
    }
  Rnorms rn{};  // by value in the kernel parameters (no copy)
  for (int i = 0; i < nr; ++i) rn.r[i] = rnorms[i];
  k_window_max<<<nr, 256, 0, (cudaStream_t)stream>>>(reinterpret_cast<const double2 *>(x),
                                                     reinterpret_cast<const double2 *>(y), pl->M,
                                                     pl->offsets, rn, out);
  SWE_LAUNCH_CHECK();
  return OK;
}

extern "C" int swe_grid_sqdiff(const double *x, const double *y, long long n, double *out,
                               void *stream) {
  if (!x || !y || !out || n < 1) {
    set_error("swe_grid_sqdiff: null argument or n < 1");
    return E_SHAPE;
  }
  k_grid_sqdiff<<<1, 1024, 0, (cudaStream_t)stream>>>(x, y, n, out);
  SWE_LAUNCH_CHECK();
  return OK;
}
