// DMMA.8x8x4 issue rate vs warps per SMSP: each warp runs ITER rounds of NACC
// independent m8n8k4 f64 MMAs; prints DMMAs per SM per cycle (peak: 4 SMSPs x 1/16).
#include <cstdio>
#include <cuda_runtime.h>
template <int NACC>
__global__ void k(double *out, int iters, long long *cyc) {
  double c0[NACC], c1[NACC];
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
#pragma unroll
  for (int i = 0; i < NACC; ++i) c0[i] = c1[i] = 0.0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0[i]), "+d"(c1[i]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c0[i] + c1[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double *out; long long *cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 1 << 16);
  const int iters = 2000;
  for (int wps = 1; wps <= 4; wps *= 2) {  // warps per SMSP
    const int nt = 128 * wps;
    k<16><<<nsm, nt>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, cyc, sizeof(long long) * nsm, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
    const double dmma = (double)iters * 16 * (nt / 32);  // per SM
    printf("warps/SMSP %d: %.3f DMMA per SM per cycle (peak 0.25), %.1f cycles per DMMA per warp\n", wps,
           dmma / mx, mx / ((double)iters * 16));
  }
  return 0;
}
