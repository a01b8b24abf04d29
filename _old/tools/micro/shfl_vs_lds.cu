// Microbenchmark: warp-shuffle vs shared-memory (LDS.128) throughput on one SM and
// whether the two contend for the same pipe (decides how the FFT exchanges data).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITERS = 4096;
template <int MODE>  // 0 shfl only, 1 lds only, 2 both
__global__ void __launch_bounds__(256, 2) kern(double *out) {
  __shared__ double2 buf[8 * 256];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 8 * 256; i += 256) buf[i] = make_double2(i, -i);
  __syncthreads();
  unsigned a0 = tid, a1 = tid * 3, a2 = tid * 5, a3 = tid * 7;
  double2 s0 = make_double2(0, 0), s1 = s0;
  for (int it = 0; it < ITERS; ++it) {
    if (MODE != 1) {
      a0 = __shfl_xor_sync(0xffffffffu, a0, 1) + 1;
      a1 = __shfl_xor_sync(0xffffffffu, a1, 2) + 1;
      a2 = __shfl_xor_sync(0xffffffffu, a2, 4) + 1;
      a3 = __shfl_xor_sync(0xffffffffu, a3, 8) + 1;
    }
    if (MODE != 0) {
      // 16-byte loads, a warp reads one 512-byte line (4 wavefronts, conflict-free)
      const int base = ((it * 7 + (tid >> 5)) & 7) * 256;
      const double2 x = buf[base + lane], y = buf[base + 32 + lane];
      s0.x += x.x; s0.y += x.y; s1.x += y.x; s1.y += y.y;
    }
  }
  out[blockIdx.x * 256 + tid] = a0 + a1 + a2 + a3 + s0.x + s0.y + s1.x + s1.y;
}
template <int MODE>
float run(double *d, int grid) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<MODE><<<grid, 256>>>(d);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<MODE><<<grid, 256>>>(d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int grid = 2 * sms;
  double *d;
  cudaMalloc(&d, grid * 256 * sizeof(double));
  const float t0 = run<0>(d, grid), t1 = run<1>(d, grid), t2 = run<2>(d, grid);
  const double warps = 2.0 * 8;  // per SM
  const double shfl = warps * ITERS * 4, lds_wf = warps * ITERS * 2 * 4;  // per SM
  printf("shfl only %.3f ms: %.2f warp-shfl/ns/SM\n", t0, shfl / (t0 * 1e6));
  printf("lds only  %.3f ms: %.2f wavefronts/ns/SM\n", t1, lds_wf / (t1 * 1e6));
  printf("both      %.3f ms (sum %.3f, max %.3f)\n", t2, t0 + t1, t0 > t1 ? t0 : t1);
  printf("clock %d kHz\n", clk);
  return 0;
}
