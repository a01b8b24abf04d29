// Shared device helpers for the B200 fine-propagator kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define SWE_DEV __device__ __forceinline__

// a / b, correctly rounded, from r = RN(1 / b) (Markstein: q0 = RN(a r), the
// remainder e = a - b q0 exact by FMA, RN(q0 + e r) = RN(a / b) for normal
// operands); 3 DFMA instead of the division sequence when b repeats.  e == 0: q0 is
// exact (keeps the sign of a zero quotient)
SWE_DEV double ddiv_r(double a, double b, double r) {
  const double q0 = a * r;
  const double e = fma(-q0, b, a);
  return e == 0.0 ? q0 : fma(e, r, q0);
}

namespace swe {

// ---- error plumbing (host) -------------------------------------------------
enum Status { OK = 0, E_SHAPE = 1, E_NOCONV = 2, E_NONFINITE = 3, E_CUDA = 4, E_NCCL = 5 };
void set_error(const char *fmt, ...);
int cuda_fail(cudaError_t e, const char *what, const char *file, int line);
#define SWE_CUDA(call)                                                         \
  do {                                                                         \
    cudaError_t _e = (call);                                                   \
    if (_e != cudaSuccess) return ::swe::cuda_fail(_e, #call, __FILE__, __LINE__); \
  } while (0)
extern long long g_launches;  // kernels launched by this library (evidence counter)
#define SWE_LAUNCH_CHECK()   \
  do {                       \
    ++::swe::g_launches;     \
    SWE_CUDA(cudaGetLastError()); \
  } while (0)

// ---- cp.async (Ampere+ LDGSTS; 16-byte chunks, zero-fill when src_bytes=0) ---
SWE_DEV void cp_async16(void *smem, const void *gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
SWE_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
SWE_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col) -------------
// Fragment ownership (PTX ISA, mma.m8n8k4 .f64): lane = 4*g + t,
//   A: a = A[g][t]        B: b = B[t][g]        C/D: c0,c1 = C[g][2t], C[g][2t+1]
// Lowers to SASS DMMA.8x8x4 on sm_100a.
SWE_DEV void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct cplx {
  double x, y;
};
SWE_DEV cplx cmul(cplx a, cplx b) { return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
SWE_DEV cplx cadd(cplx a, cplx b) { return {a.x + b.x, a.y + b.y}; }
SWE_DEV cplx csub(cplx a, cplx b) { return {a.x - b.x, a.y - b.y}; }
SWE_DEV cplx cconj(cplx a) { return {a.x, -a.y}; }

// Non-negative doubles order like their bit patterns: max via integer atomics.
SWE_DEV void atomic_max_nonneg(double *addr, double v) {
  if (!(v >= 0.0)) {  // NaN: record it so finiteness checks see it
    atomicExch((unsigned long long *)addr, 0x7ff8000000000000ULL);
    return;
  }
  atomicMax((unsigned long long *)addr, (unsigned long long)__double_as_longlong(v));
}

}  // namespace swe
