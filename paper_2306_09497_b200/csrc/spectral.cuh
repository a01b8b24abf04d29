// Spectral-space kernels (declarations); see spectral.cu.
#pragma once

#include <algorithm>

#include "common.cuh"

namespace swe {

struct SpecPtrs {
  double *p[8];
};
struct SpecPtrsC {
  const double *p[8];
};
struct Ptr3 {
  double *p[3];
};
struct Ptr3C {
  const double *p[3];
};

// sstride: slice stride of the boundary array in complex elements (0: packed, F * K)
int to_internal(const double *src, const SpecPtrs &dst, int B, int F, int K, const int *perm,
                cudaStream_t st, size_t sstride = 0);
// skip (nullable, device): the copy is skipped when *skip != 0 (an unconverged graph
// step leaves the caller's input in place for the host-driven rerun)
int to_boundary(const SpecPtrsC &src, double *dst, int B, int F, int K, const int *perm,
                cudaStream_t st, const int *skip = nullptr, size_t sstride = 0);
int lin_rhs(int K, int B, const double *const U[3], const double *lcx, const double *lcd,
            double alpha, const double *eps, const double *phibar, double *const R[3],
            cudaStream_t st);
int lin_tend(int K, int B, const double *U0, const double *U2, const double *lcx,
             const double *lcd, const double *eps, const double *phibar, double *const T[3],
             cudaStream_t st);
// spectral Coriolis operator (plan.cu cor_nb / cor_cf) applied to (x, d) = (xi, delta)
struct CorOp {
  const double *x, *d;
  const int2 *nb;
  const double4 *cf;
};
int coriolis_spec(int K, int B, const CorOp &c, double *lcx, double *lcd, cudaStream_t st);
// cor != nullptr: L_C is evaluated inline from the previous iterate, which for
// slice b is in A = (cor->x, cor->d) when iters[b] is even and in B = (U[1], U[2])
// when odd; the new xi/delta go to the other pair (Phi stays in U[0]).
// counter (nullable) is zeroed for the k_decide that follows; with hdone (a
// zeroed device word) the kernel's last block makes that decision itself
// (k_decide fused) and writes the active count to *counter.
int helm(int K, int B, const double *const R[3], const double *lcx, const double *lcd,
         double alpha, const double *eps, const double *phibar, double *const U[3],
         const int *active, double *stats, cudaStream_t st, const CorOp *cor = nullptr,
         int *iters = nullptr, int *counter = nullptr, double tol = 0.0,
         unsigned *hdone = nullptr);
int publish(int B, const int *counter, const int *iters, int *pub, cudaStream_t st);
// tiled fused fixed-point iterate for batches >= 32 (see k_helm_tiled)
int helm_tiled(int M, int K, int B, const int *offsets, const int2 *tiles, int ntiles,
               const double *const R[3], double alpha, const double *eps, const double *phibar,
               double *U0, double *A1, double *A2, double *B1, double *B2, const double4 *cf,
               const int *active, double *stats, const int *iters, int *counter,
               cudaStream_t st);
// whole CN half step for K <= 2800 modes (coarse levels), one CTA per slice
int cn_small_ok(int K);
int cn_small(int K, int B, Ptr3C x0, Ptr3C x1, Ptr3C x2, double s, double alpha,
             const double *eps, const double *phibar, const int2 *nb, const double4 *cf,
             int rhs_given, Ptr3 R, Ptr3 dst, int max_iter, double tol, double dtnu,
             double halfq, int *iters, int *flags, int *counter, double *resid, int *fail,
             cudaStream_t st);
// the same for K up to ~38k modes (the fine level M = 256): one thread-block
// cluster per slice; cn_cluster_size(M, want) = CTAs per cluster (at least `want`
// when the m-blocks allow), 0 when not applicable
int cn_cluster_size(int M, int want);
int cn_cluster(int M, int want, int B, Ptr3C x0, Ptr3C x1, Ptr3C x2, double s, double alpha,
               const double *eps, const double *phibar, const int2 *nb, const double4 *cf,
               int rhs_given, Ptr3 dst, int max_iter, double tol, double dtnu, double halfq,
               int *iters, int *flags, int *counter, double *resid, int *fail, cudaStream_t st);
// direct (block-tridiagonal) solve of the same implicit system instead of the fixed
// point (StepperConfig.implicit_solver = "direct"); scratch = 5 spectral arrays
int cn_direct(int M, int B, Ptr3C x0, Ptr3C x1, Ptr3C x2, double s, double alpha,
              const double *eps, const double *phibar, const int2 *nb, const double4 *cf,
              int rhs_given, double *const scratch[5], Ptr3 dst, double dtnu, double halfq,
              cudaStream_t st);
// speculative fused fixed point (fine level, M <= 262; see k_cn_fused): G guessed
// iterations with per-iteration maxima in fst [B][cn_fused_kmax()][6]; target
// (nullable: all G) per slice: > 0 the final (viscosity-applied) result of that
// iteration, < 0 the raw iterate -target for the k_helm_tiled loop, 0 skip
int cn_fused_ok(int M, int B);
int cn_fused_kmax();
int cn_fused(int M, int B, const int *offsets, const double4 *cf, const double *eps,
             const double *phibar, Ptr3C x0, Ptr3C x1, Ptr3C x2, double s, double alpha,
             Ptr3 R, int write_r, double *U0, double *A1, double *A2, double *B1, double *B2,
             const int *target, int G, unsigned long long *fst, double dtnu, double halfq,
             cudaStream_t st, const int *Gp = nullptr);
// Gp (graph replays): device-resident iteration guess, read by the first fused pass
// and k_cn_decide (capped at G) and updated by k_cn_decide for the next solve
int cn_decide(int B, int G, unsigned long long *fst, int *flags, int *iters, int *target2,
              int *counter, int *loop, double tol, const cudaGraphConditionalHandle *h,
              int max_iter, cudaStream_t st, int *Gp = nullptr);
// serial-sweep point (B = 1): y += g[:, col] if g.p[0], then y -> dst (boundary layout)
int sweep_point(int K, int n, int col, Ptr3 y, Ptr3C g, double *dst, const int *perm,
                cudaStream_t st);
int cn_start(int K, int B, Ptr3C x0, Ptr3C x1, Ptr3C x2, double s, double alpha,
             const double *eps, const double *phibar, const CorOp &c, Ptr3 R, Ptr3 dst,
             cudaStream_t st);
// counter/fail (nullable): graph mode records an unconverged fixed point in *fail;
// skip (nullable): slices with skip[b] >= 0 were finished by k_cn_fused
int cn_finish(int K, int B, Ptr3 u, const double *b1, const double *b2, const int *iters,
              const double *nn1a2, double dtnu, double halfq, cudaStream_t st,
              const int *counter = nullptr, int *fail = nullptr, const int *skip = nullptr);
int loop_cond(cudaGraphConditionalHandle h, const int *counter, int *loop, int max_iter,
              cudaStream_t st);
int decide(int B, double *stats, int *active, int *iters, int *counter, double tol,
           cudaStream_t st);
int fill_int(int *p, int n, int v, cudaStream_t st);
int axpy3(size_t n, Ptr3C a, Ptr3C x1, Ptr3C x2, double s, Ptr3 y, cudaStream_t st);
// kd -= lap ke (k_tend_finish), then mid = us + s (k1 with kd as its third field)
int finish_axpy(int K, int B, double *kd, const double *ke, const double *lap, Ptr3C us, Ptr3C k1,
                double s, Ptr3 mid, cudaStream_t st);
int tend_finish(int K, int B, double *kd, const double *ke, const double *lap, double *kx,
                const double *lcx, const double *lcd, cudaStream_t st);
int visc(int K, int B, Ptr3 u, const double *nn1a2, double dtnu, double halfq, cudaStream_t st);
int copy3(size_t n, Ptr3C a, Ptr3 y, cudaStream_t st);
int set_phibar(int B, const double *phibar, double *pb, double *phi0, cudaStream_t st);
int resid(int K, int B, Ptr3C u, Ptr3C rhs, const double *lcx, const double *lcd, double alpha,
          const double *eps, const double *phibar, double *res, cudaStream_t st);
int state_stats(const double *s, int B, int K, double *maxabs, int *finite, cudaStream_t st);
int truncate_pad(const double *src, double *dst, int nb, int Ms, int Md, const int *offs_s,
                 const int *offs_d, cudaStream_t st);

}  // namespace swe
