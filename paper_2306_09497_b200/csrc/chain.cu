// Persistent serial IMEX chain on one thread-block cluster (see chain.cuh).
//
// One slice, C CTAs of CC_NT threads (the cluster of the Crank-Nicolson half step,
// cn_cluster.cuh: CTA c owns the whole m-blocks of internal rows [rg.k[c], rg.k[c+1])).
// Per step (steppers.py:155-168, the spectral-Coriolis path of stepper.cu
// imex_internal with one slice):
//   U* = CN_half(U)                      cn_cluster_body (rows owned per CTA)
//   K1 = N(U*): synthesis gemv groups    all cluster threads  | cluster barrier
//               lane FFT + grid products latitude pairs c, c+C, ... | barrier
//               analysis gemv groups     all cluster threads  | barrier
//               K1_d -= lap ke, MID = U* + dt K1   own rows   | barrier
//   K2 = N(MID)                          as above
//   U = visc(CN_half(U* + dt/2 (K1 + K2)))   cn_cluster_body
//   U += g[j]; u[j] = U (reference packed layout)   own rows
// Intermediates live in the plan workspace (L2-resident at coarse truncations) and
// are read through L2 (ld.global.cg) after the barrier that publishes them.  Every
// phase runs the per-step kernels' device code on the same element -> thread-group
// arithmetic, so the result is bitwise the per-step sweep (test_gpu_pint.py).
#include <vector>

#include "chain.cuh"
#include "fft_lanes_dev.cuh"
#include "legendre_gemv.cuh"

namespace swe {

namespace {

// synthesis -> FFT -> analysis of one nonlinear evaluation (dynamics.py:142-160)
SWE_DEV void chain_nonlinear(const ChainArgs &a, int e, cg::cluster_group &cl, int c,
                             double2 *dsm) {
  const int tid = threadIdx.x, C = a.C;
  const long long gw = ((long long)c * CC_NT + (tid & ~31)) / GV_L, step = (long long)C * CC_NT / GV_L;
  const int gl = tid & (GV_L - 1), sub = (tid & 31) / GV_L;
  {
    const LegArgs &sa = a.syn[e];
    const long long ng = (long long)sa.nout * (a.M + 1) * sa.Jh;
    for (long long g0 = gw; g0 < ng; g0 += step)
      synth_gemv_group<1, true>(sa, g0 + sub, gl, g0 + sub < ng);
  }
  cl.sync();
  {
    const FftArgs &f = a.fft;
    LCtx lc;
    lc.X = dsm;
    lc.ct = dsm + (size_t)f.N2 * 16;
    lc.S = lane_slices(FOP_NONLINEAR, 16);
    lc.split = 0;
    lc.hem = 0;
    lc.b0 = 0;
    lc.nsl = 1;
    lc.tid = tid;
    lc.nthr = CC_NT;
    for (int p = c; p < f.Jh; p += C) {
      lc.p = p;
      lc.jn = p;
      lc.js = f.J - 1 - p;
      lc.eq = lc.js == lc.jn;
      lane_nonlinear<16, false, true>(f, lc);
      __syncthreads();  // the next pair reuses the rows
    }
  }
  cl.sync();
  {
    const LegArgs &aa = a.an[e];
    const long long ng = (long long)aa.nout * a.K;
    for (long long g0 = gw; g0 < ng; g0 += step)
      anal_gemv_group<1, true>(aa, a.K, g0 + sub, gl, g0 + sub < ng);
  }
  cl.sync();
}

__global__ void __launch_bounds__(CC_NT, 1) k_chain(const ChainArgs *__restrict__ pa) {
  const ChainArgs &a = *pa;
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank(), tid = threadIdx.x;
  extern __shared__ __align__(16) double2 dsm[];
  __shared__ CcShared sh;
  const int K = a.K, k0 = a.rg.k[c], k1 = a.rg.k[c + 1];
  const Ptr3C none = {{nullptr, nullptr, nullptr}};
  const Ptr3C U = {{a.U[0], a.U[1], a.U[2]}}, US = {{a.US[0], a.US[1], a.US[2]}};
  const Ptr3C K1 = {{a.K1[0], a.K1[1], a.K1[2]}}, K2 = {{a.K2[0], a.K2[1], a.K2[2]}};
  const Ptr3 dUS = {{a.US[0], a.US[1], a.US[2]}}, dU = {{a.U[0], a.U[1], a.U[2]}};
  for (int j = 1; j <= a.n; ++j) {
    // U* = CN_half(U, dt/4)   (steppers.py:160)
    if (!cn_cluster_body<true>(K, 1, a.rg, a.cap, U, none, none, 0.0, a.alpha, a.eps, a.phibar,
                               a.nbt, a.cft, 0, dUS, a.max_iter, a.tol, 0.0, a.halfq, a.iters,
                               a.flags, a.counter, a.resid, a.fail, dsm, sh))
      return;  // the host reruns the sweep on the per-step path, which raises
    // Heun on N (steppers.py:162-166): K1 = N(U*), MID = U* + dt K1
    chain_nonlinear(a, 0, cl, c, dsm);
    for (int k = k0 + tid; k < k1; k += CC_NT) {
      // k_tend_finish: d = curl - lap(ke) (dynamics.py:151)
      const double2 ke2 = __ldcg(reinterpret_cast<const double2 *>(a.TMP) + k);
      const double l = a.lap[k];
      double2 d = ldx2<true>(a.K1[2], k);
      d = make_double2(d.x - ke2.x * l, d.y - ke2.y * l);
      st2(a.K1[2], k, d);
      // k_axpy3: MID = U* + dt K1
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        const double2 t = f == 2 ? d : ldx2<true>(a.K1[f], k);
        st2(a.MID[f], k, add2(ldx2<true>(a.US[f], k), sc2(a.dt, t)));
      }
    }
    cl.sync();
    chain_nonlinear(a, 1, cl, c, dsm);
    for (int k = k0 + tid; k < k1; k += CC_NT) {
      const double2 ke2 = __ldcg(reinterpret_cast<const double2 *>(a.TMP) + k);
      const double l = a.lap[k];
      double2 d = ldx2<true>(a.K2[2], k);
      d = make_double2(d.x - ke2.x * l, d.y - ke2.y * l);
      st2(a.K2[2], k, d);
    }
    // U = visc(CN_half(U* + dt/2 (K1 + K2)))   (steppers.py:167-168); reads own rows only
    if (!cn_cluster_body<true>(K, 1, a.rg, a.cap, US, K1, K2, 0.5 * a.dt, a.alpha, a.eps,
                               a.phibar, a.nbt, a.cft, 0, dU, a.max_iter, a.tol, a.dtnu, a.halfq,
                               a.iters, a.flags, a.counter, a.resid, a.fail, dsm, sh))
      return;
    // forcing (k_add_col) and u[j] in the reference's packed layout (k_to_boundary)
    for (int k = k0 + tid; k < k1; k += CC_NT) {
      const int kb = a.iperm[k];
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        double2 v = ldx2<true>(a.U[f], k);
        if (a.g) {
          v = add2(v, ldx2<true>(a.g + (size_t)f * K * 2 * a.n, (size_t)k * a.n + (j - 1)));
          st2(a.U[f], k, v);
        }
        reinterpret_cast<double2 *>(a.u)[((size_t)j * 3 + f) * K + kb] = v;
      }
    }
    // the next step's first phase reads only this CTA's own rows of U and starts
    // with a cluster barrier (cn_cluster_body)
  }
}

}  // namespace

int chain_smem(int N2, int cap) {
  return (int)std::max<size_t>((size_t)6 * cap * sizeof(double2),
                               (size_t)N2 * 16 * sizeof(double2));
}

bool chain_ok(int C, int smem) {
  static std::vector<int3> cache;  // (C, smem, ok)
  static int attr_smem = 0;        // the attribute only grows (plans of other truncations)
  for (const int3 &e : cache)
    if (e.x == C && e.y == smem) return e.z != 0;
  int ok = 0;
  if ((smem <= attr_smem ||
       cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) ==
           cudaSuccess) &&
      (C <= 8 ||
       cudaFuncSetAttribute(k_chain, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
           cudaSuccess)) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(CC_NT);
    cfg.dynamicSmemBytes = smem;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, k_chain, &cfg) == cudaSuccess && nc > 0) ok = 1;
    attr_smem = std::max(attr_smem, smem);
  }
  cudaGetLastError();
  cache.push_back(make_int3(C, smem, ok));
  return ok != 0;
}

int chain_launch(const ChainArgs *dev_args, int C, int smem, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(CC_NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  SWE_CUDA(cudaLaunchKernelEx(&cfg, k_chain, dev_args));
  SWE_LAUNCH_CHECK();
  return OK;
}

}  // namespace swe
