// Crank-Nicolson half step on one thread-block cluster per slice (device body) and
// the per-mode helpers it shares with spectral.cu; included by spectral.cu (the
// standalone k_cn_cluster) and any kernel that fuses the half step.  CG:
// inputs produced earlier in the same kernel are read through L2 (ld.global.cg).
#pragma once
#include <cooperative_groups.h>

#include "spectral.cuh"

namespace swe {

namespace cg = cooperative_groups;


SWE_DEV double2 ld2(const double *p, size_t i) { return reinterpret_cast<const double2 *>(p)[i]; }
SWE_DEV void st2(double *p, size_t i, double2 v) { reinterpret_cast<double2 *>(p)[i] = v; }
SWE_DEV double2 sc2(double s, double2 v) { return make_double2(s * v.x, s * v.y); }
SWE_DEV double2 add2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

template <bool CG>
SWE_DEV double2 ldx2(const double *p, size_t i) {
  if constexpr (CG) return __ldcg(reinterpret_cast<const double2 *>(p) + i);
  else return ld2(p, i);
}

SWE_DEV unsigned long long sqmag_bits(double x, double y) {
  return (unsigned long long)__double_as_longlong(x * x + y * y);
}

template <bool CG>
SWE_DEV double2 comb(const Ptr3C &x0, const Ptr3C &x1, const Ptr3C &x2, double s, int f,
                     size_t i) {
  if (!x1.p[f]) return ldx2<CG>(x0.p[f], i);
  const double2 a = ldx2<CG>(x1.p[f], i), b = ldx2<CG>(x2.p[f], i);
  return add2(ldx2<CG>(x0.p[f], i), sc2(s, make_double2(a.x + b.x, a.y + b.y)));
}

// the standalone kernels keep their plain loads
SWE_DEV double2 comb(const Ptr3C &x0, const Ptr3C &x1, const Ptr3C &x2, double s, int f,
                     size_t i) {
  return comb<false>(x0, x1, x2, s, f, i);
}

// Whole Crank-Nicolson half step for mid-size truncations (K up to ~38k modes,
// the fine level M = 256): one thread-block CLUSTER per slice.  CTA c of the
// C-CTA cluster owns the whole m-blocks of modes [rg.k[c], rg.k[c+1]) (balanced
// split on block boundaries) and keeps Phi, xi, delta and the three rhs fields of
// them in shared memory for the whole half step, so HBM sees the inputs once and
// the result once instead of ~10 state passes.  The L_C recurrence couples
// (m, n -+ 1) inside one m-block only, so every neighbour is CTA-local; the
// per-slice convergence maxima are combined over the cluster through distributed
// shared memory (one cluster barrier per iteration).  Same per-mode arithmetic as
// k_cn_small / k_cn_start + k_helm + k_cn_finish, so the result is bitwise the
// multi-kernel one.
constexpr int CC_NT = 512, CC_CHUNK = 2400, CC_MPT = (CC_CHUNK + CC_NT - 1) / CC_NT, CC_MAXC = 16;
struct CcRanges {
  int k[CC_MAXC + 1];
};
// the balanced m-block split of a C-CTA cluster (spectral.cu); returns the largest
// range (0: a range exceeds CC_CHUNK)
int cn_cluster_ranges(int M, int C, CcRanges *rg);
struct CcShared {
  unsigned long long red[6][CC_NT / 32];
  unsigned long long part[2][8];                // residual exchange (cluster barrier)
  unsigned long long inbox[2][CC_MAXC][6];      // peers' maxima by iteration parity
  unsigned long long mbar[2];                   // inbox arrival barriers (bytes)
  int done;
};
SWE_DEV unsigned cc_smem(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
// 16 bytes into peer `rank`'s copy of the shared location `p`, counted in bytes on
// that peer's mbarrier `bar` (st.async: no cluster-wide barrier, no GPU-scope fence)
SWE_DEV void cc_send16(const void *p, const unsigned long long *bar, int rank,
                       unsigned long long a, unsigned long long b) {
  unsigned ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(cc_smem(p)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(cc_smem(bar)), "r"(rank));
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(ra),
      "l"(a), "l"(b), "r"(rb)
      : "memory");
}
SWE_DEV void cc_wait(const unsigned long long *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "CCW_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra CCW_%=;\n}\n" ::"r"(cc_smem(bar)),
      "r"(parity)
      : "memory");
}

// returns the slice's convergence (the same in every CTA of the cluster)
template <bool CG>
SWE_DEV bool cn_cluster_body(
    int K, int B, const CcRanges &rg, int cap, const Ptr3C &x0, const Ptr3C &x1, const Ptr3C &x2,
    double s, double alpha, const double *eps, const double *phibar, const int2 *nbt,
    const double4 *cft, int rhs_given, const Ptr3 &dst, int max_iter, double tol, double dtnu,
    double halfq, int *iters, int *flags, int *counter, double *resid, int *fail, double2 *ccm,
    CcShared &sh) {
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks(), c = (int)cl.block_rank();
  const int b = blockIdx.x / C, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k0 = rg.k[c], k1 = rg.k[c + 1], n = k1 - k0;
  double2 *P = ccm, *X = ccm + cap, *D = ccm + 2 * cap;
  double2 *R0 = ccm + 3 * cap, *R1 = ccm + 4 * cap, *R2 = ccm + 5 * cap;
  const bool cor = nbt != nullptr;
  const double pb = phibar[b], apb = alpha * pb, aap = alpha * alpha * pb;
  auto at = [&](int k) { return (size_t)k * B + b; };
  // neighbour j (global mode index): always inside this CTA's m-blocks
  auto nbr = [&](int j, int, double2 &xv, double2 &dv) {
    xv = X[j - k0];
    dv = D[j - k0];
  };
  auto lcop = [&](int k, int ver, double2 x, double2 d, double2 &lx, double2 &lc) {
    const int2 nb = nbt[k];
    const double4 cf = cft[k];
    double2 xl = make_double2(0.0, 0.0), dl = xl, xh = xl, dh = xl;
    if (nb.x >= 0) nbr(nb.x, ver, xl, dl);
    if (nb.y >= 0) nbr(nb.y, ver, xh, dh);
    lx = make_double2(-(cf.x * dl.x + cf.y * dh.x + cf.z * x.y),
                      -(cf.x * dl.y + cf.y * dh.y - cf.z * x.x));
    lc = make_double2(cf.x * xl.x + cf.y * xh.x - cf.z * d.y,
                      cf.x * xl.y + cf.y * xh.y + cf.z * d.x);
    if (cf.w != 0.0) {
      lx.y = 0.0;
      lc.y = 0.0;
    }
  };
  if (tid == 0) {
    for (int i = 0; i < 2; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cc_smem(&sh.mbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();  // peers' barriers initialised before any st.async reaches them
  // ---- version 0: X's xi / delta
  for (int kk = tid; kk < n; kk += CC_NT) {
    const double2 xv = comb<CG>(x0, x1, x2, s, 1, at(k0 + kk)), dv = comb<CG>(x0, x1, x2, s, 2, at(k0 + kk));
    X[kk] = xv;
    D[kk] = dv;
  }
  __syncthreads();
  // ---- rhs R and the first Helmholtz iterate (version 1)
  double2 vx[CC_MPT], vd[CC_MPT];
  double rden[CC_MPT];
#pragma unroll
  for (int j = 0; j < CC_MPT; ++j) {
    const int kk = tid + j * CC_NT, k = k0 + kk;
    if (kk >= n) break;
    const double2 ph = comb<CG>(x0, x1, x2, s, 0, at(k)), xi = X[kk], de = D[kk];
    const double e = eps[k];
    double2 r0, r1, r2;
    if (rhs_given) {
      r0 = ph;
      r1 = xi;
      r2 = de;
    } else {
      double2 lx = make_double2(0.0, 0.0), lc = lx;
      if (cor) lcop(k, 0, xi, de, lx, lc);
      const double2 lphi = make_double2(-pb * de.x, -pb * de.y);
      const double2 lde = add2(sc2(e, ph), lc);
      r0 = add2(ph, sc2(alpha, lphi));
      r1 = add2(xi, sc2(alpha, lx));
      r2 = add2(de, sc2(alpha, lde));
    }
    R0[kk] = r0;
    R1[kk] = r1;
    R2[kk] = r2;
    const double denom = 1.0 + aap * e;
    rden[j] = 1.0 / denom;  // the iterations divide by the reciprocal (ddiv_r, exact)
    const double2 nph = make_double2(ddiv_r(r0.x - apb * r2.x, denom, rden[j]),
                                     ddiv_r(r0.y - apb * r2.y, denom, rden[j]));
    const double ae = alpha * e;
    P[kk] = nph;
    vx[j] = r1;
    vd[j] = make_double2(r2.x + ae * nph.x, r2.y + ae * nph.y);
  }
  __syncthreads();  // reads of version 0 done
#pragma unroll
  for (int j = 0; j < CC_MPT; ++j) {
    const int kk = tid + j * CC_NT;
    if (kk >= n) break;
    X[kk] = vx[j];
    D[kk] = vd[j];
  }
  __syncthreads();
  // ---- fixed point (steppers.py:96-112), the slice's own loop over the cluster
  int it = 0, done = !cor, ver = 1;
  for (; !done && it < max_iter; ++it) {
    unsigned long long mx[6] = {0, 0, 0, 0, 0, 0};
    double2 vp[CC_MPT];
#pragma unroll
    for (int j = 0; j < CC_MPT; ++j) {
      const int kk = tid + j * CC_NT, k = k0 + kk;
      if (kk >= n) break;
      const double2 rp = R0[kk], r1 = R1[kk], r2 = R2[kk];
      const double e = eps[k];
      const double2 x = X[kk], d = D[kk];
      double2 lx, lc;
      lcop(k, ver, x, d, lx, lc);
      const double2 rx = add2(r1, sc2(alpha, lx)), rd = add2(r2, sc2(alpha, lc));
      const double denom = 1.0 + aap * e;
      const double2 ph = make_double2(ddiv_r(rp.x - apb * rd.x, denom, rden[j]),
                                      ddiv_r(rp.y - apb * rd.y, denom, rden[j]));
      const double ae = alpha * e;
      const double2 de = make_double2(rd.x + ae * ph.x, rd.y + ae * ph.y);
      const double2 o0 = P[kk];
      mx[0] = max(mx[0], sqmag_bits(ph.x, ph.y));
      mx[1] = max(mx[1], sqmag_bits(rx.x, rx.y));
      mx[2] = max(mx[2], sqmag_bits(de.x, de.y));
      mx[3] = max(mx[3], sqmag_bits(ph.x - o0.x, ph.y - o0.y));
      mx[4] = max(mx[4], sqmag_bits(rx.x - x.x, rx.y - x.y));
      mx[5] = max(mx[5], sqmag_bits(de.x - d.x, de.y - d.y));
      vp[j] = ph;
      vx[j] = rx;
      vd[j] = de;
    }
#pragma unroll
    for (int q = 0; q < 6; ++q)
      for (int o = 16; o > 0; o >>= 1) mx[q] = max(mx[q], __shfl_xor_sync(0xffffffffu, mx[q], o));
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 6; ++q) sh.red[q][warp] = mx[q];
    __syncthreads();  // local reads of version `ver` done, warp maxima staged
    ++ver;
#pragma unroll
    for (int j = 0; j < CC_MPT; ++j) {
      const int kk = tid + j * CC_NT;
      if (kk >= n) break;
      P[kk] = vp[j];
      X[kk] = vx[j];
      D[kk] = vd[j];
    }
    if (warp == 0) {
      // this CTA's 6 maxima -> every peer's inbox[it & 1][c] (3 x 16 bytes each); the
      // parity double buffer is safe: a peer can only reach iteration it + 2 after
      // this CTA has sent (so finished reading) iteration it + 1
      unsigned long long v[6];
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        v[q] = lane < CC_NT / 32 ? sh.red[q][lane] : 0ULL;
        for (int o = 16; o > 0; o >>= 1) v[q] = max(v[q], __shfl_xor_sync(0xffffffffu, v[q], o));
      }
      const int par = it & 1;
      if (C > 1) {  // a one-CTA "cluster" (coarse levels) already holds the slice maxima
        if (lane == 0) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                           cc_smem(&sh.mbar[par])),
                       "r"(48 * C)
                       : "memory");
        }
        if (lane < C)
#pragma unroll
          for (int q = 0; q < 6; q += 2)
            cc_send16(&sh.inbox[par][c][q], &sh.mbar[par], lane, v[q], v[q + 1]);
        cc_wait(&sh.mbar[par], (it >> 1) & 1);
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          v[q] = lane < C ? sh.inbox[par][lane][q] : 0ULL;
          for (int o = 16; o > 0; o >>= 1) v[q] = max(v[q], __shfl_xor_sync(0xffffffffu, v[q], o));
        }
      }
      if (lane == 0) {
        double w[6];
        for (int q = 0; q < 6; ++q) w[q] = sqrt(__longlong_as_double((long long)v[q]));  // as decide_slice
        double overall = fmax(fmax(w[0], w[1]), w[2]);
        if (isnan(w[0]) || isnan(w[1]) || isnan(w[2])) overall = nan("");
        overall = (overall > 1e-300 || isnan(overall)) ? overall : 1e-300;
        bool ok = true;
        for (int f = 0; f < 3; ++f) {
          const double tiny = 1e-13 * overall;
          const double scale = (w[f] >= tiny || isnan(w[f])) ? w[f] : tiny;
          if (w[3 + f] > tol * scale) ok = false;
        }
        sh.done = ok;
      }
    }
    __syncthreads();
    done = sh.done;
  }
  if (c == 0 && tid == 0) {
    iters[b] = it;
    flags[b] = !done;
    resid[b] = 0.0;
  }
  if (!done) {
    // residual |u - alpha (L_G + L_C) u - rhs| (steppers.py:113-118)
    double rmax = 0.0;
    for (int kk = tid; kk < n; kk += CC_NT) {
      const int k = k0 + kk;
      const double2 x = X[kk], d = D[kk], ph = P[kk];
      double2 lx, lc;
      lcop(k, ver, x, d, lx, lc);
      const double2 lph = make_double2(-pb * d.x, -pb * d.y);
      const double2 lde = add2(sc2(eps[k], ph), lc);
      const double2 v[3] = {ph, x, d}, l[3] = {lph, lx, lde}, rr[3] = {R0[kk], R1[kk], R2[kk]};
      for (int f = 0; f < 3; ++f)
        rmax = fmax(rmax, hypot(v[f].x - alpha * l[f].x - rr[f].x, v[f].y - alpha * l[f].y - rr[f].y));
    }
    unsigned long long u = (unsigned long long)__double_as_longlong(rmax);
    for (int o = 16; o > 0; o >>= 1) u = max(u, __shfl_xor_sync(0xffffffffu, u, o));
    if (lane == 0) sh.red[0][warp] = u;
    __syncthreads();
    if (warp == 0) {
      u = lane < CC_NT / 32 ? sh.red[0][lane] : 0ULL;
      for (int o = 16; o > 0; o >>= 1) u = max(u, __shfl_xor_sync(0xffffffffu, u, o));
      if (lane == 0) sh.part[0][6] = u;
    }
    cl.sync();
    if (c == 0 && warp == 0) {
      u = lane < C ? cl.map_shared_rank(&sh, lane)->part[0][6] : 0ULL;
      for (int o = 16; o > 0; o >>= 1) u = max(u, __shfl_xor_sync(0xffffffffu, u, o));
      if (lane == 0) {
        resid[b] = __longlong_as_double((long long)u);
        atomicAdd(counter, 1);
        if (fail) *fail = 1;
      }
    }
  }
  // ---- epilogue: viscosity factor (dynamics.py:191-200) and the result
  for (int kk = tid; kk < n; kk += CC_NT) {
    const int k = k0 + kk;
    double bh = 1.0;
    if (dtnu != 0.0 && done) bh = 1.0 / (1.0 + dtnu * pow(eps[k], halfq));
    const double2 ph = P[kk], x = X[kk], d = D[kk];
    st2(dst.p[0], at(k), dtnu != 0.0 && done ? sc2(bh, ph) : ph);
    st2(dst.p[1], at(k), dtnu != 0.0 && done ? sc2(bh, x) : x);
    st2(dst.p[2], at(k), dtnu != 0.0 && done ? sc2(bh, d) : d);
  }
  cl.sync();  // peers may still read this CTA's maxima
  return done;
}


}  // namespace swe
