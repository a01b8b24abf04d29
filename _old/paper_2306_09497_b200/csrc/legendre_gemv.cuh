// Few-slice Legendre "gemv" groups (see legendre.cu): one 8-lane group per
// (output, m, pair) dot product for the synthesis, per (output, mode row) for the
// analysis.  The dot-product cores take accessors for the table and input reads,
// so any kernel that reuses them runs the same arithmetic in the same order.
#pragma once
#include "legendre.cuh"

namespace swe {

constexpr int GV_L = 8;  // lanes per dot product group

// LDM 0: read-only path (__ldg), 1: through L2 (ld.global.cg, for inputs written
// earlier in the same kernel), 2: generic load (shared-memory copies)
template <int LDM, typename T>
SWE_DEV T gv_ld(const T *p) {
  if constexpr (LDM == 1) return __ldcg(p);
  else if constexpr (LDM == 2) return *p;
  else return __ldg(p);
}

// Synthesis dot products of group (output o, order m, latitude pair p): E and O sums
// (acc[0], acc[1]) over the mode rows of m, split over the 8 lanes (rows gl, gl + 8,
// ...), reduced by shuffles (every lane ends with the totals).  tab(ti, r) = table
// value of term ti at mode row r (this pair), src(ti, r, j) = its spectral input of
// slice j.
template <int NS, class Tab, class Src>
SWE_DEV void synth_group_core(const LegOut &o, int M, int m, int gl, const int *offsets, Tab tab,
                              Src src, double (&acc)[2][NS][2]) {
  const int km = M + 1 - m, ne = (km + 1) >> 1, no = km >> 1, off = offsets[m];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int j = 0; j < NS; ++j) acc[h][j][0] = acc[h][j][1] = 0.0;
  for (int ti = 0; ti < o.nterms; ++ti) {
    const LegTerm &T = o.t[ti];
    const double sgm = T.sign * (T.times_im ? (double)m : 1.0);
    for (int par = 0; par < 2; ++par) {
      const int nr = par ? no : ne, r0 = off + (par ? ne : 0), h = par ^ T.flip;
#pragma unroll 2
      for (int tt = gl; tt < nr; tt += GV_L) {
        const int r = r0 + tt;
        const double a = tab(ti, r);
        const double sc = sgm * (T.scale ? __ldg(T.scale + r) : 1.0);
#pragma unroll
        for (int j = 0; j < NS; ++j) {
          const double2 v = src(ti, r, j);
          double x = v.x;
          if (T.phi0 != nullptr && r == 0) x -= T.phi0[j];  // phi_prime (dynamics.py:52-56)
          // i m X: (re, im) -> (-im, re)
          const double bRe = T.times_im ? -v.y * sc : x * sc;
          const double bIm = T.times_im ? x * sc : v.y * sc;
          acc[h][j][0] = fma(a, bRe, acc[h][j][0]);
          acc[h][j][1] = fma(a, bIm, acc[h][j][1]);
        }
      }
    }
  }
#pragma unroll
  for (int w = GV_L / 2; w > 0; w >>= 1)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        acc[h][j][0] += __shfl_xor_sync(0xffffffffu, acc[h][j][0], w);
        acc[h][j][1] += __shfl_xor_sync(0xffffffffu, acc[h][j][1], w);
      }
}

// synthesis group gi of the standalone kernel (all 8 lanes of the group call it;
// gl = lane & 7); `live` false: the lanes take part in the shuffles only
template <int NS, int CG>
SWE_DEV void synth_gemv_group(const LegArgs &args, long long gi, int gl, bool live) {
  const int M = args.M, Jh = args.Jh, Jp = args.Jp, ld = args.ld;
  if (!live) gi = 0;
  const int p = (int)(gi % Jh);
  const long long q = gi / Jh;
  const int m = (int)(q % (M + 1)), oi = (int)(q / (M + 1));
  const LegOut &o = args.out[oi];
  double acc[2][NS][2];  // [E / O][slice][re / im]
  synth_group_core<NS>(
      o, M, m, gl, args.offsets, [&](int ti, int r) { return __ldg(o.t[ti].tab + (size_t)r * Jp + p); },
      [&](int ti, int r, int j) {
        return gv_ld<CG>(reinterpret_cast<const double2 *>(o.t[ti].src + (size_t)r * ld) + j);
      },
      acc);
  if (live && gl < NS) {  // lane j writes slice j
    const double z = m ? 1.0 : 0.0;  // irfft ignores Im of the mean bin (spharm.py:257)
    double *dE = o.dst + (size_t)m * 2 * Jp * ld, *dO = dE + (size_t)Jp * ld;
#pragma unroll
    for (int j = 0; j < NS; ++j)
      if (j == gl) {
        *reinterpret_cast<double2 *>(dE + (size_t)p * ld + 2 * j) =
            make_double2(acc[0][j][0], z * acc[0][j][1]);
        *reinterpret_cast<double2 *>(dO + (size_t)p * ld + 2 * j) =
            make_double2(acc[1][j][0], z * acc[1][j][1]);
      }
  }
}

// order m and parity of internal mode row k (binary search of the block offsets)
SWE_DEV void row_m_par(const int *offsets, int M, int k, int &m, int &par) {
  int lo = 0, hi = M;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (offsets[mid] <= k) lo = mid;
    else hi = mid - 1;
  }
  m = lo;
  const int km = M + 1 - m, ne = (km + 1) >> 1;
  par = (k - offsets[m]) >= ne;
}

// Analysis dot products of group (output o, mode row k of order m, parity par):
// sums over the latitude pairs split over the 8 lanes, reduced by shuffles.
// tab(ti, p) = table value of term ti at pair p (this row), f(ti, fsel, p, j) = the
// F+ (fsel 0) / F- (1) input of order m at pair p, slice j.
template <int NS, class Tab, class Fin>
SWE_DEV void anal_group_core(const LegOut &o, int m, int par, int Jh, int gl, Tab tab, Fin fin,
                             double (&acc)[NS][2]) {
#pragma unroll
  for (int j = 0; j < NS; ++j) acc[j][0] = acc[j][1] = 0.0;
  for (int ti = 0; ti < o.nterms; ++ti) {
    const LegTerm &T = o.t[ti];
    const int fsel = par ^ T.flip;  // 0: F+, 1: F-
    double s[NS][2];
#pragma unroll
    for (int j = 0; j < NS; ++j) s[j][0] = s[j][1] = 0.0;
#pragma unroll 2
    for (int p = gl; p < Jh; p += GV_L) {
      const double a = tab(ti, p) * (T.pscale ? __ldg(T.pscale + p) : 1.0);
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        const double2 v = fin(ti, fsel, p, j);
        s[j][0] = fma(a, v.x, s[j][0]);
        s[j][1] = fma(a, v.y, s[j][1]);
      }
    }
    // i m X: (re, im) -> (-m im, m re)
    const double fc = T.sign * (T.times_im ? (double)m : 1.0);
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      acc[j][0] += T.times_im ? -fc * s[j][1] : fc * s[j][0];
      acc[j][1] += T.times_im ? fc * s[j][0] : fc * s[j][1];
    }
  }
#pragma unroll
  for (int w = GV_L / 2; w > 0; w >>= 1)
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      acc[j][0] += __shfl_xor_sync(0xffffffffu, acc[j][0], w);
      acc[j][1] += __shfl_xor_sync(0xffffffffu, acc[j][1], w);
    }
}

// analysis group gi = (output, mode row k) of the standalone kernel
template <int NS, int CG>
SWE_DEV void anal_gemv_group(const LegArgs &args, int K, long long gi, int gl, bool live) {
  const int M = args.M, Jh = args.Jh, Jp = args.Jp, ld = args.ld;
  if (!live) gi = 0;
  const int k = (int)(gi % K), oi = (int)(gi / K);
  const LegOut &o = args.out[oi];
  int m, par;
  row_m_par(args.offsets, M, k, m, par);
  double acc[NS][2];
  anal_group_core<NS>(
      o, m, par, Jh, gl, [&](int ti, int p) { return __ldg(o.t[ti].tab + (size_t)k * Jp + p); },
      [&](int ti, int fsel, int p, int j) {
        const LegTerm &T = o.t[ti];
        const double *F = T.src + ((size_t)m * 2 + (fsel ^ T.swap_pm)) * Jp * ld;
        return gv_ld<CG>(reinterpret_cast<const double2 *>(F + (size_t)p * ld) + j);
      },
      acc);
  if (live)
#pragma unroll
    for (int j = 0; j < NS; ++j)
      if (j == gl)
        *reinterpret_cast<double2 *>(o.dst + (size_t)k * ld + 2 * j) =
            make_double2(acc[j][0], acc[j][1]);
}

}  // namespace swe
