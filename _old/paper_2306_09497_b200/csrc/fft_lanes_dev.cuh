// Device code of the "lane = row" longitude FFT (see fft_lanes.cu), shared by the
// FFT kernels (fft_lanes.cu) and any kernel that fuses the pass.  CG
// (lane_load_eo): the E/O inputs are read through L2 (ld.global.cg), for inputs
// produced earlier in the same kernel.
#pragma once
#include <cooperative_groups.h>

#include <algorithm>

#include "fft.cuh"
#include "fft_core.cuh"

namespace cg = cooperative_groups;

namespace swe {

using namespace fftcore;

namespace {

// LW rows per CTA.  16: a half-warp covers them, each warp runs two butterflies per
// instruction and two CTAs fit on an SM (N2 <= 907).  8: longer rows (N2 <= 1815,
// e.g. M = 1024), one 512-thread CTA per SM; the 14-row nonlinear pass is then split
// by hemisphere over a two-CTA cluster that combines F+- through distributed shared
// memory.
constexpr int GT = 4;  // generic radix: output pairs (t, R - t) per thread item

// Shared-memory position of (slot, row): the 16 rows of a slot stay one 256-byte
// line, permuted by the slot (XOR swizzle), so that accesses to one row across
// consecutive slots (put_z, the grid products, extraction) spread over the banks
// while a butterfly's 16 (or 8) rows of one slot remain a conflict-free line.
//
// 16 rows: 2*slot (4 aligned consecutive slots x 2 hemispheres of one field hit 8
// distinct 16-byte bank groups in the grid products) plus bit 2 of the slot in bit 0,
// so rows (2f + h) of one hemisphere land on both bank parities across scattered
// slots (put_z stores and the F+- extraction read one hemisphere's rows of several
// slots per instruction); other widths keep slot << 1.
template <int LW>
SWE_DEV int swz(int slot) {
  return LW == 16 ? (((slot << 1) | ((slot >> 2) & 1)) & 15) : ((slot << 1) & (LW - 1));
}
template <int LW>
SWE_DEV int xs(int slot, int row) { return slot * LW + (row ^ swz<LW>(slot)); }

// MODE 0 DIT, 1 DIF, 2 prime-factor (no twiddles); see fft.cu.  RW rows take part
// (RW lanes per butterfly, 32/RW butterflies per warp instruction).
template <int R, int MODE, int RW, int LW>
SWE_DEV void lane_stage(double2 *X, int N2, int Lp, double dir, const double2 *tw, int warp,
                        int nw, int lane) {
  constexpr int H = (R - 1) / 2, BW = 32 / RW;
  double cr[H + 1], sr[H + 1];
  if constexpr (R != 2 && R != 4) {
#pragma unroll
    for (int e = 0; e <= H; ++e) {
      const double2 w = __ldg(tw + e * (N2 / R));
      cr[e] = w.x;
      sr[e] = w.y;
    }
  }
  const int L = Lp * R, nbf = N2 / R, tws = N2 / L;
  const int row = lane & (RW - 1);
  const float inv_lp = 1.0f / (float)Lp;  // exact quotient for bf < 2^12 (N2 <= 4096)
  for (int bf = BW * warp + lane / RW; bf < nbf; bf += BW * nw) {
    const int g = (int)(((float)bf + 0.5f) * inv_lp), k = bf - g * Lp, base = g * L + k;
    double2 v[R], y[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      v[q] = X[xs<LW>(base + q * Lp, row)];
      if (MODE == 0 && q && k) v[q] = cm(v[q], twd(tw, q * k * tws, dir));
    }
    dft<R>(v, dir, cr, sr, y);
#pragma unroll
    for (int t = 0; t < R; ++t)
      X[xs<LW>(base + t * Lp, row)] =
          (MODE == 1 && t && k) ? cm(y[t], twd(tw, t * k * tws, dir)) : y[t];
  }
}

// Any odd radix R, CTA-wide (call with every thread, between barriers).  The same
// sums as dft<R>: with S_q = v_q + v_{R-q}, D_q = v_q - v_{R-q} (q = 1..H),
//   y_t, y_{R-t} = v_0 + sum_q S_q cos(2 pi q t / R) -+ dir i sum_q D_q sin(...)
// Thread item (butterfly, group of GT consecutive t in 0..H, row): a round takes as
// many whole butterflies as the CTA holds items for, reads their inputs, then (after
// a barrier) overwrites them in place.  ct = shared (cos, sin)(2 pi e / R), e < R.
template <int MODE, int RW, int LW>
SWE_DEV void lane_stage_gen(double2 *X, double2 *ct, int N2, int Lp, int R, double dir,
                            const double2 *tw, int tid, int nthr) {
  for (int e = tid; e < R; e += nthr) ct[e] = __ldg(tw + e * (N2 / R));
  __syncthreads();
  const int H = (R - 1) / 2, G = (H + GT) / GT;
  const int L = Lp * R, nbf = N2 / R, tws = N2 / L;
  const int row = tid % RW, item = tid / RW, bpr = (nthr / RW) / G;
  const int bl = item / G, grp = item - bl * G;
  for (int b0 = 0; b0 < nbf; b0 += bpr) {
    const int bf = b0 + bl;
    const bool act = bl < bpr && bf < nbf;
    double re[GT], im[GT], sx[GT], sy[GT];
    int e[GT];
    int base = 0, k = 0;
    if (act) {
      const int g = bf / Lp;
      k = bf - g * Lp;
      base = g * L + k;
      const double2 v0 = X[xs<LW>(base, row)];
#pragma unroll
      for (int j = 0; j < GT; ++j) {
        re[j] = v0.x;
        im[j] = v0.y;
        sx[j] = 0.0;
        sy[j] = 0.0;
        e[j] = 0;
      }
      for (int q = 1; q <= H; ++q) {
        double2 p = X[xs<LW>(base + q * Lp, row)], m = X[xs<LW>(base + (R - q) * Lp, row)];
        if (MODE == 0 && k) {
          p = cm(p, twd(tw, q * k * tws, dir));
          m = cm(m, twd(tw, (R - q) * k * tws, dir));
        }
        const double Sx = p.x + m.x, Sy = p.y + m.y, Dx = p.x - m.x, Dy = p.y - m.y;
#pragma unroll
        for (int j = 0; j < GT; ++j) {
          e[j] += grp * GT + j;
          if (e[j] >= R) e[j] -= R;
          const double2 w = ct[e[j]];
          re[j] = fma(Sx, w.x, re[j]);
          im[j] = fma(Sy, w.x, im[j]);
          sx[j] = fma(Dx, w.y, sx[j]);
          sy[j] = fma(Dy, w.y, sy[j]);
        }
      }
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int j = 0; j < GT; ++j) {
        const int t = grp * GT + j;
        if (t > H) break;
        double2 y = make_double2(re[j] - dir * sy[j], im[j] + dir * sx[j]);
        if (MODE == 1 && t && k) y = cm(y, twd(tw, t * k * tws, dir));
        X[xs<LW>(base + t * Lp, row)] = y;
        if (t) {
          double2 y2 = make_double2(re[j] + dir * sy[j], im[j] - dir * sx[j]);
          if (MODE == 1 && k) y2 = cm(y2, twd(tw, (R - t) * k * tws, dir));
          X[xs<LW>(base + (R - t) * Lp, row)] = y2;
        }
      }
    }
    __syncthreads();
  }
}

// Radix set of a kernel instantiation (RM): bit r_bit(R) for each unrolled radix it
// contains, RM_PFA / RM_CT when the transform kind is known; RM = 0: every radix,
// kind chosen at run time.  A launch of few CTAs (a single-slice coarse step) runs
// each stage body once, so it pays the instruction fetch of all code it contains:
// the factorisations of the hot levels get kernels holding only their stages.
constexpr int r_bit(int R) {
  return R == 2 ? 1 : R == 3 ? 2 : R == 4 ? 4 : R == 5 ? 8 : R == 7 ? 16 : R == 11 ? 32 : R == 13 ? 64 : 0;
}
constexpr int RM_PFA = 128, RM_CT = 256;
constexpr bool rm_ok(int RM, int R) { return RM == 0 || (RM & r_bit(R)) != 0; }

// one stage over rows 0..RW-1, ends with a CTA barrier.  GEN: the length has a
// non-unrolled radix (kernels without it keep the small-radix register budget)
template <int MODE, int RW, int LW, bool GEN, int RM = 0>
SWE_DEV void lane_run_stage(double2 *X, double2 *ct, int N2, int Lp, int R, double dir,
                            const double2 *tw, int tid, int nthr) {
  const int warp = tid >> 5, nw = nthr >> 5, lane = tid & 31;
  switch (R) {
    case 2: if constexpr (rm_ok(RM, 2)) lane_stage<2, MODE, RW, LW>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    case 3: if constexpr (rm_ok(RM, 3)) lane_stage<3, MODE, RW, LW>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    case 4: if constexpr (rm_ok(RM, 4)) lane_stage<4, MODE, RW, LW>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    case 5: if constexpr (rm_ok(RM, 5)) lane_stage<5, MODE, RW, LW>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    case 7: if constexpr (rm_ok(RM, 7)) lane_stage<7, MODE, RW, LW>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    // (with a generic radix in the length, 11 and 13 go generic too: their unrolled
    // register footprint next to the generic stage would spill)
    case 11:
      if constexpr (!GEN) {
        if constexpr (rm_ok(RM, 11)) lane_stage<11, MODE, RW, LW>(X, N2, Lp, dir, tw, warp, nw, lane);
        break;
      }
    case 13:
      if constexpr (!GEN) {
        if constexpr (rm_ok(RM, 13)) lane_stage<13, MODE, RW, LW>(X, N2, Lp, dir, tw, warp, nw, lane);
        break;
      }
    default:
      if constexpr (GEN) {
        lane_stage_gen<MODE, RW, LW>(X, ct, N2, Lp, R, dir, tw, tid, nthr);
        return;
      }
      break;
  }
  __syncthreads();
}

struct LCtx {
  double2 *X, *ct;
  int p, jn, js, eq, b0, nsl, S, tid, nthr;
  int pin;  // row of the E/O input planes holding pair p (= p in fft_lanes.cu)
  int split, hem;  // split: this CTA holds only hemisphere hem's rows (row = f*S + s)
};

SWE_DEV int lrow(const LCtx &c, int f, int h, int s) {
  return c.split ? f * c.S + s : (f * 2 + h) * c.S + s;
}

// prime-factor (no twiddles) or Cooley-Tukey: fixed by RM or read from a.pfa
template <int RM>
SWE_DEV bool rm_pfa(const FftArgs &a) {
  return (RM & RM_PFA) ? true : (RM & RM_CT) ? false : a.pfa != 0;
}

template <int LW, bool GEN, int RM = 0>
SWE_DEV void lane_ifft(const FftArgs &a, const LCtx &c) {
  int Lp = 1;
  for (int s = 0; s < a.nst; ++s) {
    if (rm_pfa<RM>(a)) {
      if constexpr (!(RM & RM_CT))
        lane_run_stage<2, LW, LW, GEN, RM>(c.X, c.ct, a.N2, Lp, a.radix[s], 1.0, a.tw, c.tid, c.nthr);
    } else {
      if constexpr (!(RM & RM_PFA))
        lane_run_stage<0, LW, LW, GEN, RM>(c.X, c.ct, a.N2, Lp, a.radix[s], 1.0, a.tw, c.tid, c.nthr);
    }
    Lp *= a.radix[s];
  }
}

// forward transform of rows 0..RW-1
template <int RW, int LW, bool GEN, int RM = 0>
SWE_DEV void lane_fft(const FftArgs &a, const LCtx &c) {
  if (rm_pfa<RM>(a)) {
    if constexpr (!(RM & RM_CT)) {
      int Lp = 1;
      for (int s = 0; s < a.nst; ++s) {
        lane_run_stage<2, RW, LW, GEN, RM>(c.X, c.ct, a.N2, Lp, a.radix[s], -1.0, a.tw, c.tid, c.nthr);
        Lp *= a.radix[s];
      }
    }
    return;
  }
  if constexpr (!(RM & RM_PFA)) {
    int L = a.N2;
    for (int s = a.nst - 1; s >= 0; --s) {
      const int R = a.radix[s];
      lane_run_stage<1, RW, LW, GEN, RM>(c.X, c.ct, a.N2, L / R, R, -1.0, a.tw, c.tid, c.nthr);
      L /= R;
    }
  }
}

// Z of one hemisphere row from its half spectrum X (see fft.cu build comment):
//   Z[k] = (X[k] + conj X[N2-k]) + i w^k (X[k] - conj X[N2-k])
// (w1, w2) = twh[k], twh[N2-k] and (z1, z2) = pos_z[k], pos_z[N2-k], prefetched
template <int LW>
SWE_DEV void put_z(const LCtx &c, int row, int k, int k2, double2 Xk, double2 Xc, double2 w1,
                   double2 w2, int z1, int z2) {
  if (k == 0) {
    c.X[xs<LW>(z1, row)] = make_double2(Xk.x, Xk.x);
    return;
  }
  const double2 A = make_double2(Xk.x + Xc.x, Xk.y - Xc.y);
  const double2 D = make_double2(Xk.x - Xc.x, Xk.y + Xc.y);
  const double2 Bk = cm(D, w1);
  c.X[xs<LW>(z1, row)] = make_double2(A.x - Bk.y, A.y + Bk.x);
  if (k2 != k) {
    const double2 A2 = make_double2(Xc.x + Xk.x, Xc.y - Xk.y);
    const double2 D2 = make_double2(Xc.x - Xk.x, Xc.y + Xk.y);
    const double2 B2 = cm(D2, w2);
    c.X[xs<LW>(z2, row)] = make_double2(A2.x - B2.y, A2.y + B2.x);
  }
}

// fields a.in[0..nf-1]: E/O half spectra [m][2][Jp][ld] of pair p -> Z of their north
// and south rows (only hemisphere c.hem when split).  One flattened loop over (k pair,
// slice, field), field fastest: the lanes of a warp store to the same slot of
// different rows (one line, no bank conflicts) and keep many loads in flight; field
// `subf` has phisub subtracted from E at m = 0 (phi_prime, dynamics.py:52-56).  With
// a.dlam, field 2 is i m times field 5 (d_lambda Phi).
// flattened (k, slice, field) item -> (k, s, f): field fastest, or with SF slice
// fastest (adjacent slices share 32-byte sectors of the [..][m][slice] layouts)
template <bool SF>
SWE_DEV void item_ksf(int idx, int nf, int S, int &k, int &s, int &f) {
  if constexpr (SF) {
    const int r = idx / S;
    s = idx - r * S;
    k = r / nf;
    f = r - k * nf;
  } else {
    const int r = idx / nf;
    f = idx - r * nf;
    k = r / S;
    s = r - k * S;
  }
}

// E and O of one pair-major (pair, m, slice) item: one 32-byte load (sm_100 256-bit LDG)
template <int CG>
SWE_DEV void ldg_eo(const double2 *p, double2 &e, double2 &o) {
  if constexpr (CG == 2) {
    e = p[0];
    o = p[1];
  } else if constexpr (CG == 1)
    asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(e.x), "=d"(e.y), "=d"(o.x), "=d"(o.y)
                 : "l"(p));
  else
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(e.x), "=d"(e.y), "=d"(o.x), "=d"(o.y)
                 : "l"(p));
}
// CG 0: read-only path, 1: through L2 (ld.global.cg), 2: generic (shared memory)
template <int CG>
SWE_DEV double2 ld_in(const double2 *p) {
  if constexpr (CG == 1) return __ldcg(p);
  else if constexpr (CG == 2) return *p;
  else return __ldg(p);
}

template <int LW, int CG = 0>
SWE_DEV void lane_load_eo(const FftArgs &a, const LCtx &c, int nf, int subf) {
  const int N2 = a.N2, M = a.M, npair = N2 / 2 + 1, S = c.S;
  const size_t eo = (size_t)a.Jp * a.ld / 2;  // E -> O offset (double2)
  const size_t mstride = 2 * eo;
  const int per = npair * S, total = nf * per;
  constexpr int U = 2;
  for (int i0 = c.tid; i0 < total; i0 += U * c.nthr) {
    double2 e[U], o[U], e2[U], o2[U], w1[U], w2[U];
    int z1[U], z2[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = i0 + u * c.nthr;
      int k, s, f;
      item_ksf<false>(idx, nf, S, k, s, f);
      const bool ok = idx < total && s < c.nsl;
      const int k2 = k == 0 ? N2 : N2 - k;
      const double2 z = make_double2(0.0, 0.0);
      const int fs = (f == 2 && a.dlam) ? 5 : f;
      const double2 *pk, *pk2;
      size_t eoo;
      if (a.in_pm) {  // [Jh][M+1][ld/2][E,O]: one (pair, m, slice) is one 32-byte E/O item
        const int nsl = a.ld >> 1;
        const double2 *blk = reinterpret_cast<const double2 *>(a.in[ok ? fs : 0]) +
                             ((size_t)c.p * (M + 1) * nsl + c.b0 + s) * 2;
        pk = blk + (size_t)2 * nsl * k;
        pk2 = blk + (size_t)2 * nsl * k2;
        eoo = 1;
      } else {
        const double2 *base =
            reinterpret_cast<const double2 *>(a.in[ok ? fs : 0] + (size_t)c.pin * a.ld) + c.b0;
        pk = base + (size_t)k * mstride + s;
        pk2 = base + (size_t)k2 * mstride + s;
        eoo = eo;
      }
      if (a.v4ld) {
        e[u] = o[u] = e2[u] = o2[u] = z;
        if (ok && k <= M) ldg_eo<CG>(pk, e[u], o[u]);
        if (ok && k2 <= M) ldg_eo<CG>(pk2, e2[u], o2[u]);
      } else {
        e[u] = (ok && k <= M) ? ld_in<CG>(pk) : z;
        o[u] = (ok && k <= M) ? ld_in<CG>(pk + eoo) : z;
        e2[u] = (ok && k2 <= M) ? ld_in<CG>(pk2) : z;
        o2[u] = (ok && k2 <= M) ? ld_in<CG>(pk2 + eoo) : z;
      }
      w1[u] = ok ? __ldg(a.twh + k) : z;
      w2[u] = (ok && k) ? __ldg(a.twh + k2) : z;
      z1[u] = ok ? __ldg(a.pos_z + k) : 0;
      z2[u] = (ok && k) ? __ldg(a.pos_z + k2) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = i0 + u * c.nthr;
      int k, s, f;
      item_ksf<false>(idx, nf, S, k, s, f);
      if (idx >= total || s >= c.nsl) continue;
      if (f == subf && k == 0) e[u].x -= a.phisub[c.b0 + s];
      const int k2 = N2 - k;
      if (f == 2 && a.dlam) {  // i m X (m = k for e/o, N2 - k for e2/o2)
        const double mk = k, mk2 = k2;
        e[u] = make_double2(-mk * e[u].y, mk * e[u].x);
        o[u] = make_double2(-mk * o[u].y, mk * o[u].x);
        e2[u] = make_double2(-mk2 * e2[u].y, mk2 * e2[u].x);
        o2[u] = make_double2(-mk2 * o2[u].y, mk2 * o2[u].x);
      }
      if (!c.split || c.hem == 0)
        put_z<LW>(c, lrow(c, f, 0, s), k, k2, make_double2(e[u].x + o[u].x, e[u].y + o[u].y),
                  make_double2(e2[u].x + o2[u].x, e2[u].y + o2[u].y), w1[u], w2[u], z1[u],
                  z2[u]);
      if (!c.split || c.hem == 1)
        put_z<LW>(c, lrow(c, f, 1, s), k, k2, make_double2(e[u].x - o[u].x, e[u].y - o[u].y),
                  make_double2(e2[u].x - o2[u].x, e2[u].y - o2[u].y), w1[u], w2[u], z1[u],
                  z2[u]);
    }
  }
}

// grid sample n of row r lives in X[pos_g[n/2]][r].{x,y}
template <int LW>
SWE_DEV double &gval(const FftArgs &a, const LCtx &c, int n, int row) {
  double *p = reinterpret_cast<double *>(c.X + xs<LW>(__ldg(a.pos_g + (n >> 1)), row));
  return p[n & 1];
}
template <int LW>
SWE_DEV double &gslot(const LCtx &c, int p, int h, int row) {
  return reinterpret_cast<double *>(c.X + xs<LW>(p, row))[h];
}

template <int LW>
SWE_DEV void lane_load_grid(const FftArgs &a, const LCtx &c, const double *src, int f) {
  for (int h = 0; h < 2; ++h) {
    const int j = (h && !c.eq) ? c.js : c.jn;
    for (int s = 0; s < c.nsl; ++s) {
      const double *g = src + ((size_t)(c.b0 + s) * a.J + j) * a.I;
      for (int n = c.tid; n < a.I; n += c.nthr) gval<LW>(a, c, n, lrow(c, f, h, s)) = __ldg(g + n);
    }
  }
}

template <int LW>
SWE_DEV void lane_store_grid(const FftArgs &a, const LCtx &c, double *dst, int f, double scale) {
  for (int h = 0; h < 2 - c.eq; ++h) {
    const int j = h ? c.js : c.jn;
    for (int s = 0; s < c.nsl; ++s) {
      double *g = dst + ((size_t)(c.b0 + s) * a.J + j) * a.I;
      for (int n = c.tid; n < a.I; n += c.nthr) g[n] = gval<LW>(a, c, n, lrow(c, f, h, s)) * scale;
    }
  }
}

// fm[k] (k = 0..M) of row `row` of the buffer X: fm = (Ge + w^{-k} Go) / I, see
// fft.cu; (z1, z2) = slots of Z[k], Z[N2-k]; w = conj twh[k].  X may be a peer
// CTA's shared memory (cluster address).
template <int LW>
SWE_DEV double2 row_fm(const double2 *X, int row, int z1, int z2, double2 w) {
  const double2 zk = X[xs<LW>(z1, row)];
  const double2 zc = X[xs<LW>(z2, row)];
  const double2 Sg = make_double2(zk.x + zc.x, zk.y - zc.y);
  const double2 D = make_double2(zk.y + zc.y, -(zk.x - zc.x));
  const double2 t = cm(w, D);
  return make_double2(Sg.x + t.x, Sg.y + t.y);  // 2 * I * fm
}

// fields 0..nf-1 -> a.out[f] as F+ = scale (fm_N + fm_S), F- = scale (fm_N - fm_S)
// ([m][2][Jp][ld]), scaled by w01 (fields 0, 1) or w23 (2, 3); one flattened loop.
// XN / XS hold the north / south rows (the same buffer unless split); items
// i0, i0 + istep, ... of the (k, slice, field) range.
// F+- of (field f, order k, slice s) handed to store(f, k, s, F+, F-)
template <int LW, class Store>
SWE_DEV void lane_extract_to(const FftArgs &a, const LCtx &c, const double2 *XN, const double2 *XS,
                             int nf, double w01, double w23, int i0, int istep, Store store) {
  const int M = a.M, S = c.S, N2 = a.N2, per = (M + 1) * S;
  for (int idx = i0; idx < nf * per; idx += istep) {
    int k, s, f;
    item_ksf<false>(idx, nf, S, k, s, f);
    if (s >= c.nsl) continue;
    const int z1 = __ldg(a.pos_z + k), z2 = __ldg(a.pos_z + (k == 0 ? 0 : N2 - k));
    double2 w = __ldg(a.twh + k);
    w.y = -w.y;
    const double h = 0.5 * (f < 2 ? w01 : w23);
    const double2 fn = row_fm<LW>(XN, lrow(c, f, 0, s), z1, z2, w);
    if (c.eq) {
      const double2 v = make_double2(fn.x * h, fn.y * h);
      store(f, k, s, v, v);
    } else {
      const double2 fs = row_fm<LW>(XS, lrow(c, f, 1, s), z1, z2, w);
      store(f, k, s, make_double2((fn.x + fs.x) * h, (fn.y + fs.y) * h),
            make_double2((fn.x - fs.x) * h, (fn.y - fs.y) * h));
    }
  }
}

template <int LW>
SWE_DEV void lane_extract(const FftArgs &a, const LCtx &c, const double2 *XN, const double2 *XS,
                          int nf, double w01, double w23, int i0, int istep) {
  const size_t pm = (size_t)a.Jp * a.ld / 2;  // F+ -> F- offset (double2)
  lane_extract_to<LW>(a, c, XN, XS, nf, w01, w23, i0, istep,
                      [&](int f, int k, int s, double2 fp, double2 fm) {
                        double2 *d = reinterpret_cast<double2 *>(a.out[f] + (size_t)c.p * a.ld) +
                                     c.b0 + (size_t)k * 2 * pm + s;
                        d[0] = fp;
                        d[pm] = fm;
                      });
}

template <int LW>
constexpr int lane_threads() { return LW == 16 ? 256 : 512; }  // 8 rows: one CTA per SM

// slices per CTA (rows = fields x 2 hemispheres x slices; the LW = 8 nonlinear pass
// holds one hemisphere of one slice per CTA)
__host__ __device__ constexpr int lane_slices(int op, int lw) {
  return lw == 16 ? fft_lane_slices(op) : (op == FOP_NONLINEAR ? 1 : fft_lane_slices(op) / 2);
}

// FOP_NONLINEAR on one CTA's rows (no hemisphere split): nonlinear_advection +
// nonlinear_rest (dynamics.py:142-160).  in: 0 u, 1 v, 2 d_lambda Phi, 3 H.Phi, 4 xi,
// 5 Phi (phi_prime applied here), 6 delta; out: F+- of (tphi, ke, xi u cos, xi v cos)
// L2 prefetch of this CTA's 1/gridDim.x share of the pair-major E/O blocks
// ([Jh][M+1][ld/2][E,O], one contiguous block per pair and field) of the pair
// a.pf_pairs ahead: CTAs run in (slice, pair) order, so that pair's CTAs start about
// one wave later and find their scattered 32-byte E/O reads in L2 instead of HBM
SWE_DEV void lane_prefetch_eo(const FftArgs &a, const LCtx &c, int nf) {
  const int pp = c.p + a.pf_pairs;
  if (!a.pf_pairs || !a.in_pm || pp >= a.Jh || c.tid >= nf) return;
  const int fs = (c.tid == 2 && a.dlam) ? 5 : c.tid;
  if (c.tid == 2 && a.dlam) return;  // field 2 is formed from field 5
  const size_t blk = (size_t)(a.M + 1) * (a.ld >> 1) * 32;  // bytes per pair and field
  const size_t chunk = ((blk + gridDim.x - 1) / gridDim.x + 15) & ~(size_t)15;
  const size_t off = (size_t)blockIdx.x * chunk;
  if (off >= blk) return;
  const unsigned bytes = (unsigned)min(chunk, blk - off);
  const char *src = reinterpret_cast<const char *>(a.in[fs]) + (size_t)pp * blk + off;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

template <int LW, bool GEN, int CG, int RM, class Store>
SWE_DEV void lane_nonlinear_to(const FftArgs &a, const LCtx &c, Store store) {
  const int p = c.p, I = a.I, S = c.S;
  const double ia = a.inv_acos[p];
  lane_prefetch_eo(a, c, 7);
  lane_load_eo<LW, CG>(a, c, 7, 5);
  __syncthreads();
  lane_ifft<LW, GEN, RM>(a, c);
  const double cs = a.coslat[p];
  constexpr int NH = 2;  // hemispheres held by this CTA
  // lanes: (slot, hemisphere, x/y) fastest, so a half-warp reads one bank each
  for (int idx = c.tid; idx < I * NH * S; idx += c.nthr) {
    const int s = idx / (NH * I), r = idx - s * NH * I;
    const int pp = r / (2 * NH), h = (r >> 1) & 1, hh = r & 1;
    auto R = [&](int f) -> double & { return gslot<LW>(c, pp, hh, lrow(c, f, h, s)); };
    const double u = R(0) * ia, v = R(1) * ia, gx = R(2) * ia, gy = R(3) * ia;
    const double xi = R(4), ph = a.no_rest ? 0.0 : R(5), de = R(6);
    R(0) = -(u * gx + v * gy) - ph * de;   // -(V.grad Phi) - Phi' delta
    R(1) = 0.5 * (u * u + v * v);          // kinetic energy
    R(2) = (xi * u) * cs;                  // (xi u) cos
    R(3) = (xi * v) * cs;                  // (xi v) cos
  }
  __syncthreads();
  // only the 4 product fields x 2 hemispheres (S = 1)
  lane_fft<8 * lane_slices(FOP_NONLINEAR, LW), LW, GEN, RM>(a, c);
  const double w = a.wq[p] * a.inv_I, wv = a.wsin2[p] * a.inv_I * a.inv_a;
  lane_extract_to<LW>(a, c, c.X, c.X, 4, w, wv, c.tid, c.nthr, store);
}

template <int LW, bool GEN, int CG, int RM = 0>
SWE_DEV void lane_nonlinear(const FftArgs &a, const LCtx &c) {
  if (a.out_il) {
    // [m][Jp][slice][F+, F-]: one 32-byte store per (field, order, slice)
    const size_t nsl = a.ld >> 1;
    lane_nonlinear_to<LW, GEN, CG, RM>(a, c, [&](int f, int k, int s, double2 fp, double2 fm) {
      double *d = a.out[f] + (((size_t)k * a.Jp + c.p) * nsl + c.b0 + s) * 4;
      asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(d), "d"(fp.x), "d"(fp.y),
                   "d"(fm.x), "d"(fm.y)
                   : "memory");
    });
    return;
  }
  const size_t pm = (size_t)a.Jp * a.ld / 2;  // F+ -> F- offset (double2)
  lane_nonlinear_to<LW, GEN, CG, RM>(a, c, [&](int f, int k, int s, double2 fp, double2 fm) {
    double2 *d = reinterpret_cast<double2 *>(a.out[f] + (size_t)c.p * a.ld) + c.b0 +
                 (size_t)k * 2 * pm + s;
    d[0] = fp;
    d[pm] = fm;
  });
}

}  // namespace
}  // namespace swe
