// Longitude FFT stage, "lane = row" variant for small-radix lengths.
//
// One CTA owns one latitude PAIR p (north row p, south row J-1-p) and S
// slices; its 16 transform rows are (field, hemisphere, slice), row index
// (f*2 + h)*S + s.  Shared memory holds X[slot][16]: the 16 rows of one slot
// form one 256-byte line, half-warp lane r works on row r, every butterfly
// access is a conflict-free full line and a half-warp shares its twiddles.
// Inputs are the parity-split Legendre outputs E/O ([m][2][Jp][ld]):
// north = E + O, south = E - O.  Outputs are the folded analysis inputs
// F+- = w (f_north +- f_south) ([m][2][Jp][ld]); on the equator (J odd) the
// south row coincides with the north row and F+ = F- = w f_north.
// Transform algebra (real packing, Cooley-Tukey / prime-factor, slot maps) is
// shared with fft.cu.
#include "fft.cuh"
#include "fft_core.cuh"

namespace swe {

using namespace fftcore;

namespace {

constexpr int LW = 16;  // rows per CTA: a half-warp covers them, so each warp runs two
                        // butterflies per instruction and two CTAs fit on an SM

// Shared-memory position of (slot, row): the 16 rows of a slot stay one 256-byte
// line, permuted by the slot (XOR swizzle), so that accesses to one row across
// consecutive slots (put_z, the grid products, extraction) spread over the banks
// while a butterfly's 16 (or 8) rows of one slot remain a conflict-free line.
SWE_DEV int xs(int slot, int row) { return slot * LW + (row ^ ((slot << 1) & (LW - 1))); }

// MODE 0 DIT, 1 DIF, 2 prime-factor (no twiddles); see fft.cu.  RW rows take part
// (RW lanes per butterfly, 32/RW butterflies per warp instruction).
template <int R, int MODE, int RW>
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
      v[q] = X[xs(base + q * Lp, row)];
      if (MODE == 0 && q && k) v[q] = cm(v[q], twd(tw, q * k * tws, dir));
    }
    dft<R>(v, dir, cr, sr, y);
#pragma unroll
    for (int t = 0; t < R; ++t)
      X[xs(base + t * Lp, row)] = (MODE == 1 && t && k) ? cm(y[t], twd(tw, t * k * tws, dir)) : y[t];
  }
}

template <int MODE, int RW>
SWE_DEV void lane_run_stage(double2 *X, int N2, int Lp, int R, double dir, const double2 *tw,
                            int warp, int nw, int lane) {
  switch (R) {
    case 2: lane_stage<2, MODE, RW>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    case 3: lane_stage<3, MODE, RW>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    case 4: lane_stage<4, MODE, RW>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    case 5: lane_stage<5, MODE, RW>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    case 7: lane_stage<7, MODE, RW>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    case 11: lane_stage<11, MODE, RW>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    default: lane_stage<13, MODE, RW>(X, N2, Lp, dir, tw, warp, nw, lane); break;
  }
}

struct LCtx {
  double2 *X;
  int p, jn, js, eq, b0, nsl, S, tid, nthr, warp, lane, nw;
};

SWE_DEV int lrow(const LCtx &c, int f, int h, int s) { return (f * 2 + h) * c.S + s; }

SWE_DEV void lane_ifft(const FftArgs &a, const LCtx &c) {
  int Lp = 1;
  for (int s = 0; s < a.nst; ++s) {
    if (a.pfa) lane_run_stage<2, LW>(c.X, a.N2, Lp, a.radix[s], 1.0, a.tw, c.warp, c.nw, c.lane);
    else lane_run_stage<0, LW>(c.X, a.N2, Lp, a.radix[s], 1.0, a.tw, c.warp, c.nw, c.lane);
    Lp *= a.radix[s];
    __syncthreads();
  }
}

// forward transform of rows 0..RW-1
template <int RW = LW>
SWE_DEV void lane_fft(const FftArgs &a, const LCtx &c) {
  if (a.pfa) {
    int Lp = 1;
    for (int s = 0; s < a.nst; ++s) {
      lane_run_stage<2, RW>(c.X, a.N2, Lp, a.radix[s], -1.0, a.tw, c.warp, c.nw, c.lane);
      Lp *= a.radix[s];
      __syncthreads();
    }
    return;
  }
  int L = a.N2;
  for (int s = a.nst - 1; s >= 0; --s) {
    const int R = a.radix[s];
    lane_run_stage<1, RW>(c.X, a.N2, L / R, R, -1.0, a.tw, c.warp, c.nw, c.lane);
    L /= R;
    __syncthreads();
  }
}

// Z of one hemisphere row from its half spectrum X (see fft.cu build comment):
//   Z[k] = (X[k] + conj X[N2-k]) + i w^k (X[k] - conj X[N2-k])
// (w1, w2) = twh[k], twh[N2-k] and (z1, z2) = pos_z[k], pos_z[N2-k], prefetched
SWE_DEV void put_z(const LCtx &c, int row, int k, int k2, double2 Xk, double2 Xc, double2 w1,
                   double2 w2, int z1, int z2) {
  if (k == 0) {
    c.X[xs(z1, row)] = make_double2(Xk.x, Xk.x);
    return;
  }
  const double2 A = make_double2(Xk.x + Xc.x, Xk.y - Xc.y);
  const double2 D = make_double2(Xk.x - Xc.x, Xk.y + Xc.y);
  const double2 Bk = cm(D, w1);
  c.X[xs(z1, row)] = make_double2(A.x - Bk.y, A.y + Bk.x);
  if (k2 != k) {
    const double2 A2 = make_double2(Xc.x + Xk.x, Xc.y - Xk.y);
    const double2 D2 = make_double2(Xc.x - Xk.x, Xc.y + Xk.y);
    const double2 B2 = cm(D2, w2);
    c.X[xs(z2, row)] = make_double2(A2.x - B2.y, A2.y + B2.x);
  }
}

// fields a.in[0..nf-1]: E/O half spectra [m][2][Jp][ld] of pair p -> Z of their north
// and south rows.  One flattened loop over (k pair, slice, field), field fastest: the
// lanes of a warp store to the same slot of different rows (one 256-byte line, no
// bank conflicts) and keep many loads in flight; field `subf` has phisub subtracted from E at m = 0 (phi_prime,
// dynamics.py:52-56).  With a.dlam, field 2 is i m times field 5 (d_lambda Phi).
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
      const int r = idx / nf, f = idx - r * nf, k = r / S, s = r - k * S;
      const bool ok = idx < total && s < c.nsl;
      const int k2 = k == 0 ? N2 : N2 - k;
      const double2 z = make_double2(0.0, 0.0);
      const int fs = (f == 2 && a.dlam) ? 5 : f;
      const double2 *pk, *pk2;
      size_t eoo;
      if (a.in_pm) {  // [Jh][ld/2][M+1][E,O]: this (pair, slice) is one contiguous block
        const int nsl = a.ld >> 1;
        const double2 *blk = reinterpret_cast<const double2 *>(a.in[ok ? fs : 0]) +
                             ((size_t)c.p * (M + 1) * nsl + c.b0 + s) * 2;
        pk = blk + (size_t)2 * nsl * k;
        pk2 = blk + (size_t)2 * nsl * k2;
        eoo = 1;
      } else {
        const double2 *base =
            reinterpret_cast<const double2 *>(a.in[ok ? fs : 0] + (size_t)c.p * a.ld) + c.b0;
        pk = base + (size_t)k * mstride + s;
        pk2 = base + (size_t)k2 * mstride + s;
        eoo = eo;
      }
      e[u] = (ok && k <= M) ? __ldg(pk) : z;
      o[u] = (ok && k <= M) ? __ldg(pk + eoo) : z;
      e2[u] = (ok && k2 <= M) ? __ldg(pk2) : z;
      o2[u] = (ok && k2 <= M) ? __ldg(pk2 + eoo) : z;
      w1[u] = ok ? __ldg(a.twh + k) : z;
      w2[u] = (ok && k) ? __ldg(a.twh + k2) : z;
      z1[u] = ok ? __ldg(a.pos_z + k) : 0;
      z2[u] = (ok && k) ? __ldg(a.pos_z + k2) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = i0 + u * c.nthr;
      const int r = idx / nf, f = idx - r * nf, k = r / S, s = r - k * S;
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
      put_z(c, lrow(c, f, 0, s), k, k2, make_double2(e[u].x + o[u].x, e[u].y + o[u].y),
            make_double2(e2[u].x + o2[u].x, e2[u].y + o2[u].y), w1[u], w2[u], z1[u], z2[u]);
      put_z(c, lrow(c, f, 1, s), k, k2, make_double2(e[u].x - o[u].x, e[u].y - o[u].y),
            make_double2(e2[u].x - o2[u].x, e2[u].y - o2[u].y), w1[u], w2[u], z1[u], z2[u]);
    }
  }
}

// grid sample n of row r lives in X[pos_g[n/2]][r].{x,y}
SWE_DEV double &gval(const FftArgs &a, const LCtx &c, int n, int row) {
  double *p = reinterpret_cast<double *>(c.X + xs(__ldg(a.pos_g + (n >> 1)), row));
  return p[n & 1];
}
SWE_DEV double &gslot(const LCtx &c, int p, int h, int row) {
  return reinterpret_cast<double *>(c.X + xs(p, row))[h];
}

SWE_DEV void lane_load_grid(const FftArgs &a, const LCtx &c, const double *src, int f) {
  for (int h = 0; h < 2; ++h) {
    const int j = (h && !c.eq) ? c.js : c.jn;
    for (int s = 0; s < c.nsl; ++s) {
      const double *g = src + ((size_t)(c.b0 + s) * a.J + j) * a.I;
      for (int n = c.tid; n < a.I; n += c.nthr) gval(a, c, n, lrow(c, f, h, s)) = __ldg(g + n);
    }
  }
}

SWE_DEV void lane_store_grid(const FftArgs &a, const LCtx &c, double *dst, int f, double scale) {
  for (int h = 0; h < 2 - c.eq; ++h) {
    const int j = h ? c.js : c.jn;
    for (int s = 0; s < c.nsl; ++s) {
      double *g = dst + ((size_t)(c.b0 + s) * a.J + j) * a.I;
      for (int n = c.tid; n < a.I; n += c.nthr) g[n] = gval(a, c, n, lrow(c, f, h, s)) * scale;
    }
  }
}

// fm[k] (k = 0..M) of rows (f, h, s): fm = (Ge + w^{-k} Go) / I, see fft.cu;
// F+ = scale (fm_N + fm_S), F- = scale (fm_N - fm_S)  ->  a.out[f] [m][2][Jp][ld]
// (z1, z2) = slots of Z[k], Z[N2-k]; w = conj twh[k]
SWE_DEV double2 row_fm(const LCtx &c, int row, int z1, int z2, double2 w) {
  const double2 zk = c.X[xs(z1, row)];
  const double2 zc = c.X[xs(z2, row)];
  const double2 Sg = make_double2(zk.x + zc.x, zk.y - zc.y);
  const double2 D = make_double2(zk.y + zc.y, -(zk.x - zc.x));
  const double2 t = cm(w, D);
  return make_double2(Sg.x + t.x, Sg.y + t.y);  // 2 * I * fm
}

// fields 0..nf-1 -> a.out[f], scaled by w01 (fields 0, 1) or w23 (2, 3); one flattened loop
SWE_DEV void lane_extract(const FftArgs &a, const LCtx &c, int nf, double w01, double w23) {
  const int M = a.M, S = c.S, N2 = a.N2, per = (M + 1) * S;
  const size_t pm = (size_t)a.Jp * a.ld / 2;  // F+ -> F- offset (double2)
  for (int idx = c.tid; idx < nf * per; idx += c.nthr) {
    const int r = idx / nf, f = idx - r * nf, k = r / S, s = r - k * S;
    if (s >= c.nsl) continue;
    const int z1 = __ldg(a.pos_z + k), z2 = __ldg(a.pos_z + (k == 0 ? 0 : N2 - k));
    double2 w = __ldg(a.twh + k);
    w.y = -w.y;
    const double h = 0.5 * (f < 2 ? w01 : w23);
    double2 *d = reinterpret_cast<double2 *>(a.out[f] + (size_t)c.p * a.ld) + c.b0 +
                 (size_t)k * 2 * pm + s;
    const double2 fn = row_fm(c, lrow(c, f, 0, s), z1, z2, w);
    if (c.eq) {
      const double2 v = make_double2(fn.x * h, fn.y * h);
      d[0] = v;
      d[pm] = v;
    } else {
      const double2 fs = row_fm(c, lrow(c, f, 1, s), z1, z2, w);
      d[0] = make_double2((fn.x + fs.x) * h, (fn.y + fs.y) * h);
      d[pm] = make_double2((fn.x - fs.x) * h, (fn.y - fs.y) * h);
    }
  }
}

}  // namespace

template <int OP>
__global__ void __launch_bounds__(256, 2) fft_lanes_kernel(const __grid_constant__ FftArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LCtx c;
  c.X = reinterpret_cast<double2 *>(smem_raw);
  c.S = fft_lane_slices(OP);
  // consecutive CTAs take consecutive slice groups of one pair: they share the
  // 32-byte sectors of the [m][2][Jp][ld] rows, which then hit in L2
  c.p = blockIdx.y;
  c.jn = c.p;
  c.js = a.J - 1 - c.p;
  c.eq = c.js == c.jn;
  c.b0 = blockIdx.x * c.S;
  c.nsl = min(c.S, a.nslices - c.b0);
  c.tid = threadIdx.x;
  c.nthr = blockDim.x;
  c.warp = threadIdx.x >> 5;
  c.lane = threadIdx.x & 31;
  c.nw = blockDim.x >> 5;
  const int p = c.p, I = a.I, S = c.S;
  const double ia = a.inv_acos[p];

  if constexpr (OP == FOP_SYNTH_GRID || OP == FOP_SYNTH2_GRID) {
    constexpr int NF = OP == FOP_SYNTH_GRID ? 1 : 2;
    lane_load_eo(a, c, NF, -1);
    __syncthreads();
    lane_ifft(a, c);
    const double sc = (OP == FOP_SYNTH2_GRID || a.scale_mode) ? ia : 1.0;
    for (int f = 0; f < NF; ++f) lane_store_grid(a, c, a.gout[f], f, sc);
  } else if constexpr (OP == FOP_ANALYSIS || OP == FOP_VORTDIV) {
    constexpr int NF = OP == FOP_ANALYSIS ? 1 : 2;
    for (int f = 0; f < NF; ++f) lane_load_grid(a, c, a.gin[f], f);
    __syncthreads();
    if constexpr (OP == FOP_VORTDIV) {
      const double cs = a.coslat[p];
      for (int idx = c.tid; idx < a.N2 * LW; idx += c.nthr) {
        c.X[idx].x *= cs;
        c.X[idx].y *= cs;
      }
      __syncthreads();
    }
    lane_fft(a, c);
    const double w = OP == FOP_ANALYSIS ? a.wq[p] * a.inv_I : a.wsin2[p] * a.inv_I * a.inv_a;
    lane_extract(a, c, NF, w, w);
  } else if constexpr (OP == FOP_CORIOLIS) {
    // linear_coriolis (dynamics.py:129-135): f u, f v -> vortdiv_from_uv; f = -f on the south row
    lane_load_eo(a, c, 2, -1);
    __syncthreads();
    lane_ifft(a, c);
    const double cs = a.coslat[p], fc = a.fcor[p];
    for (int idx = c.tid; idx < a.N2 * LW; idx += c.nthr) {
      const int row = (idx & (LW - 1)) ^ (((idx / LW) << 1) & (LW - 1));  // undo xs()
      const double fr = ((row / S) & 1) ? -fc : fc;
      const double2 z = c.X[idx];
      c.X[idx] = make_double2((fr * (z.x * ia)) * cs, (fr * (z.y * ia)) * cs);
    }
    __syncthreads();
    lane_fft(a, c);
    const double w = a.wsin2[p] * a.inv_I * a.inv_a;
    lane_extract(a, c, 2, w, w);
  } else if constexpr (OP == FOP_NONLINEAR) {
    // nonlinear_advection + nonlinear_rest (dynamics.py:142-160)
    // in: 0 u, 1 v, 2 d_lambda Phi, 3 H.Phi, 4 xi, 5 Phi (phi_prime applied here), 6 delta
    lane_load_eo(a, c, 7, 5);
    __syncthreads();
    lane_ifft(a, c);
    const double cs = a.coslat[p];
    // lanes: (slot, hemisphere, x/y) fastest, so a half-warp reads one bank each
    for (int idx = c.tid; idx < I * 2 * S; idx += c.nthr) {
      const int s = idx / (2 * I), r = idx - s * 2 * I;
      const int pp = r >> 2, h = (r >> 1) & 1, hh = r & 1;
      auto R = [&](int f) -> double & { return gslot(c, pp, hh, lrow(c, f, h, s)); };
      const double u = R(0) * ia, v = R(1) * ia, gx = R(2) * ia, gy = R(3) * ia;
      const double xi = R(4), ph = R(5), de = R(6);
      R(0) = -(u * gx + v * gy) - ph * de;   // -(V.grad Phi) - Phi' delta
      R(1) = 0.5 * (u * u + v * v);          // kinetic energy
      R(2) = (xi * u) * cs;                  // (xi u) cos
      R(3) = (xi * v) * cs;                  // (xi v) cos
    }
    __syncthreads();
    lane_fft<8>(a, c);  // only the 4 product fields x 2 hemispheres (rows 0..7, S = 1)
    const double w = a.wq[p] * a.inv_I, wv = a.wsin2[p] * a.inv_I * a.inv_a;
    lane_extract(a, c, 4, w, wv);
  }
}

template <int OP>
static int launch_lanes(const FftArgs &a, int smem, int nthreads, cudaStream_t st) {
  static int attr = 0;
  if (smem > attr) {
    SWE_CUDA(cudaFuncSetAttribute(fft_lanes_kernel<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem));
    attr = smem;
  }
  const int S = fft_lane_slices(OP);
  dim3 grid((a.nslices + S - 1) / S, a.Jh);
  fft_lanes_kernel<OP><<<grid, nthreads, smem, st>>>(a);
  SWE_LAUNCH_CHECK();
  return OK;
}

int fft_lanes_launch(int op, const FftArgs &a, cudaStream_t st) {
  const int smem = a.N2 * LW * (int)sizeof(double2);
  const int nthr = 256;
  switch (op) {
    case FOP_SYNTH_GRID: return launch_lanes<FOP_SYNTH_GRID>(a, smem, nthr, st);
    case FOP_SYNTH2_GRID: return launch_lanes<FOP_SYNTH2_GRID>(a, smem, nthr, st);
    case FOP_ANALYSIS: return launch_lanes<FOP_ANALYSIS>(a, smem, nthr, st);
    case FOP_VORTDIV: return launch_lanes<FOP_VORTDIV>(a, smem, nthr, st);
    case FOP_CORIOLIS: return launch_lanes<FOP_CORIOLIS>(a, smem, nthr, st);
    case FOP_NONLINEAR: return launch_lanes<FOP_NONLINEAR>(a, smem, nthr, st);
  }
  set_error("unknown fft op %d", op);
  return E_SHAPE;
}

bool fft_lanes_ok(const FftArgs &a) {
  for (int s = 0; s < a.nst; ++s)
    if (!fft_small_radix(a.radix[s])) return false;
  return (size_t)a.N2 * LW * sizeof(double2) <= 227 * 1024;
}

}  // namespace swe
