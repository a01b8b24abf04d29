// Longitude FFT stage, "lane = row" variant for small-radix lengths.
//
// One CTA owns one latitude row j and up to 32 transform rows (fields x
// slices).  Shared memory holds X[k][32]: the 32 rows of one frequency/sample
// index form one 512-byte line, so lane r of every warp works on row r and each
// butterfly access is a conflict-free full line; all lanes of a warp execute
// the same butterfly, so twiddles are warp-uniform broadcasts.  Warps split
// the butterflies of a stage.  Same digit-reversed in-place Cooley-Tukey
// (DIT inverse / DIF forward) and the same fused grid products as fft.cu.
#include "fft.cuh"
#include "fft_core.cuh"

namespace swe {

using namespace fftcore;

namespace {

constexpr int LW = 32;  // rows per CTA (lanes)

// MODE 0 DIT, 1 DIF, 2 prime-factor (no twiddles); see fft.cu
template <int R, int MODE>
SWE_DEV void lane_stage(double2 *X, int N2, int Lp, double dir, const double2 *tw, int warp,
                        int nw, int lane) {
  constexpr int H = (R - 1) / 2;
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
  for (int bf = warp; bf < nbf; bf += nw) {
    const int g = bf / Lp, k = bf - g * Lp, base = g * L + k;
    double2 v[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      v[q] = X[(base + q * Lp) * LW + lane];
      if (MODE == 0 && q && k) v[q] = cm(v[q], twd(tw, q * k * tws, dir));
    }
    dft_store<R>(v, dir, cr, sr, X + base * LW + lane, Lp * LW, tw, MODE == 1 ? k * tws : 0);
  }
}

template <int MODE>
SWE_DEV void lane_run_stage(double2 *X, int N2, int Lp, int R, double dir, const double2 *tw,
                            int warp, int nw, int lane) {
  switch (R) {
    case 2: lane_stage<2, MODE>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    case 3: lane_stage<3, MODE>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    case 4: lane_stage<4, MODE>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    case 5: lane_stage<5, MODE>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    case 7: lane_stage<7, MODE>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    case 11: lane_stage<11, MODE>(X, N2, Lp, dir, tw, warp, nw, lane); break;
    default: lane_stage<13, MODE>(X, N2, Lp, dir, tw, warp, nw, lane); break;
  }
}

struct LCtx {
  double2 *X;
  int j, b0, nsl, S, tid, nthr, warp, lane, nw;
};

// inverse transforms of all 32 rows: pos_z order in, pos_g order out
SWE_DEV void lane_ifft(const FftArgs &a, const LCtx &c) {
  int Lp = 1;
  for (int s = 0; s < a.nst; ++s) {
    if (a.pfa) lane_run_stage<2>(c.X, a.N2, Lp, a.radix[s], 1.0, a.tw, c.warp, c.nw, c.lane);
    else lane_run_stage<0>(c.X, a.N2, Lp, a.radix[s], 1.0, a.tw, c.warp, c.nw, c.lane);
    Lp *= a.radix[s];
    __syncthreads();
  }
}

// forward transforms of all 32 rows: pos_g order in, pos_z order out
SWE_DEV void lane_fft(const FftArgs &a, const LCtx &c) {
  if (a.pfa) {
    int Lp = 1;
    for (int s = 0; s < a.nst; ++s) {
      lane_run_stage<2>(c.X, a.N2, Lp, a.radix[s], -1.0, a.tw, c.warp, c.nw, c.lane);
      Lp *= a.radix[s];
      __syncthreads();
    }
    return;
  }
  int L = a.N2;
  for (int s = a.nst - 1; s >= 0; --s) {
    const int R = a.radix[s];
    lane_run_stage<1>(c.X, a.N2, L / R, R, -1.0, a.tw, c.warp, c.nw, c.lane);
    L /= R;
    __syncthreads();
  }
}

// half spectrum of field f (rows f*S + s) -> Z in digit-reversed order (see fft.cu)
SWE_DEV void lane_load_half_z(const FftArgs &a, const LCtx &c, const double *src, int f) {
  const int N2 = a.N2, M = a.M, npair = N2 / 2 + 1, S = c.S;
  const double2 *base = reinterpret_cast<const double2 *>(src + (size_t)c.j * a.ld) + c.b0;
  const size_t mstride = (size_t)a.J * a.ld / 2;
  const int total = npair * S;
  constexpr int U = 4;  // items per thread in flight (8 independent global loads)
  for (int i0 = c.tid; i0 < total; i0 += U * c.nthr) {
    double2 xk[U], xc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = i0 + u * c.nthr;
      const int k = idx / S, s = idx - k * S;
      const bool ok = idx < total && s < c.nsl;
      const int k2 = k == 0 ? N2 : N2 - k;
      xk[u] = (ok && k <= M) ? __ldg(base + (size_t)k * mstride + s) : make_double2(0.0, 0.0);
      xc[u] = (ok && k2 <= M) ? __ldg(base + (size_t)k2 * mstride + s) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = i0 + u * c.nthr;
      const int k = idx / S, s = idx - k * S;
      if (idx >= total || s >= c.nsl) continue;
      const int row = f * S + s;
      const double2 Xk = xk[u], Xc = xc[u];
      if (k == 0) {
        c.X[__ldg(a.pos_z) * LW + row] = make_double2(Xk.x, Xk.x);
        continue;
      }
      const int k2 = N2 - k;
      const double2 A = make_double2(Xk.x + Xc.x, Xk.y - Xc.y);
      const double2 D = make_double2(Xk.x - Xc.x, Xk.y + Xc.y);
      const double2 Bk = cm(D, __ldg(a.twh + k));
      c.X[__ldg(a.pos_z + k) * LW + row] = make_double2(A.x - Bk.y, A.y + Bk.x);
      if (k2 != k) {
        const double2 A2 = make_double2(Xc.x + Xk.x, Xc.y - Xk.y);
        const double2 D2 = make_double2(Xc.x - Xk.x, Xc.y + Xk.y);
        const double2 B2 = cm(D2, __ldg(a.twh + k2));
        c.X[__ldg(a.pos_z + k2) * LW + row] = make_double2(A2.x - B2.y, A2.y + B2.x);
      }
    }
  }
}

// grid sample n of row r lives in X[pos_g[n/2]][r].{x,y}
SWE_DEV double &gval(const FftArgs &a, const LCtx &c, int n, int row) {
  double *p = reinterpret_cast<double *>(c.X + __ldg(a.pos_g + (n >> 1)) * LW + row);
  return p[n & 1];
}
// component h (0/1) of transform slot p of row r (pointwise ops need no map)
SWE_DEV double &gslot(const LCtx &c, int p, int h, int row) {
  return reinterpret_cast<double *>(c.X + p * LW + row)[h];
}

SWE_DEV void lane_load_grid(const FftArgs &a, const LCtx &c, const double *src, int f) {
  for (int s = 0; s < c.nsl; ++s) {
    const double *g = src + ((size_t)(c.b0 + s) * a.J + c.j) * a.I;
    for (int n = c.tid; n < a.I; n += c.nthr) gval(a, c, n, f * c.S + s) = __ldg(g + n);
  }
}

SWE_DEV void lane_store_grid(const FftArgs &a, const LCtx &c, double *dst, int f, double scale) {
  for (int s = 0; s < c.nsl; ++s) {
    double *g = dst + ((size_t)(c.b0 + s) * a.J + c.j) * a.I;
    for (int n = c.tid; n < a.I; n += c.nthr) g[n] = gval(a, c, n, f * c.S + s) * scale;
  }
}

// fm[k] * scale (k = 0..M) of rows orow*S + s -> a.out[o]  (see fft.cu r2c_outputs)
SWE_DEV void lane_extract(const FftArgs &a, const LCtx &c, int orow, int o, double scale) {
  const int N2 = a.N2, M = a.M, S = c.S;
  const double h = 0.5 * scale;
  double2 *dst = reinterpret_cast<double2 *>(a.out[o] + (size_t)c.j * a.ld) + c.b0;
  const size_t mstride = (size_t)a.J * a.ld / 2;
  for (int idx = c.tid; idx < (M + 1) * S; idx += c.nthr) {
    const int k = idx / S, s = idx - k * S;
    if (s >= c.nsl) continue;
    const int row = orow * S + s;
    const double2 zk = c.X[__ldg(a.pos_z + k) * LW + row];
    const double2 z2 = c.X[__ldg(a.pos_z + (k == 0 ? 0 : N2 - k)) * LW + row];
    const double2 zc = make_double2(z2.x, -z2.y);
    const double2 Sg = make_double2(zk.x + zc.x, zk.y + zc.y);
    const double2 D = make_double2(zk.y - zc.y, -(zk.x - zc.x));
    double2 w = __ldg(a.twh + k);
    w.y = -w.y;
    const double2 t = cm(w, D);
    dst[(size_t)k * mstride + s] = make_double2((Sg.x + t.x) * h, (Sg.y + t.y) * h);
  }
}

}  // namespace

template <int OP>
__global__ void __launch_bounds__(256) fft_lanes_kernel(const __grid_constant__ FftArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LCtx c;
  c.X = reinterpret_cast<double2 *>(smem_raw);
  c.S = fft_lane_slices(OP);
  c.j = blockIdx.x;
  c.b0 = blockIdx.y * c.S;
  c.nsl = min(c.S, a.nslices - c.b0);
  c.tid = threadIdx.x;
  c.nthr = blockDim.x;
  c.warp = threadIdx.x >> 5;
  c.lane = threadIdx.x & 31;
  c.nw = blockDim.x >> 5;
  const int j = c.j, I = a.I, S = c.S;
  const double ia = a.inv_acos[j];

  if constexpr (OP == FOP_SYNTH_GRID || OP == FOP_SYNTH2_GRID) {
    constexpr int NF = OP == FOP_SYNTH_GRID ? 1 : 2;
    for (int f = 0; f < NF; ++f) lane_load_half_z(a, c, a.in[f], f);
    __syncthreads();
    lane_ifft(a, c);
    const double sc = (OP == FOP_SYNTH2_GRID || a.scale_mode) ? ia : 1.0;
    for (int f = 0; f < NF; ++f) lane_store_grid(a, c, a.gout[f], f, sc);
  } else if constexpr (OP == FOP_ANALYSIS || OP == FOP_VORTDIV) {
    constexpr int NF = OP == FOP_ANALYSIS ? 1 : 2;
    for (int f = 0; f < NF; ++f) lane_load_grid(a, c, a.gin[f], f);
    __syncthreads();
    if constexpr (OP == FOP_VORTDIV) {
      const double cs = a.coslat[j];
      for (int idx = c.tid; idx < a.N2 * LW; idx += c.nthr) {
        c.X[idx].x *= cs;
        c.X[idx].y *= cs;
      }
      __syncthreads();
    }
    lane_fft(a, c);
    const double w = OP == FOP_ANALYSIS ? a.wq[j] * a.inv_I : a.wsin2[j] * a.inv_I * a.inv_a;
    for (int f = 0; f < NF; ++f) lane_extract(a, c, f, f, w);
  } else if constexpr (OP == FOP_CORIOLIS) {
    // linear_coriolis (dynamics.py:129-135): f u, f v -> vortdiv_from_uv
    lane_load_half_z(a, c, a.in[0], 0);
    lane_load_half_z(a, c, a.in[1], 1);
    __syncthreads();
    lane_ifft(a, c);
    const double cs = a.coslat[j], fc = a.fcor[j];
    for (int idx = c.tid; idx < a.N2 * LW; idx += c.nthr) {
      const double2 z = c.X[idx];
      c.X[idx] = make_double2((fc * (z.x * ia)) * cs, (fc * (z.y * ia)) * cs);
    }
    __syncthreads();
    lane_fft(a, c);
    const double w = a.wsin2[j] * a.inv_I * a.inv_a;
    lane_extract(a, c, 0, 0, w);
    lane_extract(a, c, 1, 1, w);
  } else if constexpr (OP == FOP_NONLINEAR) {
    // nonlinear_advection + nonlinear_rest (dynamics.py:142-160); rows f*S + s,
    // in: 0 u, 1 v, 2 d_lambda Phi, 3 H.Phi, 4 xi, 5 Phi', 6 delta
    for (int f = 0; f < 7; ++f) lane_load_half_z(a, c, a.in[f], f);
    __syncthreads();
    lane_ifft(a, c);
    const double cs = a.coslat[j];
    for (int idx = c.tid; idx < I * S; idx += c.nthr) {
      const int n = idx / S, s = idx - n * S, p = n >> 1, h = n & 1;
      const double u = gslot(c, p, h, s) * ia, v = gslot(c, p, h, S + s) * ia;
      const double gx = gslot(c, p, h, 2 * S + s) * ia, gy = gslot(c, p, h, 3 * S + s) * ia;
      const double xi = gslot(c, p, h, 4 * S + s), ph = gslot(c, p, h, 5 * S + s);
      const double de = gslot(c, p, h, 6 * S + s);
      gslot(c, p, h, s) = -(u * gx + v * gy) - ph * de;   // -(V.grad Phi) - Phi' delta
      gslot(c, p, h, S + s) = 0.5 * (u * u + v * v);     // kinetic energy
      gslot(c, p, h, 2 * S + s) = (xi * u) * cs;          // (xi u) cos
      gslot(c, p, h, 3 * S + s) = (xi * v) * cs;          // (xi v) cos
    }
    __syncthreads();
    lane_fft(a, c);
    const double w = a.wq[j] * a.inv_I, wv = a.wsin2[j] * a.inv_I * a.inv_a;
    lane_extract(a, c, 0, 0, w);
    lane_extract(a, c, 1, 1, w);
    lane_extract(a, c, 2, 2, wv);
    lane_extract(a, c, 3, 3, wv);
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
  dim3 grid(a.J, (a.nslices + S - 1) / S);
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
