// Longitude FFT stage with fused grid products (see fft.cuh).
//
// Complex transforms of length N2 = I/2 run in place in shared memory, one
// warp per row, as mixed-radix Cooley-Tukey:
//   inverse (c2r): decimation in time; the input Z is written directly in
//                  digit-reversed order by the spectral loader, output natural;
//   forward (r2c): decimation in frequency; natural input, digit-reversed
//                  output read back through the same permutation.
// Every butterfly reads and writes the same R slots, so a lane needs only R
// complex registers.  Radices 2,3,4,5,7,11,13 are unrolled (odd R uses the
// conjugate-pair symmetric form); other primes run warp-cooperatively.
#include "fft.cuh"
#include "fft_core.cuh"

namespace swe {

namespace {

using namespace fftcore;

// in-place stage of radix R over blocks of span L = Lp*R.
// MODE 0 (DIT): inputs twiddled by W_L^{qk}; 1 (DIF): outputs twiddled by W_L^{tk};
// 2 (prime-factor / Good-Thomas): no twiddles.
template <int R, int MODE>
SWE_DEV void stage_small(double2 *x, int N2, int Lp, double dir, const double2 *tw, int lane) {
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
  for (int bf = lane; bf < nbf; bf += 32) {
    const int g = bf / Lp, k = bf - g * Lp, base = g * L + k;
    double2 v[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      v[q] = x[base + q * Lp];
      if (MODE == 0 && q && k) v[q] = cm(v[q], twd(tw, q * k * tws, dir));
    }
    dft_store<R>(v, dir, cr, sr, x + base, Lp, tw, MODE == 1 ? k * tws : 0);
  }
  __syncwarp();
}

// any radix: one butterfly at a time, lanes split the R outputs (scr holds R inputs)
template <int MODE>
SWE_DEV void stage_generic(double2 *x, double2 *scr, int N2, int Lp, int R, double dir,
                           const double2 *tw, int lane) {
  const int L = Lp * R, nbf = N2 / R, tws = N2 / L, rstep = N2 / R;
  for (int bf = 0; bf < nbf; ++bf) {
    const int g = bf / Lp, k = bf - g * Lp, base = g * L + k;
    for (int q = lane; q < R; q += 32) {
      double2 v = x[base + q * Lp];
      if (MODE == 0 && q && k) v = cm(v, twd(tw, q * k * tws, dir));
      scr[q] = v;
    }
    __syncwarp();
    for (int t = lane; t < R; t += 32) {
      double2 acc = make_double2(0.0, 0.0);
      int e = 0;
      for (int q = 0; q < R; ++q) {
        const double2 z = cm(scr[q], twd(tw, e * rstep, dir));
        acc.x += z.x;
        acc.y += z.y;
        e += t;
        if (e >= R) e -= R;
      }
      if (MODE == 1 && t && k) acc = cm(acc, twd(tw, t * k * tws, dir));
      x[base + t * Lp] = acc;
    }
    __syncwarp();
  }
}

template <int MODE>
SWE_DEV void run_stage(double2 *x, double2 *scr, int N2, int Lp, int R, double dir,
                       const double2 *tw, int lane) {
  switch (R) {
    case 2: stage_small<2, MODE>(x, N2, Lp, dir, tw, lane); break;
    case 3: stage_small<3, MODE>(x, N2, Lp, dir, tw, lane); break;
    case 4: stage_small<4, MODE>(x, N2, Lp, dir, tw, lane); break;
    case 5: stage_small<5, MODE>(x, N2, Lp, dir, tw, lane); break;
    case 7: stage_small<7, MODE>(x, N2, Lp, dir, tw, lane); break;
    case 11: stage_small<11, MODE>(x, N2, Lp, dir, tw, lane); break;
    case 13: stage_small<13, MODE>(x, N2, Lp, dir, tw, lane); break;
    default: stage_generic<MODE>(x, scr, N2, Lp, R, dir, tw, lane); break;
  }
}

// inverse: spectral order pos_z in -> grid order pos_g out.  Cooley-Tukey:
// digit-reversed -> natural (DIT, stages r_0 .. r_{S-1}); prime-factor:
// Ruritanian -> CRT (twiddle-free stages along each axis).
SWE_DEV void warp_ifft(double2 *x, double2 *scr, const FftArgs &a, int lane) {
  int Lp = 1;
  for (int s = 0; s < a.nst; ++s) {
    if (a.pfa) run_stage<2>(x, scr, a.N2, Lp, a.radix[s], 1.0, a.tw, lane);
    else run_stage<0>(x, scr, a.N2, Lp, a.radix[s], 1.0, a.tw, lane);
    Lp *= a.radix[s];
  }
}

// forward: grid order pos_g in -> spectral order pos_z out (DIF r_{S-1} .. r_0, or PFA)
SWE_DEV void warp_fft(double2 *x, double2 *scr, const FftArgs &a, int lane) {
  if (a.pfa) {
    int Lp = 1;
    for (int s = 0; s < a.nst; ++s) {
      run_stage<2>(x, scr, a.N2, Lp, a.radix[s], -1.0, a.tw, lane);
      Lp *= a.radix[s];
    }
    return;
  }
  int L = a.N2;
  for (int s = a.nst - 1; s >= 0; --s) {
    const int R = a.radix[s];
    run_stage<1>(x, scr, a.N2, L / R, R, -1.0, a.tw, lane);
    L /= R;
  }
}

struct Ctx {
  double2 *rows, *scr;
  int p, jn, js, eq, b0, nsl, tid, nthr, warp, lane, nw;
};

SWE_DEV double2 *row_of(const FftArgs &a, const Ctx &c, int f, int s) {
  return c.rows + (size_t)(f * a.spb + s) * a.N2;
}

// One hemisphere row h of field f for pair p: half spectrum X = E + O (north) or
// E - O (south) from the parity-split Legendre output [m][2][Jp][ld], written as
// Z in spectral slot order:  Z[k] = (X[k] + conj X[N2-k]) + i w^k (X[k] - conj X[N2-k])
// with w = e^{2 pi i / I}, so IDFT_N2(Z)[r] = g[2r] + i g[2r+1],
// g = irfft(X * I, n = I) (numpy drops Im X[0]).  sub (nullable) is
// subtracted from E at m = 0 (phi_prime, dynamics.py:52-56); imk: X -> i m X
// (longitude derivative of the synthesised field).
SWE_DEV void load_eo(const FftArgs &a, const Ctx &c, const double *src, int f, int h,
                     const double *sub, bool imk = false) {
  const int N2 = a.N2, M = a.M, npair = N2 / 2 + 1;
  const size_t eo = (size_t)a.Jp * a.ld / 2;
  const double2 *base = reinterpret_cast<const double2 *>(src + (size_t)c.p * a.ld) + c.b0;
  const size_t mstride = 2 * eo;
  const double sg = h ? -1.0 : 1.0;
  for (int idx = c.tid; idx < npair * c.nsl; idx += c.nthr) {
    const int k = idx / c.nsl, s = idx - k * c.nsl;
    double2 *x = row_of(a, c, f, s);
    const int k2 = k == 0 ? N2 : N2 - k;
    const double2 z = make_double2(0.0, 0.0);
    double2 e = k <= M ? __ldg(base + (size_t)k * mstride + s) : z;
    const double2 o = k <= M ? __ldg(base + (size_t)k * mstride + eo + s) : z;
    const double2 e2 = k2 <= M ? __ldg(base + (size_t)k2 * mstride + s) : z;
    const double2 o2 = k2 <= M ? __ldg(base + (size_t)k2 * mstride + eo + s) : z;
    if (sub != nullptr && k == 0) e.x -= sub[c.b0 + s];
    double2 Xk = make_double2(e.x + sg * o.x, e.y + sg * o.y);
    double2 Xc = make_double2(e2.x + sg * o2.x, e2.y + sg * o2.y);
    if (imk) {
      Xk = make_double2(-(double)k * Xk.y, (double)k * Xk.x);
      Xc = make_double2(-(double)k2 * Xc.y, (double)k2 * Xc.x);
    }
    if (k == 0) {
      x[__ldg(a.pos_z)] = make_double2(Xk.x, Xk.x);
      continue;
    }
    const double2 A = make_double2(Xk.x + Xc.x, Xk.y - Xc.y);
    const double2 D = make_double2(Xk.x - Xc.x, Xk.y + Xc.y);
    const double2 Bk = cm(D, __ldg(a.twh + k));
    x[__ldg(a.pos_z + k)] = make_double2(A.x - Bk.y, A.y + Bk.x);
    if (k2 != k) {
      const double2 A2 = make_double2(Xc.x + Xk.x, Xc.y - Xk.y);
      const double2 D2 = make_double2(Xc.x - Xk.x, Xc.y + Xk.y);
      const double2 B2 = cm(D2, __ldg(a.twh + k2));
      x[__ldg(a.pos_z + k2)] = make_double2(A2.x - B2.y, A2.y + B2.x);
    }
  }
}

SWE_DEV int row_j(const Ctx &c, int h) { return h ? c.js : c.jn; }

SWE_DEV void load_grid(const FftArgs &a, const Ctx &c, const double *src, int f, int h) {
  for (int s = 0; s < c.nsl; ++s) {
    const double *g = src + ((size_t)(c.b0 + s) * a.J + row_j(c, h)) * a.I;
    double *r = reinterpret_cast<double *>(row_of(a, c, f, s));
    // grid sample n is component n&1 of transform slot pos_g[n/2]
    for (int n = c.tid; n < a.I; n += c.nthr) r[2 * __ldg(a.pos_g + (n >> 1)) + (n & 1)] = __ldg(g + n);
  }
}

SWE_DEV void store_grid(const FftArgs &a, const Ctx &c, double *dst, int f, int h, double scale) {
  for (int s = 0; s < c.nsl; ++s) {
    double *g = dst + ((size_t)(c.b0 + s) * a.J + row_j(c, h)) * a.I;
    const double *r = reinterpret_cast<const double *>(row_of(a, c, f, s));
    for (int n = c.tid; n < a.I; n += c.nthr) g[n] = r[2 * __ldg(a.pos_g + (n >> 1)) + (n & 1)] * scale;
  }
}

SWE_DEV double2 *warp_scr(const FftArgs &a, const Ctx &c) { return c.scr + (size_t)c.warp * a.rgen; }

SWE_DEV void c2r_fields(const FftArgs &a, const Ctx &c, int f0, int nf) {
  for (int task = c.warp; task < nf * c.nsl; task += c.nw) {
    const int f = f0 + task / c.nsl, s = task % c.nsl;
    warp_ifft(row_of(a, c, f, s), warp_scr(a, c), a, c.lane);
  }
}

// forward transforms of fields fld[o] of hemisphere h; fm[k] = (Ge + w^{-k} Go)/I.
// h = 0: stash scale*fm_N in the F+ slot (and F- on the equator);
// h = 1: F+ = stash + scale*fm_S, F- = stash - scale*fm_S.
template <int NOUT>
SWE_DEV void r2c_outputs(const FftArgs &a, const Ctx &c, const int (&fld)[NOUT],
                         const double (&scale)[NOUT], int h) {
  const int N2 = a.N2, M = a.M;
  const size_t pm = (size_t)a.Jp * a.ld / 2;
  for (int task = c.warp; task < NOUT * c.nsl; task += c.nw) {
    const int o = task / c.nsl, s = task % c.nsl;
    double2 *x = row_of(a, c, fld[o], s);
    warp_fft(x, warp_scr(a, c), a, c.lane);
    const double hs = 0.5 * scale[o];
    double2 *dst = reinterpret_cast<double2 *>(a.out[o] + (size_t)c.p * a.ld) + c.b0 + s;
    for (int k = c.lane; k <= M; k += 32) {
      const double2 zk = x[__ldg(a.pos_z + k)];
      const double2 z2 = x[__ldg(a.pos_z + (k == 0 ? 0 : N2 - k))];
      const double2 Sg = make_double2(zk.x + z2.x, zk.y - z2.y);     // 2 Ge
      const double2 D = make_double2(zk.y + z2.y, -(zk.x - z2.x));   // 2 Go
      double2 w = __ldg(a.twh + k);
      w.y = -w.y;
      const double2 t = cm(w, D);
      const double2 v = make_double2((Sg.x + t.x) * hs, (Sg.y + t.y) * hs);
      double2 *d = dst + (size_t)k * 2 * pm;
      if (h == 0) {
        d[0] = v;
        if (c.eq) d[pm] = v;
      } else {
        const double2 n = d[0];
        d[0] = make_double2(n.x + v.x, n.y + v.y);
        d[pm] = make_double2(n.x - v.x, n.y - v.y);
      }
    }
  }
}

}  // namespace

template <int OP>
__global__ void __launch_bounds__(256) fft_kernel(const __grid_constant__ FftArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Ctx c;
  c.p = blockIdx.x;
  c.jn = c.p;
  c.js = a.J - 1 - c.p;
  c.eq = c.js == c.jn;
  c.b0 = blockIdx.y * a.spb;
  c.nsl = min(a.spb, a.nslices - c.b0);
  c.tid = threadIdx.x;
  c.nthr = blockDim.x;
  c.warp = threadIdx.x >> 5;
  c.lane = threadIdx.x & 31;
  c.nw = blockDim.x >> 5;
  c.rows = reinterpret_cast<double2 *>(smem_raw);
  c.scr = c.rows + (size_t)fft_rows_per_slice(OP) * a.spb * a.N2;
  const int p = c.p;
  const double ia = a.inv_acos[p];
  const int I = a.I;

  auto pointwise = [&](auto fn) {
    for (int idx = c.tid; idx < c.nsl * I; idx += c.nthr) {
      const int s = idx / I, n = idx - s * I;
      fn(s, n);
    }
  };
  auto rd = [&](int f, int s) { return reinterpret_cast<double *>(row_of(a, c, f, s)); };

  // north row, then south row (skipped on the equator); spectra of the north
  // pass are stashed in the output's F+ slot and folded by the south pass
  for (int h = 0; h < 2 - c.eq; ++h) {
    if constexpr (OP == FOP_SYNTH_GRID) {
      load_eo(a, c, a.in[0], 0, h, nullptr);
      __syncthreads();
      c2r_fields(a, c, 0, 1);
      __syncthreads();
      store_grid(a, c, a.gout[0], 0, h, a.scale_mode ? ia : 1.0);
    } else if constexpr (OP == FOP_SYNTH2_GRID) {
      load_eo(a, c, a.in[0], 0, h, nullptr);
      load_eo(a, c, a.in[1], 1, h, nullptr);
      __syncthreads();
      c2r_fields(a, c, 0, 2);
      __syncthreads();
      store_grid(a, c, a.gout[0], 0, h, ia);
      store_grid(a, c, a.gout[1], 1, h, ia);
    } else if constexpr (OP == FOP_ANALYSIS) {
      load_grid(a, c, a.gin[0], 0, h);
      __syncthreads();
      const int f[1] = {0};
      const double sc[1] = {a.wq[p] * a.inv_I};
      r2c_outputs<1>(a, c, f, sc, h);
    } else if constexpr (OP == FOP_VORTDIV) {
      load_grid(a, c, a.gin[0], 0, h);
      load_grid(a, c, a.gin[1], 1, h);
      __syncthreads();
      const double cs = a.coslat[p];
      pointwise([&](int s, int n) {
        rd(0, s)[n] *= cs;
        rd(1, s)[n] *= cs;
      });
      __syncthreads();
      const int f[2] = {0, 1};
      const double w = a.wsin2[p] * a.inv_I * a.inv_a;
      const double sc[2] = {w, w};
      r2c_outputs<2>(a, c, f, sc, h);
    } else if constexpr (OP == FOP_CORIOLIS) {
      // linear_coriolis (dynamics.py:129-135); f = 2 Omega mu flips sign in the south
      load_eo(a, c, a.in[0], 0, h, nullptr);
      load_eo(a, c, a.in[1], 1, h, nullptr);
      __syncthreads();
      c2r_fields(a, c, 0, 2);
      __syncthreads();
      const double cs = a.coslat[p], fc = h ? -a.fcor[p] : a.fcor[p];
      pointwise([&](int s, int n) {
        double *u = rd(0, s), *v = rd(1, s);
        u[n] = (fc * (u[n] * ia)) * cs;
        v[n] = (fc * (v[n] * ia)) * cs;
      });
      __syncthreads();
      const int f[2] = {0, 1};
      const double w = a.wsin2[p] * a.inv_I * a.inv_a;
      const double sc[2] = {w, w};
      r2c_outputs<2>(a, c, f, sc, h);
    } else if constexpr (OP == FOP_NONLINEAR) {
      // nonlinear_advection + nonlinear_rest (dynamics.py:142-160)
      // in: 0 u, 1 v, 2 d_lambda Phi, 3 H.Phi, 4 xi, 5 Phi (phi_prime applied here), 6 delta
      for (int f = 0; f < 4; ++f)
        load_eo(a, c, (f == 2 && a.dlam) ? a.in[5] : a.in[f], f, h, nullptr, f == 2 && a.dlam);
      __syncthreads();
      c2r_fields(a, c, 0, 4);
      __syncthreads();
      pointwise([&](int s, int n) {
        double *r0 = rd(0, s), *r1 = rd(1, s), *r2 = rd(2, s), *r3 = rd(3, s);
        const double u = r0[n] * ia, v = r1[n] * ia, gx = r2[n] * ia, gy = r3[n] * ia;
        r0[n] = u;
        r1[n] = v;
        r2[n] = -(u * gx + v * gy);
        r3[n] = 0.5 * (u * u + v * v);
      });
      load_eo(a, c, a.in[4], 4, h, nullptr);
      __syncthreads();
      c2r_fields(a, c, 4, 1);
      __syncthreads();
      const double cs = a.coslat[p];
      pointwise([&](int s, int n) {
        double *r0 = rd(0, s), *r1 = rd(1, s);
        const double xi = rd(4, s)[n];
        r0[n] = (xi * r0[n]) * cs;
        r1[n] = (xi * r1[n]) * cs;
      });
      __syncthreads();
      load_eo(a, c, a.in[5], 4, h, a.phisub);
      load_eo(a, c, a.in[6], 5, h, nullptr);
      __syncthreads();
      c2r_fields(a, c, 4, 2);
      __syncthreads();
      if (!a.no_rest) pointwise([&](int s, int n) { rd(2, s)[n] -= rd(4, s)[n] * rd(5, s)[n]; });
      __syncthreads();
      const int f[4] = {2, 3, 0, 1};
      const double w = a.wq[p] * a.inv_I, wv = a.wsin2[p] * a.inv_I * a.inv_a;
      const double sc[4] = {w, w, wv, wv};
      r2c_outputs<4>(a, c, f, sc, h);
    }
    __syncthreads();
  }
}

bool fft_small_radix(int R) {
  return R == 2 || R == 3 || R == 4 || R == 5 || R == 7 || R == 11 || R == 13;
}

template <int OP>
static int launch_op(const FftArgs &a, int smem, cudaStream_t st) {
  static int attr = 0;
  if (smem > attr) {
    SWE_CUDA(cudaFuncSetAttribute(fft_kernel<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = smem;
  }
  dim3 grid(a.Jh, (a.nslices + a.spb - 1) / a.spb);
  fft_kernel<OP><<<grid, a.nwarps * 32, smem, st>>>(a);
  SWE_LAUNCH_CHECK();
  return OK;
}

int fft_launch(int op, const FftArgs &a, int smem, cudaStream_t st) {
  switch (op) {
    case FOP_SYNTH_GRID: return launch_op<FOP_SYNTH_GRID>(a, smem, st);
    case FOP_SYNTH2_GRID: return launch_op<FOP_SYNTH2_GRID>(a, smem, st);
    case FOP_ANALYSIS: return launch_op<FOP_ANALYSIS>(a, smem, st);
    case FOP_VORTDIV: return launch_op<FOP_VORTDIV>(a, smem, st);
    case FOP_CORIOLIS: return launch_op<FOP_CORIOLIS>(a, smem, st);
    case FOP_NONLINEAR: return launch_op<FOP_NONLINEAR>(a, smem, st);
  }
  set_error("unknown fft op %d", op);
  return E_SHAPE;
}

}  // namespace swe
