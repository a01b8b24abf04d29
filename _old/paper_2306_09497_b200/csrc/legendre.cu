// Grouped, parity-folded FP64 DMMA Legendre GEMMs (see legendre.cuh).
#include "legendre.cuh"
#include "legendre_gemv.cuh"

#include <algorithm>

namespace swe {

// ---------------------------------------------------------------------------
// Synthesis: for one order m, latitude-pair tile [p0, p0+64) and column tile
// [c0, c0+64):   E[p][c] = sum_{n-m even} T(p,n) f(src[n][c]),
//                O[p][c] = sum_{n-m odd}  T(p,n) f(src[n][c])     (P-like term)
// north row p = E + O, south row J-1-p = E - O.  H-like terms swap E/O.
// 4 warps (2x2), warp tile 32 pairs x 32 columns, E and O accumulators.
// ---------------------------------------------------------------------------
namespace {
constexpr int SY_KT = 8;      // modes per parity per k-chunk
constexpr int SY_STAGES = 3;  // cp.async pipeline depth
constexpr int SY_LDA = SY_BM + 4;
constexpr int SY_LDB = SY_BN + 4;

struct SynthSmem {
  double A[SY_STAGES][2 * SY_KT][SY_LDA];
  double B[SY_STAGES][2 * SY_KT][SY_LDB];
  double S[SY_STAGES][2 * SY_KT];
};
}  // namespace

__global__ void __launch_bounds__(128) leg_synth_kernel(const __grid_constant__ LegArgs args) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SynthSmem &sm = *reinterpret_cast<SynthSmem *>(smem_raw);
  const LegOut &o = args.out[blockIdx.z];
  const int2 item = args.items[blockIdx.x];
  const int m = item.x, p0 = item.y * SY_BM, c0 = blockIdx.y * SY_BN;
  const int M = args.M, Jp = args.Jp, ld = args.ld;
  const int km = M + 1 - m, ne = (km + 1) >> 1, no = km >> 1;
  const int off = args.offsets[m];
  const int nch_t = (ne + SY_KT - 1) / SY_KT;
  const int nch = nch_t * o.nterms;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3, wr = warp >> 1, wc = warp & 1;

  auto load_chunk = [&](int c, int stage) {
    const int term = c / nch_t, t0 = (c - term * nch_t) * SY_KT;
    const LegTerm &T = o.t[term];
    for (int i = tid; i < 2 * SY_KT * (SY_BM / 2); i += 128) {
      const int r = i / (SY_BM / 2), cc = (i - r * (SY_BM / 2)) * 2;
      const int par = r / SY_KT, tt = t0 + (r - par * SY_KT);
      const bool v = (tt < (par ? no : ne)) && (p0 + cc < Jp);
      const size_t row = (size_t)off + (par ? ne : 0) + tt;
      cp_async16(&sm.A[stage][r][cc], T.tab + (v ? row * Jp + p0 + cc : 0), v);
    }
    for (int i = tid; i < 2 * SY_KT * (SY_BN / 2); i += 128) {
      const int r = i / (SY_BN / 2), cc = (i - r * (SY_BN / 2)) * 2;
      const int par = r / SY_KT, tt = t0 + (r - par * SY_KT);
      const bool v = (tt < (par ? no : ne)) && (c0 + cc < ld);
      const size_t k = (size_t)off + (par ? ne : 0) + tt;  // parity-split row
      const double *src = T.src + (v ? k * ld + c0 + cc : 0);
      if (T.phi0 != nullptr && v && k == 0) {
        // phi_prime: subtract phibar*sqrt(2) from Re of mode (0,0) (dynamics.py:52-56)
        sm.B[stage][r][cc] = src[0] - T.phi0[(c0 + cc) >> 1];
        sm.B[stage][r][cc + 1] = src[1];
      } else {
        cp_async16(&sm.B[stage][r][cc], src, v);
      }
    }
    if (tid < 2 * SY_KT) {
      const int par = tid / SY_KT, tt = t0 + (tid - par * SY_KT);
      double s = 0.0;
      if (tt < (par ? no : ne)) {
        const int k = off + (par ? ne : 0) + tt;
        s = T.sign * (T.scale ? T.scale[k] : 1.0) * (T.times_im ? (double)m : 1.0);
      }
      sm.S[stage][tid] = s;
    }
  };

  double accE[4][4][2], accO[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) accE[i][j][0] = accE[i][j][1] = accO[i][j][0] = accO[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < SY_STAGES - 1; ++s) {
    if (s < nch) load_chunk(s, s);
    cp_async_commit();
  }
  for (int c = 0; c < nch; ++c) {
    cp_async_wait<SY_STAGES - 2>();
    __syncthreads();
    {
      const int cn = c + SY_STAGES - 1;
      if (cn < nch) load_chunk(cn, cn % SY_STAGES);
      cp_async_commit();
    }
    const int st = c % SY_STAGES;
    const LegTerm &T = o.t[c / nch_t];
    const int flip = T.flip, tim = T.times_im;
    // lane's column within its 8-wide fragment; i*m swaps re/im with a sign
    const int bsel = g ^ tim;
    const double bsgn = tim ? ((g & 1) ? 1.0 : -1.0) : 1.0;
#pragma unroll
    for (int kk = 0; kk < SY_KT / 4; ++kk) {
#pragma unroll
      for (int par = 0; par < 2; ++par) {
        const int r = par * SY_KT + kk * 4 + t;
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = sm.A[st][r][wr * 32 + i * 8 + g];
        const double sc = sm.S[st][r] * bsgn;
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = sm.B[st][r][wc * 32 + j * 8 + bsel] * sc;
        if ((par ^ flip) == 0) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma(accE[i][j][0], accE[i][j][1], a[i], b[j]);
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma(accO[i][j][0], accO[i][j][1], a[i], b[j]);
        }
      }
    }
  }
  cp_async_wait<0>();

  // epilogue: E and O planes of [m][2][Jp][ld] (the FFT stage forms north = E + O,
  // south = E - O)
  const int Jh = args.Jh;
  double *dE = o.dst + (size_t)m * 2 * Jp * ld, *dO = dE + (size_t)Jp * ld;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int p = p0 + wr * 32 + i * 8 + g;
    if (p >= Jh) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = c0 + wc * 32 + j * 8 + 2 * t;
      if (col >= ld) continue;
      // m = 0: irfft ignores Im of the mean bin, so store it as 0 (spharm.py:257)
      const double z = m ? 1.0 : 0.0;
      *reinterpret_cast<double2 *>(dE + (size_t)p * ld + col) = make_double2(accE[i][j][0], z * accE[i][j][1]);
      *reinterpret_cast<double2 *>(dO + (size_t)p * ld + col) = make_double2(accO[i][j][0], z * accO[i][j][1]);
    }
  }
}

// ---------------------------------------------------------------------------
// Analysis: for one order m, a tile of 16 even + 16 odd modes and column tile
// [c0, c0+64):  out[n][c] = sum_p T(p,n) F±[p][c],  F± = f_north ± f_south
// (rows already weighted by the FFT stage).  Even n-m of a P-like term reads
// F+, odd reads F-; H-like terms swap.  4 warps = (parity, column half),
// warp tile 16 modes x 32 columns.
// ---------------------------------------------------------------------------
namespace {
constexpr int AN_STAGES = 3;
constexpr int AN_LDA = AN_KP + 4;
constexpr int AN_LDB = AN_BN + 4;

struct AnalSmem {
  double A[AN_STAGES][2 * AN_BR][AN_LDA];
  double F[AN_STAGES][2][AN_KP][AN_LDB];  // F+ / F-
  double Ps[AN_STAGES][AN_KP];            // per-pair scale (LegTerm::pscale)
};
}  // namespace

__global__ void __launch_bounds__(128) leg_anal_kernel(const __grid_constant__ LegArgs args) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  AnalSmem &sm = *reinterpret_cast<AnalSmem *>(smem_raw);
  const LegOut &o = args.out[blockIdx.z];
  const int2 item = args.items[blockIdx.x];
  const int m = item.x, r0 = item.y * AN_BR, c0 = blockIdx.y * AN_BN;
  const int M = args.M, Jh = args.Jh, Jp = args.Jp, ld = args.ld;
  const int km = M + 1 - m, ne = (km + 1) >> 1, no = km >> 1;
  const int off = args.offsets[m];
  const int nch_t = Jp / AN_KP;
  const int nch = nch_t * o.nterms;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3, wpar = warp >> 1, wc = warp & 1;

  auto load_chunk = [&](int c, int stage) {
    const int term = c / nch_t, q0 = (c - term * nch_t) * AN_KP;
    const LegTerm &T = o.t[term];
    // table rows: 16 even + 16 odd modes, columns p in [q0, q0+16)
    for (int i = tid; i < 2 * AN_BR * (AN_KP / 2); i += 128) {
      const int r = i / (AN_KP / 2), cc = (i - r * (AN_KP / 2)) * 2;
      const int par = r / AN_BR, tt = r0 + (r - par * AN_BR);
      const bool v = tt < (par ? no : ne);
      const size_t row = (size_t)off + (par ? ne : 0) + tt;
      cp_async16(&sm.A[stage][r][cc], T.tab + (v ? row * Jp + q0 + cc : 0), v);
    }
    // folded rows F+ (hs 0) and F- (hs 1) of [m][2][Jp][ld], pairs q0..q0+15
    const double *base = T.src + (size_t)m * 2 * Jp * ld;
    for (int i = tid; i < 2 * AN_KP * (AN_BN / 2); i += 128) {
      const int hs = i / (AN_KP * (AN_BN / 2));
      const int rem = i - hs * (AN_KP * (AN_BN / 2));
      const int pr = rem / (AN_BN / 2), cc = (rem - pr * (AN_BN / 2)) * 2;
      const int p = q0 + pr;
      const bool v = (p < Jh) && (c0 + cc < ld);
      cp_async16(&sm.F[stage][hs][pr][cc],
                 base + (v ? ((size_t)(hs ^ T.swap_pm) * Jp + p) * ld + c0 + cc : 0), v);
    }
    if (tid < AN_KP) sm.Ps[stage][tid] = T.pscale ? T.pscale[q0 + tid] : 1.0;
  };

  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < AN_STAGES - 1; ++s) {
    if (s < nch) load_chunk(s, s);
    cp_async_commit();
  }
  for (int c = 0; c < nch; ++c) {
    cp_async_wait<AN_STAGES - 2>();
    __syncthreads();
    const int st = c % AN_STAGES;
    {
      const int cn = c + AN_STAGES - 1;
      if (cn < nch) load_chunk(cn, cn % AN_STAGES);
      cp_async_commit();
    }
    const LegTerm &T = o.t[c / nch_t];
    const int tim = T.times_im;
    const int fsel = wpar ^ T.flip;  // 0: F+, 1: F-
    const int bsel = g ^ tim;
    const double fac = T.sign * (tim ? ((g & 1) ? (double)m : -(double)m) : 1.0);
#pragma unroll
    for (int kk = 0; kk < AN_KP / 4; ++kk) {
      double a[2], b[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) a[i] = sm.A[st][wpar * AN_BR + i * 8 + g][kk * 4 + t];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        b[j] = sm.F[st][fsel][kk * 4 + t][wc * 32 + j * 8 + bsel] * (fac * sm.Ps[st][kk * 4 + t]);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();

  const int nt = wpar ? no : ne;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int tt = r0 + i * 8 + g;
    if (tt >= nt) continue;
    const size_t k = (size_t)off + (wpar ? ne : 0) + tt;  // parity-split row
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = c0 + wc * 32 + j * 8 + 2 * t;
      if (col >= ld) continue;
      *reinterpret_cast<double2 *>(o.dst + k * ld + col) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
  }
}

// ---------------------------------------------------------------------------
// Small batches (a few slices: the serial coarse chain, single-slice fine runs):
// the GEMMs degenerate to matrix x (1..4 complex columns) products, which DMMA
// tiles of 64 columns serve at a few percent utilisation and with long per-CTA
// chunk chains.  These "gemv" kernels give every (output, m, pair | mode, slice)
// dot product an 8-lane group that splits the sum (rows / pairs = lane mod 8),
// keeps a few independent loads in flight per lane and reduces by shuffles.
// Same terms, signs and edge rules as leg_synth_kernel / leg_anal_kernel.
// ---------------------------------------------------------------------------
// one 8-lane group per (output, m, pair): lanes split the mode rows, every table
// element is loaded once and applied to all NS slices (legendre_gemv.cuh).  Whole
// warps iterate (a warp holds 4 groups), so the shuffles always see every lane.
template <int NS>
__global__ void __launch_bounds__(256) leg_synth_gemv(const __grid_constant__ LegArgs args) {
  const long long ng = (long long)args.nout * (args.M + 1) * args.Jh;
  const int gl = threadIdx.x & (GV_L - 1);
  const long long step = (long long)gridDim.x * blockDim.x / GV_L;
  for (long long g0 = (blockIdx.x * (long long)blockDim.x + (threadIdx.x & ~31)) / GV_L; g0 < ng;
       g0 += step) {
    const long long gi = g0 + (threadIdx.x & 31) / GV_L;
    synth_gemv_group<NS, false>(args, gi, gl, gi < ng);
  }
}

// one 8-lane group per (output, mode row): lanes split the latitude pairs
template <int NS>
__global__ void __launch_bounds__(256) leg_anal_gemv(const __grid_constant__ LegArgs args, int K) {
  const long long ng = (long long)args.nout * K;
  const int gl = threadIdx.x & (GV_L - 1);
  const long long step = (long long)gridDim.x * blockDim.x / GV_L;
  for (long long g0 = (blockIdx.x * (long long)blockDim.x + (threadIdx.x & ~31)) / GV_L; g0 < ng;
       g0 += step) {
    const long long gi = g0 + (threadIdx.x & 31) / GV_L;
    anal_gemv_group<NS, false>(args, K, gi, gl, gi < ng);
  }
}

template <int NS>
static int synth_gemv(const LegArgs &a, cudaStream_t st) {
  const long long ng = (long long)a.nout * (a.M + 1) * a.Jh;
  const int nb = (int)std::min<long long>((ng * GV_L + 255) / 256, 148 * 8);
  leg_synth_gemv<NS><<<nb, 256, 0, st>>>(a);
  SWE_LAUNCH_CHECK();
  return OK;
}
template <int NS>
static int anal_gemv(const LegArgs &a, int K, cudaStream_t st) {
  const long long ng = (long long)a.nout * K;
  const int nb = (int)std::min<long long>((ng * GV_L + 255) / 256, 148 * 8);
  leg_anal_gemv<NS><<<nb, 256, 0, st>>>(a, K);
  SWE_LAUNCH_CHECK();
  return OK;
}

int leg_synth_gemv_launch(const LegArgs &a, int nslice, cudaStream_t st) {
  switch (nslice) {
    case 1: return synth_gemv<1>(a, st);
    case 2: return synth_gemv<2>(a, st);
    case 3: return synth_gemv<3>(a, st);
    case 4: return synth_gemv<4>(a, st);
  }
  set_error("internal: dot-product synthesis takes 1..4 slices, got %d", nslice);
  return E_SHAPE;
}

int leg_anal_gemv_launch(const LegArgs &a, int nslice, int K, cudaStream_t st) {
  switch (nslice) {
    case 1: return anal_gemv<1>(a, K, st);
    case 2: return anal_gemv<2>(a, K, st);
    case 3: return anal_gemv<3>(a, K, st);
    case 4: return anal_gemv<4>(a, K, st);
  }
  set_error("internal: dot-product analysis takes 1..4 slices, got %d", nslice);
  return E_SHAPE;
}

int leg_synth_launch(const LegArgs &a, int ncoltiles, cudaStream_t st) {
  static bool attr = false;
  const int smem = (int)sizeof(SynthSmem);
  if (!attr) {
    SWE_CUDA(cudaFuncSetAttribute(leg_synth_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  dim3 grid(a.nitems, ncoltiles, a.nout);
  leg_synth_kernel<<<grid, 128, smem, st>>>(a);
  SWE_LAUNCH_CHECK();
  return OK;
}

int leg_anal_launch(const LegArgs &a, int ncoltiles, cudaStream_t st) {
  static bool attr = false;
  const int smem = (int)sizeof(AnalSmem);
  if (!attr) {
    SWE_CUDA(cudaFuncSetAttribute(leg_anal_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  dim3 grid(a.nitems, ncoltiles, a.nout);
  leg_anal_kernel<<<grid, 128, smem, st>>>(a);
  SWE_LAUNCH_CHECK();
  return OK;
}

}  // namespace swe
