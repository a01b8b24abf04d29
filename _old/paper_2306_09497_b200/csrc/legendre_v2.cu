// Legendre GEMMs, wide-tile variant (templated on the CTA column tile BN).
//
// Same contraction and data layout as legendre.cu, restructured for the DMMA
// issue model of sm_100a (every DMMA.8x8x4 holds its warp for 16 cycles):
//   synthesis: CTA = 64 latitude pairs x BN columns, BN/16 warps; a warp owns
//     one parity class (E or O) x 32 pairs x 64 columns = 4x8 fragments,
//     32 DMMA per 12 fragment loads; 16 modes per parity per cp.async stage.
//   analysis:  CTA = 32 even + 32 odd modes x BN columns; a warp owns one
//     parity x 16 modes x 64 columns; 16 latitude pairs per stage.
// Fragments of k-step kk+1 are loaded/scaled while kk's DMMAs issue.  Per-mode
// scales multiply A fragments; the i*m re/im swap flips signs with an integer
// XOR on B fragments; 8-row latitude fragments past the last pair are skipped.
#include "legendre.cuh"

namespace swe {

namespace {

constexpr int V_BM = 64, V_KT = 16, V_ST = 3;
constexpr int V_LDA = V_BM + 4;

template <int BN>
struct SynthSmemV2 {
  double A[V_ST][2 * V_KT][V_LDA];
  double B[V_ST][2 * V_KT][BN + 4];
  double S[V_ST][2 * V_KT];
};

SWE_DEV double flip_sign(double x, unsigned long long mask) {
  return __longlong_as_double(__double_as_longlong(x) ^ (long long)mask);
}

}  // namespace

template <int BN>
__global__ void __launch_bounds__(BN * 2) leg_synth_v2(const __grid_constant__ LegArgs args) {
  constexpr int NT = BN * 2;  // threads: BN/16 warps
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SynthSmemV2<BN> &sm = *reinterpret_cast<SynthSmemV2<BN> *>(smem_raw);
  const LegOut &o = args.out[blockIdx.z];
  const int2 item = args.items[blockIdx.x];
  const int m = item.x, p0 = item.y * V_BM, c0 = blockIdx.y * BN;
  const int M = args.M, Jp = args.Jp, ld = args.ld, Jh = args.Jh;
  const int km = M + 1 - m, ne = (km + 1) >> 1, no = km >> 1;
  const int off = args.offsets[m];
  const int nch_t = (ne + V_KT - 1) / V_KT;
  const int nch = nch_t * o.nterms;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wpar = warp & 1, wph = (warp >> 1) & 1, wch = warp >> 2;
  const int pw0 = p0 + wph * 32;
  const int nfr = max(0, min(4, (Jh - pw0 + 7) >> 3));  // live 8-pair fragments

  auto load_chunk = [&](int c, int stage) {
    const int term = c / nch_t, t0 = (c - term * nch_t) * V_KT;
    const LegTerm &T = o.t[term];
    // A: 32 mode rows x 64 pairs = 1024 16-byte chunks
#pragma unroll
    for (int i = tid; i < 1024; i += NT) {
      const int r = i >> 5, cc = (i & 31) * 2, par = r >> 4, tt = t0 + (r & 15);
      const bool v = (tt < (par ? no : ne)) && (p0 + cc < Jp);
      const size_t row = (size_t)off + (par ? ne : 0) + tt;
      cp_async16(&sm.A[stage][r][cc], T.tab + (v ? row * Jp + p0 + cc : 0), v);
    }
    // B: 32 mode rows x BN columns
#pragma unroll
    for (int i = tid; i < 16 * BN; i += NT) {
      const int r = i / (BN / 2), cc = (i % (BN / 2)) * 2, par = r >> 4, tt = t0 + (r & 15);
      const bool v = (tt < (par ? no : ne)) && (c0 + cc < ld);
      const size_t k = (size_t)off + (par ? ne : 0) + tt;  // parity-split row
      const double *src = T.src + (v ? k * ld + c0 + cc : 0);
      if (T.phi0 != nullptr && v && k == 0) {
        // phi_prime (dynamics.py:52-56)
        sm.B[stage][r][cc] = src[0] - T.phi0[(c0 + cc) >> 1];
        sm.B[stage][r][cc + 1] = src[1];
      } else {
        cp_async16(&sm.B[stage][r][cc], src, v);
      }
    }
    if (tid < 2 * V_KT) {
      const int par = tid >> 4, tt = t0 + (tid & 15);
      double s = 0.0;
      if (tt < (par ? no : ne)) {
        const int k = off + (par ? ne : 0) + tt;
        s = T.sign * (T.scale ? T.scale[k] : 1.0) * (T.times_im ? (double)m : 1.0);
      }
      sm.S[stage][tid] = s;
    }
  };

  double acc[4][8][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < V_ST - 1; ++s) {
    if (s < nch) load_chunk(s, s);
    cp_async_commit();
  }
  for (int c = 0; c < nch; ++c) {
    cp_async_wait<V_ST - 2>();
    __syncthreads();
    {
      const int cn = c + V_ST - 1;
      if (cn < nch) load_chunk(cn, cn % V_ST);
      cp_async_commit();
    }
    if (nfr == 0) continue;
    const int st = c % V_ST;
    const LegTerm &T = o.t[c / nch_t];
    const int rpar = wpar ^ T.flip;  // mode parity this warp contracts
    const int tim = T.times_im;
    const int bsel = wch * 64 + (g ^ tim);
    const unsigned long long bmask = (tim && !(g & 1)) ? 0x8000000000000000ULL : 0ULL;
    const double *Ab = &sm.A[st][rpar * V_KT + t][wph * 32 + g];
    const double *Bb = &sm.B[st][rpar * V_KT + t][bsel];
    const double *Sb = &sm.S[st][rpar * V_KT + t];
    double a[2][4], b[2][8];
    auto frag = [&](int kk, int q) {
      const double sc = Sb[kk * 4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[q][i] = Ab[kk * 4 * V_LDA + i * 8] * sc;
#pragma unroll
      for (int j = 0; j < 8; ++j) b[q][j] = flip_sign(Bb[kk * 4 * (BN + 4) + j * 8], bmask);
    };
    frag(0, 0);
#pragma unroll
    for (int kk = 0; kk < V_KT / 4; ++kk) {
      const int q = kk & 1;
      if (kk + 1 < V_KT / 4) frag(kk + 1, q ^ 1);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i < nfr) {
#pragma unroll
          for (int j = 0; j < 8; ++j) dmma(acc[i][j][0], acc[i][j][1], a[q][i], b[q][j]);
        }
      }
    }
  }
  cp_async_wait<0>();

  // epilogue: each warp stores its parity plane of [m][2][Jp][ld] (E or O);
  // the FFT stage forms north = E + O, south = E - O
  double *dst = o.dst + ((size_t)m * 2 + wpar) * Jp * ld;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int p = pw0 + i * 8 + g;
    if (p >= Jh) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int col = c0 + wch * 64 + j * 8 + 2 * t;
      if (col >= ld) continue;
      // m = 0: irfft ignores Im of the mean bin, so store it as 0 (spharm.py:257)
      *reinterpret_cast<double2 *>(dst + (size_t)p * ld + col) =
          make_double2(acc[i][j][0], m ? acc[i][j][1] : 0.0);
    }
  }
}

// ---------------------------------------------------------------------------
namespace {
constexpr int VA_BR = V2_ABR, VA_KP = 16, VA_ST = 3;
constexpr int VA_LDA = VA_KP + 4;
template <int BN>
struct AnalSmemV2 {
  double A[VA_ST][2 * VA_BR][VA_LDA];
  double F[VA_ST][2][VA_KP][BN + 4];
  double Ps[VA_ST][VA_KP];  // per-pair scale (LegTerm::pscale)
};
}  // namespace

template <int BN>
__global__ void __launch_bounds__(BN * 2) leg_anal_v2(const __grid_constant__ LegArgs args) {
  constexpr int NT = BN * 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  AnalSmemV2<BN> &sm = *reinterpret_cast<AnalSmemV2<BN> *>(smem_raw);
  const LegOut &o = args.out[blockIdx.z];
  const int2 item = args.items[blockIdx.x];
  const int m = item.x, r0 = item.y * VA_BR, c0 = blockIdx.y * BN;
  const int M = args.M, Jh = args.Jh, Jp = args.Jp, ld = args.ld;
  const int km = M + 1 - m, ne = (km + 1) >> 1, no = km >> 1;
  const int off = args.offsets[m];
  const int nch_t = Jp / VA_KP;
  const int nch = nch_t * o.nterms;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wpar = warp & 1, wrh = (warp >> 1) & 1, wch = warp >> 2;
  const int nrow = (wpar ? no : ne) - (r0 + wrh * 16);
  const int nfr = max(0, min(2, (nrow + 7) >> 3));

  auto load_chunk = [&](int c, int stage) {
    const int term = c / nch_t, q0 = (c - term * nch_t) * VA_KP;
    const LegTerm &T = o.t[term];
    // table: 64 mode rows x 16 pairs = 512 chunks
#pragma unroll
    for (int i = tid; i < 512; i += NT) {
      const int r = i >> 3, cc = (i & 7) * 2, par = r >> 5, tt = r0 + (r & 31);
      const bool v = tt < (par ? no : ne);
      const size_t row = (size_t)off + (par ? ne : 0) + tt;
      cp_async16(&sm.A[stage][r][cc], T.tab + (v ? row * Jp + q0 + cc : 0), v);
    }
    // folded rows F+ (hs 0) and F- (hs 1) of [m][2][Jp][ld]: 2 x 16 x BN columns
    const double *base = T.src + (size_t)m * 2 * Jp * ld;
#pragma unroll
    for (int i = tid; i < 16 * BN; i += NT) {
      const int rr = i / (BN / 2), cc = (i % (BN / 2)) * 2;
      const int hs = rr >> 4, pr = rr & 15, p = q0 + pr;
      const bool v = (p < Jh) && (c0 + cc < ld);
      cp_async16(&sm.F[stage][hs][pr][cc],
                 base + (v ? ((size_t)(hs ^ T.swap_pm) * Jp + p) * ld + c0 + cc : 0), v);
    }
    if (tid < VA_KP) sm.Ps[stage][tid] = T.pscale ? T.pscale[q0 + tid] : 1.0;
  };

  double acc[2][8][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < VA_ST - 1; ++s) {
    if (s < nch) load_chunk(s, s);
    cp_async_commit();
  }
  for (int c = 0; c < nch; ++c) {
    cp_async_wait<VA_ST - 2>();
    __syncthreads();
    const int st = c % VA_ST;
    {
      const int cn = c + VA_ST - 1;
      if (cn < nch) load_chunk(cn, cn % VA_ST);
      cp_async_commit();
    }
    if (nfr == 0) continue;
    const LegTerm &T = o.t[c / nch_t];
    const int tim = T.times_im;
    const int fsel = wpar ^ T.flip;  // 0: F+, 1: F-
    const unsigned long long bmask = (tim && !(g & 1)) ? 0x8000000000000000ULL : 0ULL;
    const double asc = T.sign * (tim ? (double)m : 1.0);
    const double *Ab = &sm.A[st][wpar * VA_BR + wrh * 16 + g][t];
    const double *Bb = &sm.F[st][fsel][t][wch * 64 + (g ^ tim)];
    double a[2][2], b[2][8];
    auto frag = [&](int kk, int q) {
      const double ak = asc * sm.Ps[st][kk * 4 + t];
#pragma unroll
      for (int i = 0; i < 2; ++i) a[q][i] = Ab[i * 8 * VA_LDA + kk * 4] * ak;
#pragma unroll
      for (int j = 0; j < 8; ++j) b[q][j] = flip_sign(Bb[kk * 4 * (BN + 4) + j * 8], bmask);
    };
    frag(0, 0);
#pragma unroll
    for (int kk = 0; kk < VA_KP / 4; ++kk) {
      const int q = kk & 1;
      if (kk + 1 < VA_KP / 4) frag(kk + 1, q ^ 1);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        if (i < nfr) {
#pragma unroll
          for (int j = 0; j < 8; ++j) dmma(acc[i][j][0], acc[i][j][1], a[q][i], b[q][j]);
        }
      }
    }
  }
  cp_async_wait<0>();

  const int nt = wpar ? no : ne;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int tt = r0 + wrh * 16 + i * 8 + g;
    if (tt >= nt) continue;
    const size_t k = (size_t)off + (wpar ? ne : 0) + tt;  // parity-split row
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int col = c0 + wch * 64 + j * 8 + 2 * t;
      if (col >= ld) continue;
      *reinterpret_cast<double2 *>(o.dst + k * ld + col) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
  }
}

template <int BN>
static int synth_v2(const LegArgs &a, cudaStream_t st) {
  static bool attr = false;
  const int smem = (int)sizeof(SynthSmemV2<BN>);
  if (!attr) {
    SWE_CUDA(cudaFuncSetAttribute(leg_synth_v2<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem));
    attr = true;
  }
  dim3 grid(a.nitems, (a.ld + BN - 1) / BN, a.nout);
  leg_synth_v2<BN><<<grid, BN * 2, smem, st>>>(a);
  SWE_LAUNCH_CHECK();
  return OK;
}

template <int BN>
static int anal_v2(const LegArgs &a, cudaStream_t st) {
  static bool attr = false;
  const int smem = (int)sizeof(AnalSmemV2<BN>);
  if (!attr) {
    SWE_CUDA(cudaFuncSetAttribute(leg_anal_v2<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem));
    attr = true;
  }
  dim3 grid(a.nitems, (a.ld + BN - 1) / BN, a.nout);
  leg_anal_v2<BN><<<grid, BN * 2, smem, st>>>(a);
  SWE_LAUNCH_CHECK();
  return OK;
}

int leg_synth_v2_launch(const LegArgs &a, int bn, cudaStream_t st) {
  return bn == 128 ? synth_v2<128>(a, st) : synth_v2<64>(a, st);
}

int leg_anal_v2_launch(const LegArgs &a, int bn, cudaStream_t st) {
  return bn == 128 ? anal_v2<128>(a, st) : anal_v2<64>(a, st);
}

}  // namespace swe
