// Longitude FFT stage, "lane = row" variant.
//
// One CTA owns one latitude PAIR p (north row p, south row J-1-p) and S
// slices; its LW (16 or 8) transform rows are (field, hemisphere, slice), row
// index (f*2 + h)*S + s.  Shared memory holds X[slot][LW]: the rows of one slot
// form one line, lane r of a row group works on row r, every butterfly access
// is a conflict-free full line and the row group shares its twiddles.
// Radices 2..13 run unrolled per thread; any other prime (29 and 53 for
// M = 1024, N2 = 1537) runs as a CTA-wide "generic" stage whose thread items
// are (butterfly, GT output pairs, row).
// Inputs are the parity-split Legendre outputs E/O ([m][2][Jp][ld]):
// north = E + O, south = E - O.  Outputs are the folded analysis inputs
// F+- = w (f_north +- f_south) ([m][2][Jp][ld]); on the equator (J odd) the
// south row coincides with the north row and F+ = F- = w f_north.
// Transform algebra (real packing, Cooley-Tukey / prime-factor, slot maps) is
// shared with fft.cu.
#include <cooperative_groups.h>

#include <algorithm>

#include "fft_lanes_dev.cuh"

namespace cg = cooperative_groups;

namespace swe {

using namespace fftcore;

int g_fft_rm = 1;  // radix-specialised nonlinear lane kernels (option "fft_rm")

template <int OP, int LW, bool GEN, int RM = 0>
__global__ void __launch_bounds__(lane_threads<LW>(), 512 / lane_threads<LW>())
    fft_lanes_kernel(const __grid_constant__ FftArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr bool SPLIT = OP == FOP_NONLINEAR && LW == 8;
  LCtx c;
  c.X = reinterpret_cast<double2 *>(smem_raw);
  c.ct = c.X + (size_t)a.N2 * LW;
  c.S = lane_slices(OP, LW);
  c.split = SPLIT;
  // consecutive CTAs take consecutive slice groups of one pair: they share the
  // 32-byte sectors of the [m][2][Jp][ld] rows, which then hit in L2.  Split: the
  // two CTAs of a cluster are the two hemispheres of one slice.
  c.hem = SPLIT ? (int)(blockIdx.x & 1) : 0;
  const int grp = SPLIT ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  c.p = blockIdx.y;
  c.pin = c.p;
  c.jn = c.p;
  c.js = a.J - 1 - c.p;
  c.eq = c.js == c.jn;
  c.b0 = grp * c.S;
  c.nsl = min(c.S, a.nslices - c.b0);
  c.tid = threadIdx.x;
  c.nthr = blockDim.x;
  const int p = c.p, I = a.I, S = c.S;
  const double ia = a.inv_acos[p];

  if constexpr (OP == FOP_SYNTH_GRID || OP == FOP_SYNTH2_GRID) {
    constexpr int NF = OP == FOP_SYNTH_GRID ? 1 : 2;
    lane_load_eo<LW>(a, c, NF, -1);
    __syncthreads();
    lane_ifft<LW, GEN>(a, c);
    const double sc = (OP == FOP_SYNTH2_GRID || a.scale_mode) ? ia : 1.0;
    for (int f = 0; f < NF; ++f) lane_store_grid<LW>(a, c, a.gout[f], f, sc);
  } else if constexpr (OP == FOP_ANALYSIS || OP == FOP_VORTDIV) {
    constexpr int NF = OP == FOP_ANALYSIS ? 1 : 2;
    for (int f = 0; f < NF; ++f) lane_load_grid<LW>(a, c, a.gin[f], f);
    __syncthreads();
    if constexpr (OP == FOP_VORTDIV) {
      const double cs = a.coslat[p];
      for (int idx = c.tid; idx < a.N2 * LW; idx += c.nthr) {
        c.X[idx].x *= cs;
        c.X[idx].y *= cs;
      }
      __syncthreads();
    }
    lane_fft<LW, LW, GEN>(a, c);
    const double w = OP == FOP_ANALYSIS ? a.wq[p] * a.inv_I : a.wsin2[p] * a.inv_I * a.inv_a;
    lane_extract<LW>(a, c, c.X, c.X, NF, w, w, c.tid, c.nthr);
  } else if constexpr (OP == FOP_CORIOLIS) {
    // linear_coriolis (dynamics.py:129-135): f u, f v -> vortdiv_from_uv; f = -f on the south row
    lane_load_eo<LW>(a, c, 2, -1);
    __syncthreads();
    lane_ifft<LW, GEN>(a, c);
    const double cs = a.coslat[p], fc = a.fcor[p];
    for (int idx = c.tid; idx < a.N2 * LW; idx += c.nthr) {
      const int row = (idx & (LW - 1)) ^ swz<LW>(idx / LW);  // undo xs()
      const double fr = ((row / S) & 1) ? -fc : fc;
      const double2 z = c.X[idx];
      c.X[idx] = make_double2((fr * (z.x * ia)) * cs, (fr * (z.y * ia)) * cs);
    }
    __syncthreads();
    lane_fft<LW, LW, GEN>(a, c);
    const double w = a.wsin2[p] * a.inv_I * a.inv_a;
    lane_extract<LW>(a, c, c.X, c.X, 2, w, w, c.tid, c.nthr);
  } else if constexpr (OP == FOP_NONLINEAR && !SPLIT) {
    lane_nonlinear<LW, GEN, false, RM>(a, c);
  } else if constexpr (OP == FOP_NONLINEAR) {
    // nonlinear_advection + nonlinear_rest (dynamics.py:142-160), hemispheres split
    // over a two-CTA cluster
    // in: 0 u, 1 v, 2 d_lambda Phi, 3 H.Phi, 4 xi, 5 Phi (phi_prime applied here), 6 delta
    lane_load_eo<LW>(a, c, 7, 5);
    __syncthreads();
    lane_ifft<LW, GEN>(a, c);
    const double cs = a.coslat[p];
    constexpr int NH = SPLIT ? 1 : 2;  // hemispheres held by this CTA
    // lanes: (slot, hemisphere, x/y) fastest, so a half-warp reads one bank each
    for (int idx = c.tid; idx < I * NH * S; idx += c.nthr) {
      const int s = idx / (NH * I), r = idx - s * NH * I;
      const int pp = r / (2 * NH), h = SPLIT ? c.hem : (r >> 1) & 1, hh = r & 1;
      auto R = [&](int f) -> double & { return gslot<LW>(c, pp, hh, lrow(c, f, h, s)); };
      const double u = R(0) * ia, v = R(1) * ia, gx = R(2) * ia, gy = R(3) * ia;
      const double xi = R(4), ph = a.no_rest ? 0.0 : R(5), de = R(6);
      R(0) = -(u * gx + v * gy) - ph * de;   // -(V.grad Phi) - Phi' delta
      R(1) = 0.5 * (u * u + v * v);          // kinetic energy
      R(2) = (xi * u) * cs;                  // (xi u) cos
      R(3) = (xi * v) * cs;                  // (xi v) cos
    }
    __syncthreads();
    // only the 4 product fields (x 2 hemispheres unless split; S = 1)
    lane_fft<SPLIT ? 4 : 8 * lane_slices(OP, LW), LW, GEN>(a, c);
    const double w = a.wq[p] * a.inv_I, wv = a.wsin2[p] * a.inv_I * a.inv_a;
    if constexpr (SPLIT) {
      // F+- needs both hemispheres: each CTA of the pair folds half of the (k, field)
      // items, reading the peer's rows through distributed shared memory
      cg::cluster_group cl = cg::this_cluster();
      cl.sync();
      const double2 *XN = cl.map_shared_rank(c.X, 0), *XS = cl.map_shared_rank(c.X, 1);
      lane_extract<LW>(a, c, XN, XS, 4, w, wv, c.hem * c.nthr + c.tid, 2 * c.nthr);
      cl.sync();  // keep this CTA's rows alive until the peer is done reading them
    } else {
      lane_extract<LW>(a, c, c.X, c.X, 4, w, wv, c.tid, c.nthr);
    }
  }
}

namespace {

int lane_width(const FftArgs &a, int *rgen) {
  int g = 0;
  for (int s = 0; s < a.nst; ++s)
    if (!fft_small_radix(a.radix[s])) g = std::max(g, a.radix[s]);
  if (g) g = std::max(g, 13);  // 11 and 13 then run generic as well
  if (rgen) *rgen = g;
  const int G = (g - 1) / 2 / GT + 1;  // thread items per row of one generic butterfly
  for (int lw : {16, 8}) {
    const size_t smem = ((size_t)a.N2 * lw + g) * sizeof(double2);
    const int items = lane_threads<16>() * (lw == 16 ? 1 : 2) / lw;
    if (smem <= 227 * 1024 && (g == 0 || (g % 2 == 1 && G <= items))) return lw;
  }
  return 0;
}

template <int OP, int LW, bool GEN, int RM = 0>
int launch_lanes(const FftArgs &a, int smem, cudaStream_t st) {
  static int attr = 0;
  if (smem > attr) {
    SWE_CUDA(cudaFuncSetAttribute(fft_lanes_kernel<OP, LW, GEN, RM>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = smem;
  }
  const int S = lane_slices(OP, LW);
  const bool split = OP == FOP_NONLINEAR && LW == 8;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3((a.nslices + S - 1) / S * (split ? 2 : 1), a.Jh);
  cfg.blockDim = dim3(lane_threads<LW>());
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  if (split) {
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  SWE_CUDA(cudaLaunchKernelEx(&cfg, fft_lanes_kernel<OP, LW, GEN, RM>, a));
  SWE_LAUNCH_CHECK();
  return OK;
}

template <int LW, bool GEN>
int launch_width(int op, const FftArgs &a, int smem, cudaStream_t st) {
  switch (op) {
    case FOP_SYNTH_GRID: return launch_lanes<FOP_SYNTH_GRID, LW, GEN>(a, smem, st);
    case FOP_SYNTH2_GRID: return launch_lanes<FOP_SYNTH2_GRID, LW, GEN>(a, smem, st);
    case FOP_ANALYSIS: return launch_lanes<FOP_ANALYSIS, LW, GEN>(a, smem, st);
    case FOP_VORTDIV: return launch_lanes<FOP_VORTDIV, LW, GEN>(a, smem, st);
    case FOP_CORIOLIS: return launch_lanes<FOP_CORIOLIS, LW, GEN>(a, smem, st);
    case FOP_NONLINEAR: return launch_lanes<FOP_NONLINEAR, LW, GEN>(a, smem, st);
  }
  set_error("unknown fft op %d", op);
  return E_SHAPE;
}

}  // namespace

int fft_lanes_launch(int op, const FftArgs &a, cudaStream_t st) {
  int g = 0;
  const int lw = lane_width(a, &g);
  if (!lw) {
    set_error("internal: lane FFT does not fit N2=%d", a.N2);
    return E_SHAPE;
  }
  const int smem = (int)(((size_t)a.N2 * lw + g) * sizeof(double2));
  // the nonlinear pass of the hot factorisations: kernels holding only their stages
  if (op == FOP_NONLINEAR && lw == 16 && !g && g_fft_rm) {
    int m = 0;
    for (int s = 0; s < a.nst; ++s) m |= r_bit(a.radix[s]);
    m |= a.pfa ? RM_PFA : RM_CT;
    constexpr int R5711 = 8 | 16 | 32 | RM_PFA, R711 = 16 | 32 | RM_PFA, R7 = 16 | RM_CT;
    if (m == R5711) return launch_lanes<FOP_NONLINEAR, 16, false, R5711>(a, smem, st);
    if (m == R711) return launch_lanes<FOP_NONLINEAR, 16, false, R711>(a, smem, st);
    if (m == R7) return launch_lanes<FOP_NONLINEAR, 16, false, R7>(a, smem, st);
  }
  if (g) return lw == 16 ? launch_width<16, true>(op, a, smem, st) : launch_width<8, true>(op, a, smem, st);
  return lw == 16 ? launch_width<16, false>(op, a, smem, st) : launch_width<8, false>(op, a, smem, st);
}

bool fft_lanes_ok(const FftArgs &a) { return lane_width(a, nullptr) != 0; }

int fft_lanes_width(const FftArgs &a, int *rgen) { return lane_width(a, rgen); }

}  // namespace swe
