// Per-mode (spectral-space) kernels: layout changes, Helmholtz/Crank-Nicolson
// updates, Heun combinations, viscosity, convergence statistics.
//
// Reference: dynamics.py:52-63 (phi_prime, add_tendency), :121-126
// (linear_gravity), :181-200 (viscosity), steppers.py:61-118 (Helmholtz solve,
// Coriolis fixed point and its convergence test), :143-168 (CN / Heun).
// Internal spectral layout: [K][ld] doubles, column 2*slice + re/im.
#include "spectral.cuh"
#include "cn_cluster.cuh"

#include <cooperative_groups.h>
#include <vector>

namespace cg = cooperative_groups;

namespace swe {

// ---- layout: boundary [B][F][K] complex <-> internal F x [K][B] complex ------
// perm[k] = internal row of the reference's packed index k (parity-split order)
// ss: slice stride of the boundary array in complex elements (F * K when packed)
__global__ void k_to_internal(const double2 *__restrict__ src, SpecPtrs dst, int B, int F, int K,
                              const int *__restrict__ perm, size_t ss) {
  __shared__ double2 tile[32][33];
  const int f = blockIdx.z, k0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int b = b0 + r, k = k0 + threadIdx.x;
    if (b < B && k < K) tile[r][threadIdx.x] = src[(size_t)b * ss + (size_t)f * K + k];
  }
  __syncthreads();
  double2 *d = reinterpret_cast<double2 *>(dst.p[f]);
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int k = k0 + r, b = b0 + threadIdx.x;
    if (b < B && k < K) d[(size_t)perm[k] * B + b] = tile[threadIdx.x][r];
  }
}

__global__ void k_to_boundary(SpecPtrsC src, double2 *__restrict__ dst, int B, int F, int K,
                              const int *__restrict__ perm, const int *__restrict__ skip, size_t ss) {
  if (skip && *skip) return;
  __shared__ double2 tile[32][33];
  const int f = blockIdx.z, k0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  const double2 *s = reinterpret_cast<const double2 *>(src.p[f]);
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int k = k0 + r, b = b0 + threadIdx.x;
    if (b < B && k < K) tile[r][threadIdx.x] = s[(size_t)perm[k] * B + b];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int b = b0 + r, k = k0 + threadIdx.x;
    if (b < B && k < K) dst[(size_t)b * ss + (size_t)f * K + k] = tile[threadIdx.x][r];
  }
}

int to_internal(const double *src, const SpecPtrs &dst, int B, int F, int K, const int *perm,
                cudaStream_t st, size_t sstride) {
  dim3 grid((K + 31) / 32, (B + 31) / 32, F), blk(32, 8);
  k_to_internal<<<grid, blk, 0, st>>>(reinterpret_cast<const double2 *>(src), dst, B, F, K, perm,
                                      sstride ? sstride : (size_t)F * K);
  SWE_LAUNCH_CHECK();
  return OK;
}

int to_boundary(const SpecPtrsC &src, double *dst, int B, int F, int K, const int *perm,
                cudaStream_t st, const int *skip, size_t sstride) {
  dim3 grid((K + 31) / 32, (B + 31) / 32, F), blk(32, 8);
  k_to_boundary<<<grid, blk, 0, st>>>(src, reinterpret_cast<double2 *>(dst), B, F, K, perm, skip,
                                      sstride ? sstride : (size_t)F * K);
  SWE_LAUNCH_CHECK();
  return OK;
}

// ---- grid-stride helper over (k, b) complex elements -------------------------
#define FOR_KB(K, B)                                                                  \
  for (size_t _i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; _i < (size_t)(K) * (B); \
       _i += (size_t)gridDim.x * blockDim.x)

static inline int nblocks(size_t n) { return (int)std::min<size_t>((n + 255) / 256, 148 * 16); }

// rhs = U + alpha * (L_G U + L_C U)   (steppers.py:143-152, dynamics.py:121-139)
__global__ void k_lin_rhs(int K, int B, const double *U0, const double *U1, const double *U2,
                          const double *lcx, const double *lcd, double alpha, const double *eps,
                          const double *phibar, double *R0, double *R1, double *R2) {
  FOR_KB(K, B) {
    const int k = (int)(_i / B), b = (int)(_i - (size_t)k * B);
    const double2 ph = ld2(U0, _i), xi = ld2(U1, _i), de = ld2(U2, _i);
    const double pb = phibar[b];
    // lin.phi = -phibar*delta ; lin.xi = L_C.xi ; lin.delta = -lap(phi) + L_C.delta
    const double2 lphi = make_double2(-pb * de.x, -pb * de.y);
    const double2 lxi = lcx ? ld2(lcx, _i) : make_double2(0.0, 0.0);
    double2 lde = sc2(eps[k], ph);
    if (lcd) lde = add2(lde, ld2(lcd, _i));
    st2(R0, _i, add2(ph, sc2(alpha, lphi)));
    st2(R1, _i, add2(xi, sc2(alpha, lxi)));
    st2(R2, _i, add2(de, sc2(alpha, lde)));
  }
}

// T = L_G U (+ L_C U)   (dynamics.py:121-139)
__global__ void k_lin_tend(int K, int B, const double *U0, const double *U2, const double *lcx,
                           const double *lcd, const double *eps, const double *phibar, double *T0,
                           double *T1, double *T2) {
  FOR_KB(K, B) {
    const int k = (int)(_i / B), b = (int)(_i - (size_t)k * B);
    const double2 ph = ld2(U0, _i), de = ld2(U2, _i);
    const double pb = phibar[b];
    st2(T0, _i, make_double2(-pb * de.x, -pb * de.y));
    st2(T1, _i, lcx ? ld2(lcx, _i) : make_double2(0.0, 0.0));
    double2 d = sc2(eps[k], ph);
    if (lcd) d = add2(d, ld2(lcd, _i));
    st2(T2, _i, d);
  }
}

// u = helm(rhs + alpha*lc) (steppers.py:61-71, :96-99) for active slices, with the
// per-slice convergence statistics of steppers.py:100-109 accumulated in stats:
// stats[b*8 + f] = max|new_f|^2, stats[b*8 + 3 + f] = max|new_f - old_f|^2, as
// ordered bit patterns (squared magnitudes are >= 0, NaN sorts above Inf, so an
// unsigned max keeps NaN like np.max); k_decide takes the square roots.
// L_C at internal row k, slice b: lx = -div(fV), ld = curl(fV)   (plan.cu cor_cf);
// x, d return xi, delta of row k
SWE_DEV void cor_at(const CorOp &c, int k, int b, int B, double2 &lx, double2 &ld, double2 &x,
                    double2 &d) {
  const int2 nb = __ldg(c.nb + k);
  const double4 cf = c.cf[k];
  const size_t i = (size_t)k * B + b;
  x = ld2(c.x, i);
  d = ld2(c.d, i);
  double2 xl = make_double2(0.0, 0.0), dl = xl, xh = xl, dh = xl;
  if (nb.x >= 0) {
    xl = ld2(c.x, (size_t)nb.x * B + b);
    dl = ld2(c.d, (size_t)nb.x * B + b);
  }
  if (nb.y >= 0) {
    xh = ld2(c.x, (size_t)nb.y * B + b);
    dh = ld2(c.d, (size_t)nb.y * B + b);
  }
  // div = clo d_{n-1} + chi d_{n+1} - i cim x ; curl = clo x_{n-1} + chi x_{n+1} + i cim d
  lx = make_double2(-(cf.x * dl.x + cf.y * dh.x + cf.z * x.y),
                    -(cf.x * dl.y + cf.y * dh.y - cf.z * x.x));
  ld = make_double2(cf.x * xl.x + cf.y * xh.x - cf.z * d.y, cf.x * xl.y + cf.y * xh.y + cf.z * d.x);
  if (cf.w != 0.0) {  // m = 0: real fields (the imaginary inputs never enter)
    lx.y = 0.0;
    ld.y = 0.0;
  }
}

__global__ void k_coriolis(int K, int B, CorOp c, double *lcx, double *lcd) {
  FOR_KB(K, B) {
    const int k = (int)(_i / B), b = (int)(_i - (size_t)k * B);
    double2 lx, ld, x, d;
    cor_at(c, k, b, B, lx, ld, x, d);
    st2(lcx, _i, lx);
    st2(lcd, _i, ld);
  }
}

// convergence decision of slice b (steppers.py:100-112) from the max-norm
// statistics; resets them.  Returns whether the slice stays active.
SWE_DEV bool decide_slice(int b, double *stats, int *active, int *iters, double tol) {
  double *s = stats + (size_t)b * 8;
  bool still = false;
  if (active[b]) {
    iters[b] += 1;
    double v[6];
    for (int q = 0; q < 6; ++q) v[q] = sqrt(s[q]);  // NaN stays NaN
    double overall = fmax(fmax(v[0], v[1]), v[2]);
    if (isnan(v[0]) || isnan(v[1]) || isnan(v[2])) overall = nan("");
    overall = (overall > 1e-300 || isnan(overall)) ? overall : 1e-300;
    bool done = true;
    for (int f = 0; f < 3; ++f) {
      const double tiny = 1e-13 * overall;
      const double scale = (v[f] >= tiny || isnan(v[f])) ? v[f] : tiny;
      if (v[3 + f] > tol * scale) done = false;
    }
    if (done) active[b] = 0;
    else still = true;
  }
  for (int q = 0; q < 8; ++q) s[q] = 0.0;
  return still;
}

template <int UN>  // modes per thread in flight
__global__ void __launch_bounds__(256, UN == 4 ? 1 : 3) k_helm(int K, int B, const double *R0, const double *R1,
                                              const double *R2, const double *lcx,
                                              const double *lcd, double alpha, const double *eps,
                                              const double *phibar, double *U0, double *U1,
                                              double *U2, const int *active, double *stats,
                                              CorOp cor, int *iters, int *counter,
                                              double tol, unsigned *hdone) {
  // block: bx slices x by mode rows (bx = 32, or the batch rounded up to a power of
  // two when smaller, so small batches keep every lane busy); grid.x over slice
  // tiles, grid.y over modes
  __shared__ unsigned long long red[256][6];
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long mx[6] = {0, 0, 0, 0, 0, 0};
  const bool fused = cor.x != nullptr;
  if (counter && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && threadIdx.y == 0)
    *counter = 0;  // k_decide (stream-ordered after this kernel) counts afresh
  const bool act = (b < B) && (active == nullptr || active[b]);
  // fused: xi/delta ping-pong per slice between A = (cor.x, cor.d) and B = (U1, U2);
  // the current iterate of slice b is in B when iters[b] is odd
  CorOp src = cor;
  double *W1 = U1, *W2 = U2;
  if (fused && act && (iters[b] & 1)) {
    src.x = U1;
    src.d = U2;
    W1 = const_cast<double *>(cor.x);
    W2 = const_cast<double *>(cor.d);
  }
  const double *O1 = fused ? src.x : U1, *O2 = fused ? src.d : U2;
  const int k0 = blockIdx.y * blockDim.y + threadIdx.y, stride = gridDim.y * blockDim.y;
  if (act) {
    const double pb = phibar[b], apb = alpha * pb, aap = alpha * alpha * pb;
    for (int kb = k0; kb < K; kb += UN * stride) {
      double2 rp[UN], rx[UN], rd[UN], o0[UN], o1[UN], o2[UN];
      double e[UN];
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        const int k = kb + u * stride;
        if (k < K) {
          const size_t i = (size_t)k * B + b;
          rp[u] = ld2(R0, i);
          rx[u] = ld2(R1, i);
          rd[u] = ld2(R2, i);
          if (fused) {
            double2 lx, ld;
            cor_at(src, k, b, B, lx, ld, o1[u], o2[u]);
            rx[u] = add2(rx[u], sc2(alpha, lx));
            rd[u] = add2(rd[u], sc2(alpha, ld));
          } else if (lcx) {
            rx[u] = add2(rx[u], sc2(alpha, ld2(lcx, i)));
            rd[u] = add2(rd[u], sc2(alpha, ld2(lcd, i)));
          }
          e[u] = eps[k];
          if (stats) {
            o0[u] = ld2(U0, i);
            if (!fused) {
              o1[u] = ld2(O1, i);
              o2[u] = ld2(O2, i);
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        const int k = kb + u * stride;
        if (k >= K) continue;
        const size_t i = (size_t)k * B + b;
        const double denom = 1.0 + aap * e[u];
        const double2 ph = make_double2((rp[u].x - apb * rd[u].x) / denom,
                                        (rp[u].y - apb * rd[u].y) / denom);
        const double ae = alpha * e[u];
        const double2 de = make_double2(rd[u].x + ae * ph.x, rd[u].y + ae * ph.y);
        if (stats) {
          mx[0] = max(mx[0], sqmag_bits(ph.x, ph.y));
          mx[1] = max(mx[1], sqmag_bits(rx[u].x, rx[u].y));
          mx[2] = max(mx[2], sqmag_bits(de.x, de.y));
          mx[3] = max(mx[3], sqmag_bits(ph.x - o0[u].x, ph.y - o0[u].y));
          mx[4] = max(mx[4], sqmag_bits(rx[u].x - o1[u].x, rx[u].y - o1[u].y));
          mx[5] = max(mx[5], sqmag_bits(de.x - o2[u].x, de.y - o2[u].y));
        }
        st2(U0, i, ph);
        st2(W1, i, rx[u]);
        st2(W2, i, de);
      }
    }
  }
  if (!stats) return;
#pragma unroll
  for (int q = 0; q < 6; ++q) red[threadIdx.y * blockDim.x + threadIdx.x][q] = mx[q];
  __syncthreads();
  if (threadIdx.y == 0 && act) {
    for (int q = 0; q < 6; ++q) {
      unsigned long long v = red[threadIdx.x][q];
      for (int r = 1; r < blockDim.y; ++r) v = max(v, red[r * blockDim.x + threadIdx.x][q]);
      atomicMax(reinterpret_cast<unsigned long long *>(stats) + (size_t)b * 8 + q, v);
    }
    if (hdone) __threadfence();  // this block's statistics before its check-in
  }
  if (!hdone) return;
  // the last block to finish decides every slice (k_decide fused: one launch less
  // per fixed-point iteration); hdone returns to 0 for the next launch
  __shared__ bool last;
  __shared__ int cnt;
  __syncthreads();
  const int tid = threadIdx.y * blockDim.x + threadIdx.x, nthr = blockDim.x * blockDim.y;
  if (tid == 0) {
    last = atomicAdd(hdone, 1u) == gridDim.x * gridDim.y - 1;
    cnt = 0;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int bb = tid; bb < B; bb += nthr)
    if (decide_slice(bb, stats, const_cast<int *>(active), iters, tol)) atomicAdd(&cnt, 1);
  __syncthreads();
  if (tid == 0) {
    *counter = cnt;
    *hdone = 0;
  }
}

// Tiled fixed-point iterate (batches of >= 32 slices): one CTA = one chunk of 64
// consecutive n of an m-block (32 even + 32 odd rows of the parity-split order)
// x 32 slices.  The previous iterate's xi/delta rows of the chunk plus one halo
// row per parity are staged in shared memory with coalesced loads, so the
// three-term Coriolis stencil reads its neighbours there; rhs and Phi stream
// straight through.  Same arithmetic and statistics as k_helm.
constexpr int HT_ROWS = 33;
__global__ void __launch_bounds__(256, 3)
    k_helm_tiled(int M, int B, const int *__restrict__ offsets, const int2 *__restrict__ tiles,
                 const double *R0, const double *R1, const double *R2, double alpha,
                 const double *eps, const double *phibar, double *U0, double *A1, double *A2,
                 double *B1, double *B2, const double4 *__restrict__ cfc, const int *active,
                 double *stats, const int *iters, int *counter) {
  extern __shared__ double2 hsm[];  // [field xi/delta][parity][HT_ROWS][32]
  if (counter && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && threadIdx.y == 0)
    *counter = 0;  // for the k_decide that follows
  const int2 tl = tiles[blockIdx.x];
  const int m = tl.x, c = tl.y;
  const int km = M + 1 - m, ne = (km + 1) >> 1, no = km >> 1, off = offsets[m];
  const int lane = threadIdx.x, ty = threadIdx.y;
  const int b = blockIdx.y * 32 + lane;
  const bool act = b < B && active[b];
  const bool odd_it = act && (iters[b] & 1);
  const double *X = odd_it ? B1 : A1, *D = odd_it ? B2 : A2;
  double *WX = odd_it ? A1 : B1, *WD = odd_it ? A2 : B2;
  auto sm = [&](int f, int p, int j) -> double2 & {
    return hsm[((f * 2 + p) * HT_ROWS + j) * 32 + lane];
  };
  for (int t = ty; t < 2 * HT_ROWS; t += blockDim.y) {
    const int p = t >= HT_ROWS, j = t - p * HT_ROWS;
    const int gi = 32 * c + j - p;  // even rows 32c.., odd rows 32c-1..
    double2 x = make_double2(0.0, 0.0), d = x;
    if (act && gi >= 0 && gi < (p ? no : ne)) {
      const size_t i = (size_t)(off + (p ? ne : 0) + gi) * B + b;
      x = ld2(X, i);
      d = ld2(D, i);
    }
    sm(0, p, j) = x;
    sm(1, p, j) = d;
  }
  __syncthreads();
  unsigned long long mx[6] = {0, 0, 0, 0, 0, 0};
  if (act) {
    const double pb = phibar[b], apb = alpha * pb, aap = alpha * alpha * pb;
#pragma unroll 2
    for (int q = 0; q < 8; ++q) {
      const int p = q & 1, li = ty * 4 + (q >> 1), gi = 32 * c + li;
      if (gi >= (p ? no : ne)) continue;
      const int k = off + (p ? ne : 0) + gi;
      const size_t i = (size_t)k * B + b;
      const double2 rp = ld2(R0, i), r1 = ld2(R1, i), r2 = ld2(R2, i), o0 = ld2(U0, i);
      const double e = eps[k];
      const double4 cf = cfc[k];
      // self row and the n-1 / n+1 rows (other parity) from shared memory
      const int js = p ? li + 1 : li;
      const double2 x = sm(0, p, js), d = sm(1, p, js);
      const double2 xl = sm(0, 1 - p, li), dl = sm(1, 1 - p, li);
      const double2 xh = sm(0, 1 - p, li + 1), dh = sm(1, 1 - p, li + 1);
      double2 lx = make_double2(-(cf.x * dl.x + cf.y * dh.x + cf.z * x.y),
                                -(cf.x * dl.y + cf.y * dh.y - cf.z * x.x));
      double2 lc = make_double2(cf.x * xl.x + cf.y * xh.x - cf.z * d.y,
                                cf.x * xl.y + cf.y * xh.y + cf.z * d.x);
      if (cf.w != 0.0) {
        lx.y = 0.0;
        lc.y = 0.0;
      }
      const double2 rx = add2(r1, sc2(alpha, lx)), rd = add2(r2, sc2(alpha, lc));
      const double denom = 1.0 + aap * e;
      const double2 ph = make_double2((rp.x - apb * rd.x) / denom, (rp.y - apb * rd.y) / denom);
      const double ae = alpha * e;
      const double2 de = make_double2(rd.x + ae * ph.x, rd.y + ae * ph.y);
      mx[0] = max(mx[0], sqmag_bits(ph.x, ph.y));
      mx[1] = max(mx[1], sqmag_bits(rx.x, rx.y));
      mx[2] = max(mx[2], sqmag_bits(de.x, de.y));
      mx[3] = max(mx[3], sqmag_bits(ph.x - o0.x, ph.y - o0.y));
      mx[4] = max(mx[4], sqmag_bits(rx.x - x.x, rx.y - x.y));
      mx[5] = max(mx[5], sqmag_bits(de.x - d.x, de.y - d.y));
      st2(U0, i, ph);
      st2(WX, i, rx);
      st2(WD, i, de);
    }
  }
  // per-slice statistics: reduce over ty in shared memory (reusing the stage)
  __syncthreads();
  unsigned long long *red = reinterpret_cast<unsigned long long *>(hsm);
#pragma unroll
  for (int q = 0; q < 6; ++q) red[(ty * 32 + lane) * 6 + q] = mx[q];
  __syncthreads();
  if (ty == 0 && act) {
    for (int q = 0; q < 6; ++q) {
      unsigned long long v = red[lane * 6 + q];
      for (int r = 1; r < blockDim.y; ++r) v = max(v, red[(r * 32 + lane) * 6 + q]);
      atomicMax(reinterpret_cast<unsigned long long *>(stats) + (size_t)b * 8 + q, v);
    }
  }
}

int helm_tiled(int M, int K, int B, const int *offsets, const int2 *tiles, int ntiles,
               const double *const R[3], double alpha, const double *eps, const double *phibar,
               double *U0, double *A1, double *A2, double *B1, double *B2, const double4 *cf,
               const int *active, double *stats, const int *iters, int *counter,
               cudaStream_t st) {
  (void)K;
  const int smem = 4 * HT_ROWS * 32 * (int)sizeof(double2);
  static bool attr = false;
  if (!attr) {
    SWE_CUDA(cudaFuncSetAttribute(k_helm_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  dim3 grid(ntiles, (B + 31) / 32), blk(32, 8);
  k_helm_tiled<<<grid, blk, smem, st>>>(M, B, offsets, tiles, R[0], R[1], R[2], alpha, eps, phibar,
                                        U0, A1, A2, B1, B2, cf, active, stats, iters, counter);
  SWE_LAUNCH_CHECK();
  return OK;
}

// Crank-Nicolson half step prologue (steppers.py:143-152) in one pass:
//   X   = x0 + s (x1 + x2)                  (x1, x2 nullable: the Heun combination)
//   R   = X + alpha (L_G X + L_C X)         (L_C spectral, omitted when c.nb == null)
//   dst = helm(R)                           (first fixed-point iterate, no L_C)

__global__ void __launch_bounds__(256) k_cn_start(int K, int B, Ptr3C x0, Ptr3C x1, Ptr3C x2,
                                                  double s, double alpha, const double *eps,
                                                  const double *phibar, CorOp c, Ptr3 R,
                                                  Ptr3 dst) {
  FOR_KB(K, B) {
    const int k = (int)(_i / B), b = (int)(_i - (size_t)k * B);
    const double2 ph = comb(x0, x1, x2, s, 0, _i), xi = comb(x0, x1, x2, s, 1, _i),
                  de = comb(x0, x1, x2, s, 2, _i);
    const double pb = phibar[b], e = eps[k];
    double2 lx = make_double2(0.0, 0.0), lc = lx;
    if (c.nb) {  // L_C of X (plan.cu cor_cf), neighbours combined on the fly
      const int2 nb = c.nb[k];
      const double4 cf = c.cf[k];
      double2 xl = lx, dl = lx, xh = lx, dh = lx;
      if (nb.x >= 0) {
        xl = comb(x0, x1, x2, s, 1, (size_t)nb.x * B + b);
        dl = comb(x0, x1, x2, s, 2, (size_t)nb.x * B + b);
      }
      if (nb.y >= 0) {
        xh = comb(x0, x1, x2, s, 1, (size_t)nb.y * B + b);
        dh = comb(x0, x1, x2, s, 2, (size_t)nb.y * B + b);
      }
      lx = make_double2(-(cf.x * dl.x + cf.y * dh.x + cf.z * xi.y),
                        -(cf.x * dl.y + cf.y * dh.y - cf.z * xi.x));
      lc = make_double2(cf.x * xl.x + cf.y * xh.x - cf.z * de.y,
                        cf.x * xl.y + cf.y * xh.y + cf.z * de.x);
      if (cf.w != 0.0) {
        lx.y = 0.0;
        lc.y = 0.0;
      }
    }
    // rhs = X + alpha * (L_G X + L_C X)  (as k_lin_rhs)
    const double2 lphi = make_double2(-pb * de.x, -pb * de.y);
    const double2 lde = add2(sc2(e, ph), lc);
    const double2 r0 = add2(ph, sc2(alpha, lphi)), r1 = add2(xi, sc2(alpha, lx)),
                  r2 = add2(de, sc2(alpha, lde));
    st2(R.p[0], _i, r0);
    st2(R.p[1], _i, r1);
    st2(R.p[2], _i, r2);
    // helm(R) (as k_helm without L_C)
    const double apb = alpha * pb, denom = 1.0 + alpha * alpha * pb * e;
    const double2 nph = make_double2((r0.x - apb * r2.x) / denom, (r0.y - apb * r2.y) / denom);
    const double ae = alpha * e;
    st2(dst.p[0], _i, nph);
    st2(dst.p[1], _i, r1);
    st2(dst.p[2], _i, make_double2(r2.x + ae * nph.x, r2.y + ae * nph.y));
  }
}

// Whole Crank-Nicolson half step for small truncations (coarse levels): one CTA
// per slice runs prologue (as k_cn_start), the complete Coriolis fixed point (as
// k_helm + k_decide, the slice's own convergence loop) and the epilogue (as
// k_cn_finish) in one launch, with the iterate (Phi and two xi/delta buffers) in
// shared memory and block-level reductions for the statistics.  Same arithmetic
// as the multi-kernel path, so results are identical; it removes ~12 launches
// per half step where launch latency dominates.  rhs_given: R = X (the SETTLS
// implicit solve).  Not converged after max_iter: the residual of
// steppers.py:113-118 goes to resid[b], *counter counts such slices.
constexpr int CS_NT = 1024;
SWE_DEV unsigned long long blk_max_u64(unsigned long long v, unsigned long long *red) {
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < (int)(blockDim.x >> 5) ? red[l] : 0ULL;
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (l == 0) red[32] = v;
  }
  __syncthreads();
  return red[32];
}

__global__ void __launch_bounds__(CS_NT) k_cn_small(int K, int B, Ptr3C x0, Ptr3C x1, Ptr3C x2,
                                                  double s, double alpha, const double *eps,
                                                  const double *phibar, const int2 *nbt,
                                                  const double4 *cft, int rhs_given, Ptr3 R,
                                                  Ptr3 dst, int max_iter, double tol, double dtnu,
                                                  double halfq, int *iters, int *flags,
                                                  int *counter, double *resid, int *fail) {
  extern __shared__ double2 csm[];  // [Phi][xi A][xi B][de A][de B], K each
  double2 *P = csm, *XA = csm + K, *XB = csm + 2 * K, *DA = csm + 3 * K, *DB = csm + 4 * K;
  __shared__ unsigned long long red[33];
  __shared__ unsigned long long red6[6][CS_NT / 32];
  __shared__ int sdone;
  const int b = blockIdx.x;
  const bool cor = nbt != nullptr;
  const double pb = phibar[b], apb = alpha * pb, aap = alpha * alpha * pb;
  auto at = [&](int k) { return (size_t)k * B + b; };
  // ---- prologue: stage X's xi/delta, then rhs R and the first iterate
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    XB[k] = comb(x0, x1, x2, s, 1, at(k));
    DB[k] = comb(x0, x1, x2, s, 2, at(k));
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const double2 ph = comb(x0, x1, x2, s, 0, at(k)), xi = XB[k], de = DB[k];
    const double e = eps[k];
    double2 r0, r1, r2;
    if (rhs_given) {
      r0 = ph;
      r1 = xi;
      r2 = de;
    } else {
      double2 lx = make_double2(0.0, 0.0), lc = lx;
      if (cor) {
        const int2 nb = nbt[k];
        const double4 cf = cft[k];
        double2 xl = lx, dl = lx, xh = lx, dh = lx;
        if (nb.x >= 0) {
          xl = XB[nb.x];
          dl = DB[nb.x];
        }
        if (nb.y >= 0) {
          xh = XB[nb.y];
          dh = DB[nb.y];
        }
        lx = make_double2(-(cf.x * dl.x + cf.y * dh.x + cf.z * xi.y),
                          -(cf.x * dl.y + cf.y * dh.y - cf.z * xi.x));
        lc = make_double2(cf.x * xl.x + cf.y * xh.x - cf.z * de.y,
                          cf.x * xl.y + cf.y * xh.y + cf.z * de.x);
        if (cf.w != 0.0) {
          lx.y = 0.0;
          lc.y = 0.0;
        }
      }
      const double2 lphi = make_double2(-pb * de.x, -pb * de.y);
      const double2 lde = add2(sc2(e, ph), lc);
      r0 = add2(ph, sc2(alpha, lphi));
      r1 = add2(xi, sc2(alpha, lx));
      r2 = add2(de, sc2(alpha, lde));
    }
    st2(R.p[0], at(k), r0);
    st2(R.p[1], at(k), r1);
    st2(R.p[2], at(k), r2);
    const double denom = 1.0 + aap * e;
    const double2 nph = make_double2((r0.x - apb * r2.x) / denom, (r0.y - apb * r2.y) / denom);
    const double ae = alpha * e;
    P[k] = nph;
    XA[k] = r1;
    DA[k] = make_double2(r2.x + ae * nph.x, r2.y + ae * nph.y);
  }
  __syncthreads();
  // ---- fixed point (steppers.py:96-112), the slice's own loop
  int it = 0, done = !cor;
  double2 *cx = XA, *cd = DA, *nx = XB, *nd = DB;
  for (; !done && it < max_iter; ++it) {
    unsigned long long mx[6] = {0, 0, 0, 0, 0, 0};
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
      const int2 nb = nbt[k];
      const double4 cf = cft[k];
      const double2 rp = ld2(R.p[0], at(k)), r1 = ld2(R.p[1], at(k)), r2 = ld2(R.p[2], at(k));
      const double e = eps[k];
      const double2 x = cx[k], d = cd[k];
      double2 xl = make_double2(0.0, 0.0), dl = xl, xh = xl, dh = xl;
      if (nb.x >= 0) {
        xl = cx[nb.x];
        dl = cd[nb.x];
      }
      if (nb.y >= 0) {
        xh = cx[nb.y];
        dh = cd[nb.y];
      }
      double2 lx = make_double2(-(cf.x * dl.x + cf.y * dh.x + cf.z * x.y),
                                -(cf.x * dl.y + cf.y * dh.y - cf.z * x.x));
      double2 lc = make_double2(cf.x * xl.x + cf.y * xh.x - cf.z * d.y,
                                cf.x * xl.y + cf.y * xh.y + cf.z * d.x);
      if (cf.w != 0.0) {
        lx.y = 0.0;
        lc.y = 0.0;
      }
      const double2 rx = add2(r1, sc2(alpha, lx)), rd = add2(r2, sc2(alpha, lc));
      const double denom = 1.0 + aap * e;
      const double2 ph = make_double2((rp.x - apb * rd.x) / denom, (rp.y - apb * rd.y) / denom);
      const double ae = alpha * e;
      const double2 de = make_double2(rd.x + ae * ph.x, rd.y + ae * ph.y);
      const double2 o0 = P[k];
      mx[0] = max(mx[0], sqmag_bits(ph.x, ph.y));
      mx[1] = max(mx[1], sqmag_bits(rx.x, rx.y));
      mx[2] = max(mx[2], sqmag_bits(de.x, de.y));
      mx[3] = max(mx[3], sqmag_bits(ph.x - o0.x, ph.y - o0.y));
      mx[4] = max(mx[4], sqmag_bits(rx.x - x.x, rx.y - x.y));
      mx[5] = max(mx[5], sqmag_bits(de.x - d.x, de.y - d.y));
      P[k] = ph;
      nx[k] = rx;
      nd[k] = de;
    }
    // the 6 block maxima in one pass: warp shuffles, one staging barrier, warp 0
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      for (int o = 16; o > 0; o >>= 1) mx[q] = max(mx[q], __shfl_xor_sync(0xffffffffu, mx[q], o));
      if (lane == 0) red6[q][warp] = mx[q];
    }
    __syncthreads();
    if (warp == 0) {
      double v[6];
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        unsigned long long x = lane < (int)(blockDim.x >> 5) ? red6[q][lane] : 0ULL;
        for (int o = 16; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
        v[q] = sqrt(__longlong_as_double((long long)x));  // as decide_slice
      }
      double overall = fmax(fmax(v[0], v[1]), v[2]);
      if (isnan(v[0]) || isnan(v[1]) || isnan(v[2])) overall = nan("");
      overall = (overall > 1e-300 || isnan(overall)) ? overall : 1e-300;
      bool ok = true;
      for (int f = 0; f < 3; ++f) {
        const double tiny = 1e-13 * overall;
        const double scale = (v[f] >= tiny || isnan(v[f])) ? v[f] : tiny;
        if (v[3 + f] > tol * scale) ok = false;
      }
      if (lane == 0) sdone = ok;
    }
    __syncthreads();
    done = sdone;
    double2 *t = cx;
    cx = nx;
    nx = t;
    t = cd;
    cd = nd;
    nd = t;
  }
  if (threadIdx.x == 0) {
    iters[b] = it;
    flags[b] = !done;
    resid[b] = 0.0;
  }
  if (!done) {
    // residual |u - alpha (L_G + L_C) u - rhs| (steppers.py:113-118)
    double rmax = 0.0;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
      const int2 nb = nbt[k];
      const double4 cf = cft[k];
      const double2 x = cx[k], d = cd[k], ph = P[k];
      double2 xl = make_double2(0.0, 0.0), dl = xl, xh = xl, dh = xl;
      if (nb.x >= 0) {
        xl = cx[nb.x];
        dl = cd[nb.x];
      }
      if (nb.y >= 0) {
        xh = cx[nb.y];
        dh = cd[nb.y];
      }
      double2 lx = make_double2(-(cf.x * dl.x + cf.y * dh.x + cf.z * x.y),
                                -(cf.x * dl.y + cf.y * dh.y - cf.z * x.x));
      double2 lc = make_double2(cf.x * xl.x + cf.y * xh.x - cf.z * d.y,
                                cf.x * xl.y + cf.y * xh.y + cf.z * d.x);
      if (cf.w != 0.0) {
        lx.y = 0.0;
        lc.y = 0.0;
      }
      const double2 lph = make_double2(-pb * d.x, -pb * d.y);
      const double2 lde = add2(sc2(eps[k], ph), lc);
      const double2 v[3] = {ph, x, d}, l[3] = {lph, lx, lde};
      for (int f = 0; f < 3; ++f) {
        const double2 rr = ld2(R.p[f], at(k));
        rmax = fmax(rmax, hypot(v[f].x - alpha * l[f].x - rr.x, v[f].y - alpha * l[f].y - rr.y));
      }
    }
    const double r = __longlong_as_double(
        (long long)blk_max_u64((unsigned long long)__double_as_longlong(rmax), red));
    if (threadIdx.x == 0) {
      resid[b] = r;
      atomicAdd(counter, 1);
      if (fail) *fail = 1;
    }
  }
  // ---- epilogue: viscosity factor (dynamics.py:191-200) and the result
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double bh = 1.0;
    if (dtnu != 0.0 && done) bh = 1.0 / (1.0 + dtnu * pow(eps[k], halfq));
    const double2 ph = P[k], x = cx[k], d = cd[k];
    st2(dst.p[0], at(k), dtnu != 0.0 && done ? sc2(bh, ph) : ph);
    st2(dst.p[1], at(k), dtnu != 0.0 && done ? sc2(bh, x) : x);
    st2(dst.p[2], at(k), dtnu != 0.0 && done ? sc2(bh, d) : d);
  }
}

int cn_small_ok(int K) { return K <= 2800; }

int cn_small(int K, int B, Ptr3C x0, Ptr3C x1, Ptr3C x2, double s, double alpha,
             const double *eps, const double *phibar, const int2 *nb, const double4 *cf,
             int rhs_given, Ptr3 R, Ptr3 dst, int max_iter, double tol, double dtnu,
             double halfq, int *iters, int *flags, int *counter, double *resid, int *fail,
             cudaStream_t st) {
  const int smem = 5 * K * (int)sizeof(double2);
  static int attr = 0;
  if (smem > attr) {
    SWE_CUDA(cudaFuncSetAttribute(k_cn_small, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = smem;
  }
  k_cn_small<<<B, CS_NT, smem, st>>>(K, B, x0, x1, x2, s, alpha, eps, phibar, nb, cf, rhs_given,
                                     R, dst, max_iter, tol, dtnu, halfq, iters, flags, counter,
                                     resid, fail);
  SWE_LAUNCH_CHECK();
  return OK;
}

// k_cn_cluster: see cn_cluster.cuh for the half step it runs
__global__ void __launch_bounds__(CC_NT, 1) k_cn_cluster(
    int K, int B, const __grid_constant__ CcRanges rg, int cap, Ptr3C x0, Ptr3C x1, Ptr3C x2, double s, double alpha,
    const double *eps, const double *phibar, const int2 *nbt, const double4 *cft,
    int rhs_given, Ptr3 dst, int max_iter, double tol, double dtnu, double halfq, int *iters,
    int *flags, int *counter, double *resid, int *fail) {
  extern __shared__ double2 ccm[];
  __shared__ CcShared sh;
  cn_cluster_body<false>(K, B, rg, cap, x0, x1, x2, s, alpha, eps, phibar, nbt, cft, rhs_given,
                         dst, max_iter, tol, dtnu, halfq, iters, flags, counter, resid, fail, ccm,
                         sh);
}

// CTA ranges for a C-CTA cluster over the m-blocks of truncation M (block m has
// M+1-m modes, packed m-major): boundaries on block starts, each placed at the block
// start nearest to c*K/C; returns the largest range (0 if it exceeds CC_CHUNK)
static int cc_ranges(int M, int C, CcRanges &rg) {
  const int K = (M + 1) * (M + 2) / 2;
  rg.k[0] = 0;
  int c = 1, cum = 0;
  for (int m = 0; m <= M && c < C; ++m) {
    const int next = cum + (M + 1 - m);
    const double t = (double)c * K / C;
    if (next >= t) {  // boundary before or after block m, whichever is nearer
      rg.k[c] = (t - cum <= next - t && cum > rg.k[c - 1]) ? cum : next;
      ++c;
    }
    cum = next;
  }
  while (c < C) rg.k[c++] = K;
  rg.k[C] = K;
  int cap = 0;
  for (int i = 0; i < C; ++i) cap = std::max(cap, rg.k[i + 1] - rg.k[i]);
  return cap <= CC_CHUNK ? cap : 0;
}

int cn_cluster_ranges(int M, int C, CcRanges *rg) { return cc_ranges(M, C, *rg); }

// cluster size for truncation M (0: the cluster path does not apply or cannot be
// scheduled)
int cn_cluster_size(int M, int want) {
  static std::vector<int3> cache;  // (M, want, C)
  static int attr_smem = 0;
  for (const int3 &e : cache)
    if (e.x == M && e.y == want) return e.z;
  const int K = (M + 1) * (M + 2) / 2;
  int C = 0, cap = 0;
  CcRanges rg;
  const int c0 = std::max(std::max(1, want), (K + CC_CHUNK - 1) / CC_CHUNK);
  for (int c = std::min(c0, CC_MAXC); c <= CC_MAXC && !cap; ++c) {
    const int cc = (c > 8 && want <= 8) ? CC_MAXC : c;  // non-portable sizes: the smallest ranges
    if ((cap = cc_ranges(M, cc, rg))) C = cc;
  }
  int ok = 0;
  if (C) {
    // the attribute only grows: graphs captured for another truncation keep launching
    const int smem = 6 * cap * (int)sizeof(double2);
    if ((smem <= attr_smem ||
         cudaFuncSetAttribute(k_cn_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) ==
             cudaSuccess) &&
        (C <= 8 || cudaFuncSetAttribute(k_cn_cluster,
                                        cudaFuncAttributeNonPortableClusterSizeAllowed,
                                        1) == cudaSuccess)) {
      attr_smem = std::max(attr_smem, smem);
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
      if (cudaOccupancyMaxActiveClusters(&nc, k_cn_cluster, &cfg) == cudaSuccess && nc > 0) ok = 1;
    }
    cudaGetLastError();  // a refused configuration is not an error: the multi-kernel path runs
  }
  cache.push_back(make_int3(M, want, ok ? C : 0));
  return ok ? C : 0;
}

int cn_cluster(int M, int want, int B, Ptr3C x0, Ptr3C x1, Ptr3C x2, double s, double alpha,
               const double *eps, const double *phibar, const int2 *nb, const double4 *cf,
               int rhs_given, Ptr3 dst, int max_iter, double tol, double dtnu, double halfq,
               int *iters, int *flags, int *counter, double *resid, int *fail, cudaStream_t st) {
  const int C = cn_cluster_size(M, want), K = (M + 1) * (M + 2) / 2;
  CcRanges rg;
  const int cap = C ? cc_ranges(M, C, rg) : 0;
  if (!cap) {
    set_error("internal: cluster CN half step not available for M=%d", M);
    return E_SHAPE;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(C * B);
  cfg.blockDim = dim3(CC_NT);
  cfg.dynamicSmemBytes = 6 * cap * sizeof(double2);
  cfg.stream = st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  SWE_CUDA(cudaLaunchKernelEx(&cfg, k_cn_cluster, K, B, rg, cap, x0, x1, x2, s, alpha, eps,
                              phibar, nb, cf, rhs_given, dst, max_iter, tol, dtnu, halfq, iters,
                              flags, counter, resid, fail));
  SWE_LAUNCH_CHECK();
  return OK;
}

// Direct solve of the Crank-Nicolson implicit system (I - a (L_G + L_C)) U = R,
// SURVEY.md §8f row 4 (the reference iterates it to tol, steppers.py:74-118; the
// converged iterate and this solution agree to ~tol).  Eliminating
// Phi = r0 - a Pb delta leaves, per order m and slice, two decoupled complex
// tridiagonal chains in n: xi_n couples to delta_{n-+1} and delta_n to xi_{n-+1}, so
// chain c = 0 holds xi at even n-m and delta at odd n-m, chain 1 the others:
//   xi_n:    (1 - i a cz_n) xi_n + a cx_n d_{n-1} + a cy_n d_{n+1} = r1_n
//   delta_n: (1 + a^2 Pb eps_n - i a cz_n) d_n - a cx_n x_{n-1} - a cy_n x_{n+1}
//            = r2_n + a eps_n r0_n
// (cx, cy, cz = plan.cu cor_cf).  m = 0 keeps real parts only in L_C, so there the
// imaginary parts decouple.  Thomas elimination, one thread per (m, chain, slice),
// slices fastest (coalesced rows of the [K][B] layout), longest chains (m = 0)
// first.  Forward pass: R from X = x0 + s (x1 + x2) on the fly (or R = X), the
// modified coefficients c'_j, d'_j and r0 to scratch; backward pass (a second
// launch, since dst may alias x0): back substitution, Phi, viscosity -> dst.
// The chains are diagonally dominant for the CN step sizes (|a cx|, |a cy| << 1).
SWE_DEV int cd_row(int M, int m, int n) {
  const int d = n - m, ne = (M + 2 - m) / 2, off = m * (M + 1) - m * (m - 1) / 2;
  return off + ((d & 1) ? ne + (d >> 1) : (d >> 1));
}
SWE_DEV double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
SWE_DEV double2 cdiv(double2 a, double2 b) {
  const double inv = 1.0 / (b.x * b.x + b.y * b.y);
  return make_double2((a.x * b.x + a.y * b.y) * inv, (a.y * b.x - a.x * b.y) * inv);
}

// pass 1 (one thread per mode and slice, fully parallel): the right-hand sides of
// both chain rows of mode k -- the xi row r1 and the delta row r2 + a eps r0 -- and
// r0, from X = x0 + s (x1 + x2) (or R = X given)
__global__ void __launch_bounds__(256) k_cn_direct_rhs(int K, int B, Ptr3C x0, Ptr3C x1,
                                                       Ptr3C x2, double s, double alpha,
                                                       const double *eps, const double *phibar,
                                                       const int2 *nbt, const double4 *cft,
                                                       int rhs_given, Ptr3 sc) {
  FOR_KB(K, B) {
    const int k = (int)(_i / B), b = (int)(_i - (size_t)k * B);
    auto at = [&](int kk) { return (size_t)kk * B + b; };
    const double a = alpha, e = eps[k], pb = phibar[b];
    const double2 ph = comb(x0, x1, x2, s, 0, _i), xi = comb(x0, x1, x2, s, 1, _i),
                  de = comb(x0, x1, x2, s, 2, _i);
    double2 r0, r1, r2;
    if (rhs_given) {
      r0 = ph;
      r1 = xi;
      r2 = de;
    } else {
      const int2 nb = nbt[k];
      const double4 cf = cft[k];
      double2 xl = make_double2(0.0, 0.0), dl = xl, xh = xl, dh = xl;
      if (nb.x >= 0) {
        xl = comb(x0, x1, x2, s, 1, at(nb.x));
        dl = comb(x0, x1, x2, s, 2, at(nb.x));
      }
      if (nb.y >= 0) {
        xh = comb(x0, x1, x2, s, 1, at(nb.y));
        dh = comb(x0, x1, x2, s, 2, at(nb.y));
      }
      double2 lx = make_double2(-(cf.x * dl.x + cf.y * dh.x + cf.z * xi.y),
                                -(cf.x * dl.y + cf.y * dh.y - cf.z * xi.x));
      double2 lc = make_double2(cf.x * xl.x + cf.y * xh.x - cf.z * de.y,
                                cf.x * xl.y + cf.y * xh.y + cf.z * de.x);
      if (cf.w != 0.0) {
        lx.y = 0.0;
        lc.y = 0.0;
      }
      r0 = add2(ph, sc2(a, make_double2(-pb * de.x, -pb * de.y)));
      r1 = add2(xi, sc2(a, lx));
      r2 = add2(de, sc2(a, add2(sc2(e, ph), lc)));
    }
    st2(sc.p[0], _i, r0);
    st2(sc.p[1], _i, r1);
    st2(sc.p[2], _i, add2(r2, sc2(a * e, r0)));
  }
}

// pass 2: one chain (m, c) of slice b solved from both ends at once ("twisted"
// factorization): lane l < 16 of a warp eliminates rows 0..p-1 downwards
// (u_j = d'_j - c'_j u_{j+1}), lane l + 16 rows L-1..p+1 upwards
// (u_j = e'_j - a'_j u_{j-1}) for the same slice; they meet at the middle row p
// through a shuffle, then back-substitute outwards.  Half the sequential depth of a
// one-sided Thomas sweep (the chains are latency-bound: up to 257 dependent rows).
// The chain's inputs are independent of the recurrence, so they are fetched CD_U
// rows at a time ahead of the dependent arithmetic.  d' / e' overwrite d in place,
// c' / a' go to cp[f]; dst may alias the step input (pass 1 has consumed it).
// m = 0: real coefficients, the imaginary parts are decoupled (u.y = d.y / b).
constexpr int CD_U = 8;
struct CdRow {
  double2 d;
  double ax, cy;  // coefficients of u_{j-1}, u_{j+1}
  double2 b;      // diagonal
  double e;       // eps (viscosity)
};
SWE_DEV CdRow cd_load(int M, int m, int c, int n, int B, int b, double a, double aap,
                      const double *__restrict__ eps, const double4 *__restrict__ cft,
                      const double *__restrict__ dxs, const double *__restrict__ dds) {
  const int f = ((n - m) + c) & 1, k = cd_row(M, m, n);
  const double4 cf = cft[k];
  CdRow r;
  r.d = __ldg(reinterpret_cast<const double2 *>(f ? dds : dxs) + (size_t)k * B + b);
  r.e = __ldg(eps + k);
  const double sg = f ? -a : a;  // xi rows (f = 0) / delta rows (f = 1)
  r.ax = sg * cf.x;
  r.cy = sg * cf.y;
  r.b = make_double2(f ? 1.0 + aap * r.e : 1.0, -a * cf.z);
  return r;
}

__global__ void __launch_bounds__(128) k_cn_direct_chain(
    int M, int B, double alpha, const double *__restrict__ eps, const double *__restrict__ phibar,
    const double4 *__restrict__ cft, const double *__restrict__ r0s, double *__restrict__ dxs,
    double *__restrict__ dds, double *__restrict__ cpx, double *__restrict__ cpd, Ptr3 dst,
    double dtnu, double halfq) {
  const int nbg = (B + 15) / 16;
  const int wi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wi >= (M + 1) * 2 * nbg) return;  // whole warps leave together
  const int mc = wi / nbg, bg = wi - mc * nbg, m = mc >> 1, c = mc & 1;
  const int b = bg * 16 + (lane & 15), up = lane >> 4;  // up: the lower half of the chain
  const bool act = b < B;
  const int bb = act ? b : 0;
  const double a = alpha, aap = alpha * alpha * phibar[bb], apb = alpha * phibar[bb];
  const int L = M + 1 - m, p = L >> 1;  // middle row (local index)
  auto at = [&](int k) { return (size_t)k * B + bb; };
  auto put = [&](double *base, int k, double2 v) {
    if (act) reinterpret_cast<double2 *>(base)[at(k)] = v;
  };
  // ---- elimination towards the middle
  double2 cprev = make_double2(0.0, 0.0), dprev = cprev;  // (c', d') or (a', e') of the last row
  const int nrow = up ? L - 1 - p : p;  // rows this lane eliminates
  for (int r0 = 0; r0 < nrow; r0 += CD_U) {
    CdRow rv[CD_U];
#pragma unroll
    for (int u = 0; u < CD_U; ++u) {
      const int r = r0 + u;
      if (r >= nrow) break;
      const int j = up ? L - 1 - r : r;
      rv[u] = cd_load(M, m, c, m + j, B, bb, a, aap, eps, cft, dxs, dds);
    }
#pragma unroll
    for (int u = 0; u < CD_U; ++u) {
      const int r = r0 + u;
      if (r >= nrow) break;
      const int j = up ? L - 1 - r : r, n = m + j;
      const int f = ((n - m) + c) & 1, k = cd_row(M, m, n);
      const CdRow &w = rv[u];
      // downwards: den = b - ax c'_{j-1}, c' = cy / den; upwards: den = b - cy a'_{j+1}, a' = ax / den
      const double lo = up ? w.cy : w.ax, hi = up ? w.ax : w.cy;
      double2 cj, dj;
      if (m == 0) {
        const double den = w.b.x - lo * cprev.x;
        cj = make_double2(hi / den, 0.0);
        dj = make_double2((w.d.x - lo * dprev.x) / den, w.d.y / w.b.x);
      } else {
        const double2 den = make_double2(w.b.x - lo * cprev.x, w.b.y - lo * cprev.y);
        cj = cdiv(make_double2(hi, 0.0), den);
        dj = cdiv(make_double2(w.d.x - lo * dprev.x, w.d.y - lo * dprev.y), den);
      }
      put(f ? cpd : cpx, k, cj);
      put(f ? dds : dxs, k, dj);
      cprev = cj;
      dprev = dj;
    }
  }
  // ---- middle row p: a u_{p-1} + b u_p + c u_{p+1} = d with u_{p-1} = d' - c' u_p
  // (upper lane) and u_{p+1} = e' - a' u_p (lower lane)
  const double2 ca = make_double2(__shfl_xor_sync(0xffffffffu, cprev.x, 16),
                                  __shfl_xor_sync(0xffffffffu, cprev.y, 16));
  const double2 de = make_double2(__shfl_xor_sync(0xffffffffu, dprev.x, 16),
                                  __shfl_xor_sync(0xffffffffu, dprev.y, 16));
  double2 uu;
  {
    const CdRow w = cd_load(M, m, c, m + p, B, bb, a, aap, eps, cft, dxs, dds);
    // (c'_{p-1}, d'_{p-1}) live in the upper lane, (a'_{p+1}, e'_{p+1}) in the lower one
    const double2 cu = up ? ca : cprev, du = up ? de : dprev;
    const double2 al = up ? cprev : ca, el = up ? dprev : de;
    if (m == 0) {
      const double den = w.b.x - w.ax * cu.x - w.cy * al.x;
      uu = make_double2((w.d.x - w.ax * du.x - w.cy * el.x) / den, w.d.y / w.b.x);
    } else {
      const double2 den = make_double2(w.b.x - w.ax * cu.x - w.cy * al.x,
                                       w.b.y - w.ax * cu.y - w.cy * al.y);
      uu = cdiv(make_double2(w.d.x - w.ax * du.x - w.cy * el.x, w.d.y - w.ax * du.y - w.cy * el.y),
                den);
    }
    if (!up) {  // the upper lane writes the middle row
      const int n = m + p, f = ((n - m) + c) & 1, k = cd_row(M, m, n);
      double bh = 1.0;
      if (dtnu != 0.0) bh = 1.0 / (1.0 + dtnu * pow(w.e, halfq));
      if (act) {
        st2(dst.p[f ? 2 : 1], at(k), dtnu != 0.0 ? sc2(bh, uu) : uu);
        if (f) {
          const double2 r0 = ld2(r0s, at(k));
          const double2 ph = make_double2(r0.x - apb * uu.x, r0.y - apb * uu.y);
          st2(dst.p[0], at(k), dtnu != 0.0 ? sc2(bh, ph) : ph);
        }
      }
    }
  }
  // ---- back substitution outwards from the middle, Phi = r0 - a Pb delta, viscosity
  for (int r0 = nrow - 1; r0 >= 0; r0 -= CD_U) {
    double2 cv[CD_U], dv[CD_U], rv[CD_U];
    double ev[CD_U];
#pragma unroll
    for (int u = 0; u < CD_U; ++u) {
      const int r = r0 - u;
      if (r < 0) break;
      const int j = up ? L - 1 - r : r, n = m + j;
      const int f = ((n - m) + c) & 1, k = cd_row(M, m, n);
      cv[u] = reinterpret_cast<const double2 *>(f ? cpd : cpx)[at(k)];
      dv[u] = reinterpret_cast<const double2 *>(f ? dds : dxs)[at(k)];
      rv[u] = f ? __ldg(reinterpret_cast<const double2 *>(r0s) + at(k)) : make_double2(0.0, 0.0);
      ev[u] = __ldg(eps + k);
    }
#pragma unroll
    for (int u = 0; u < CD_U; ++u) {
      const int r = r0 - u;
      if (r < 0) break;
      const int j = up ? L - 1 - r : r, n = m + j;
      const int f = ((n - m) + c) & 1, k = cd_row(M, m, n);
      const double2 cj = cv[u], dj = dv[u];
      if (m == 0)
        uu = make_double2(dj.x - cj.x * uu.x, dj.y);
      else
        uu = make_double2(dj.x - (cj.x * uu.x - cj.y * uu.y), dj.y - (cj.x * uu.y + cj.y * uu.x));
      double bh = 1.0;
      if (dtnu != 0.0) bh = 1.0 / (1.0 + dtnu * pow(ev[u], halfq));
      if (act) {
        st2(dst.p[f ? 2 : 1], at(k), dtnu != 0.0 ? sc2(bh, uu) : uu);
        if (f) {
          const double2 ph = make_double2(rv[u].x - apb * uu.x, rv[u].y - apb * uu.y);
          st2(dst.p[0], at(k), dtnu != 0.0 ? sc2(bh, ph) : ph);
        }
      }
    }
  }
}

int cn_direct(int M, int B, Ptr3C x0, Ptr3C x1, Ptr3C x2, double s, double alpha,
              const double *eps, const double *phibar, const int2 *nb, const double4 *cf,
              int rhs_given, double *const scratch[5], Ptr3 dst, double dtnu, double halfq,
              cudaStream_t st) {
  const int K = (M + 1) * (M + 2) / 2;
  Ptr3 sc = {{scratch[0], scratch[1], scratch[2]}};
  k_cn_direct_rhs<<<nblocks((size_t)K * B), 256, 0, st>>>(K, B, x0, x1, x2, s, alpha, eps, phibar, nb, cf,
                                                 rhs_given, sc);
  SWE_LAUNCH_CHECK();
  const int n = (M + 1) * 2 * ((B + 15) / 16) * 32, nt = 128;
  k_cn_direct_chain<<<(n + nt - 1) / nt, nt, 0, st>>>(M, B, alpha, eps, phibar, cf, scratch[0],
                                                      scratch[1], scratch[2], scratch[3],
                                                      scratch[4], dst, dtnu, halfq);
  SWE_LAUNCH_CHECK();
  return OK;
}

// Speculative fused Crank-Nicolson fixed point for the fine level (batches of
// slices, M + 2 <= CF_MAXROW): one CTA = one pair of m-blocks (m, M - m), i.e.
// M + 2 rows, x CF_S slices, with Phi, xi, delta and the rhs of all its modes
// resident in shared memory.  L_C couples (m, n -+ 1) inside an m-block only, so
// the CTA runs every fixed-point iteration without leaving the SM; what it cannot
// know is when the slice converges (a max over all m).  It therefore runs a
// GUESSED number of iterations G (the last observed count), records the per-slice
// convergence maxima of EVERY iteration 1..G ([slice][iteration][6] ordered-bit
// atomics) and stores the iterate reached at each slice's target.  k_cn_decide
// then finds each slice's true first converged iteration k*: k* = G is the common
// case (done); k* < G re-runs this kernel for those slices only with target k*;
// no convergence by G leaves the slice active for the ordinary k_helm_tiled loop,
// which continues from iterate G (xi/delta in A or B by iteration parity, as
// k_helm_tiled expects).  Per-mode arithmetic is k_cn_start's and k_helm_tiled's,
// so iterates, iteration counts and results are bitwise those of the
// multi-kernel path (steppers.py:74-118, :143-152).
constexpr int CF_S = 4, CF_EPT = 3, CF_NTMAX = 352, CF_MAXROW = CF_NTMAX * CF_EPT / CF_S,
              CF_KS = 16;
// local n-1 / n+1 rows of local row r in the parity-split m-block [base, base + km)
// (the rows cor_nb points at; -1: none)
SWE_DEV void cf_nbrs(int r, int base, int km, int &lo, int &hi) {
  const int ne = (km + 1) >> 1, no = km >> 1, li = r - base;
  if (li < ne) {  // n = m + 2 li: odd rows li - 1 and li
    lo = li >= 1 ? base + ne + li - 1 : -1;
    hi = li < no ? base + ne + li : -1;
  } else {  // n = m + 1 + 2 (li - ne): even rows li - ne and li - ne + 1
    lo = base + li - ne;
    hi = li - ne + 1 < ne ? base + li - ne + 1 : -1;
  }
}
SWE_DEV bool cf_unpack(double w, int &lo, int &hi) {
  const long long p = __double_as_longlong(w);
  lo = (int)((p >> 20) & 0xfffff) - 1;
  hi = (int)(p & 0xfffff) - 1;
  return (p >> 40) != 0;
}
// MC > 0: the truncation is known at compile time (M = 256, the fine level): the
// shared-memory array strides and the thread count become constants
template <int MC>
__global__ void __launch_bounds__(CF_NTMAX, 2)
    k_cn_fused(int M_, int B, const int *__restrict__ offsets, const double4 *__restrict__ cft,
               const double *__restrict__ eps, const double *__restrict__ phibar, Ptr3C x0,
               Ptr3C x1, Ptr3C x2, double s, double alpha, Ptr3 R, int write_r, double *U0,
               double *A1, double *A2, double *B1, double *B2, const int *__restrict__ target,
               int G, unsigned long long *__restrict__ fst, double dtnu, double halfq,
               const int *__restrict__ Gp) {
  if (Gp) G = max(1, min(*Gp, G));  // device-resident guess (graph replays), capped
  extern __shared__ double2 fsm[];
  const int M = MC ? MC : M_;
  const int m1 = blockIdx.y, m2 = M - m1;  // slice groups fastest: CTAs in flight cover whole rows
  const int km1 = M + 1 - m1, km2 = m2 > m1 ? M + 1 - m2 : 0, nrow = km1 + km2;
  // shared arrays laid out for the largest CTA (M + 2 rows, as allocated)
  const int nmax = (M + 2) * CF_S, rmax = M + 2;
  const int n = nrow * CF_S, tid = threadIdx.x;
  const int NT = MC ? std::min(CF_NTMAX, (((MC + 2) * CF_S + CF_EPT - 1) / CF_EPT + 31) / 32 * 32)
                    : (int)blockDim.x;
  // xi/delta iterates ping-pong between the A and B copies (iterate k lives in A
  // when k is even, as in global memory); the rhs xi/delta rows in Q1/Q2; Phi and
  // the rhs Phi have no stencil and stay in registers (pv, q0)
  double2 *XA = fsm, *DA = XA + nmax, *XB = DA + nmax, *DB = XB + nmax, *Q1 = DB + nmax,
          *Q2 = Q1 + nmax;
  double4 *rcf = reinterpret_cast<double4 *>(Q2 + nmax);
  double *re = reinterpret_cast<double *>(rcf + rmax), *rbh = re + rmax;
  __shared__ unsigned long long sst[CF_KS][CF_S][6];
  __shared__ int tgt[CF_S];
  const int sl = tid % CF_S, b = blockIdx.x * CF_S + sl;
  if (tid < CF_S) {
    const int bb = blockIdx.x * CF_S + tid;
    tgt[tid] = bb < B ? (target ? target[bb] : G) : 0;
  }
  __syncthreads();
  const int mytgt = tgt[sl];
  int kmax = 0;
#pragma unroll
  for (int q = 0; q < CF_S; ++q) kmax = max(kmax, abs(tgt[q]));
  if (kmax == 0) return;  // no slice of this CTA needs work (uniform; recompute pass)
  if (fst)
    for (int q = tid; q < CF_KS * CF_S * 6; q += NT) (&sst[0][0][0])[q] = 0ULL;
  const int off1 = offsets[m1], off2 = km2 ? offsets[m2] : 0;
  auto grow = [&](int r) { return r < km1 ? off1 + r : off2 + r - km1; };
  for (int r = tid; r < nrow; r += NT) {
    const int k = grow(r);
    // the shared copy's .w (the m = 0 flag) also carries the row's stencil
    // neighbours (no per-element neighbour registers across the iterations)
    double4 c = cft[k];
    int l, h;
    if (r < km1) cf_nbrs(r, 0, km1, l, h);
    else cf_nbrs(r, km1, km2, l, h);
    c.w = __longlong_as_double(((long long)(c.w != 0.0) << 40) | ((long long)(l + 1) << 20) | (h + 1));
    rcf[r] = c;
    re[r] = eps[k];
    rbh[r] = dtnu != 0.0 ? 1.0 / (1.0 + dtnu * pow(eps[k], halfq)) : 1.0;  // as k_cn_finish
  }
  __syncthreads();
  // target > 0: final result at that iteration (viscosity applied, xi/delta in A,
  // as k_cn_finish would leave it); < 0: the raw iterate -target in its parity
  // buffer for the k_helm_tiled loop to continue from; 0: nothing to do
  const bool act = mytgt != 0, fin = mytgt > 0;
  const int kout = abs(mytgt);
  const double pb = act ? phibar[b] : 0.0, apb = alpha * pb, aap = alpha * alpha * pb;
  double2 pv[CF_EPT], q0[CF_EPT];
  // ---- prologue (as k_cn_start): X staged in the B copies.  The xi/delta inputs go
  // global -> shared by cp.async (no registers, all loads of a thread in flight):
  // a single input straight into XB/DB; with the Heun terms x0 -> XA/DA, x1 ->
  // Q1/Q2, x2 -> XB/DB, combined as comb() does once they have landed.
  const bool heun = x1.p[0] != nullptr;
#pragma unroll
  for (int j = 0; j < CF_EPT; ++j) {
    const int e = tid + j * NT, r = e / CF_S;
    if (e < n && act) {
      const size_t i = (size_t)grow(r) * B + b;
      if (heun) {
        cp_async16(&XA[e], x0.p[1] + 2 * i, true);
        cp_async16(&DA[e], x0.p[2] + 2 * i, true);
        cp_async16(&Q1[e], x1.p[1] + 2 * i, true);
        cp_async16(&Q2[e], x1.p[2] + 2 * i, true);
        cp_async16(&XB[e], x2.p[1] + 2 * i, true);
        cp_async16(&DB[e], x2.p[2] + 2 * i, true);
      } else {
        cp_async16(&XB[e], x0.p[1] + 2 * i, true);
        cp_async16(&DB[e], x0.p[2] + 2 * i, true);
      }
      pv[j] = comb(x0, x1, x2, s, 0, i);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  if (heun) {
    double2 cx[CF_EPT], cd[CF_EPT];
#pragma unroll
    for (int j = 0; j < CF_EPT; ++j) {
      const int e = tid + j * NT;
      if (e < n && act) {
        const double2 ax = Q1[e], bx = XB[e], ad = Q2[e], bd = DB[e];
        cx[j] = add2(XA[e], sc2(s, make_double2(ax.x + bx.x, ax.y + bx.y)));
        cd[j] = add2(DA[e], sc2(s, make_double2(ad.x + bd.x, ad.y + bd.y)));
      }
    }
#pragma unroll
    for (int j = 0; j < CF_EPT; ++j) {
      const int e = tid + j * NT;
      if (e < n && act) {  // own elements only: no barrier needed between
        XB[e] = cx[j];
        DB[e] = cd[j];
      }
    }
    __syncthreads();
  }
  // rhs R = X + alpha (L_G X + L_C X), then the first iterate helm(R) into A
#pragma unroll
  for (int j = 0; j < CF_EPT; ++j) {
    const int e = tid + j * NT, r = e / CF_S;
    if (e < n && act) {
      const double2 ph = pv[j], xi = XB[e], de = DB[e];
      const double e_ = re[r];
      const double4 cf = rcf[r];
      int lo, hi;
      const bool m0 = cf_unpack(cf.w, lo, hi);
      double2 xl = make_double2(0.0, 0.0), dl = xl, xh = xl, dh = xl;
      if (lo >= 0) {
        xl = XB[lo * CF_S + sl];
        dl = DB[lo * CF_S + sl];
      }
      if (hi >= 0) {
        xh = XB[hi * CF_S + sl];
        dh = DB[hi * CF_S + sl];
      }
      double2 lx = make_double2(-(cf.x * dl.x + cf.y * dh.x + cf.z * xi.y),
                                -(cf.x * dl.y + cf.y * dh.y - cf.z * xi.x));
      double2 lc = make_double2(cf.x * xl.x + cf.y * xh.x - cf.z * de.y,
                                cf.x * xl.y + cf.y * xh.y + cf.z * de.x);
      if (m0) {
        lx.y = 0.0;
        lc.y = 0.0;
      }
      const double2 lphi = make_double2(-pb * de.x, -pb * de.y);
      const double2 lde = add2(sc2(e_, ph), lc);
      const double2 r0 = add2(ph, sc2(alpha, lphi)), r1 = add2(xi, sc2(alpha, lx)),
                    r2 = add2(de, sc2(alpha, lde));
      q0[j] = r0;
      Q1[e] = r1;
      Q2[e] = r2;
      if (write_r && mytgt < 0) {  // rhs only for slices the tiled loop continues
        const size_t i = (size_t)grow(r) * B + b;
        st2(R.p[0], i, r0);
        st2(R.p[1], i, r1);
        st2(R.p[2], i, r2);
      }
      const double apb_ = alpha * pb, denom = 1.0 + alpha * alpha * pb * e_;
      const double rdn = 1.0 / denom;  // divisions as ddiv_r
      const double2 nph = make_double2(ddiv_r(r0.x - apb_ * r2.x, denom, rdn),
                                       ddiv_r(r0.y - apb_ * r2.y, denom, rdn));
      const double ae = alpha * e_;
      pv[j] = nph;
      XA[e] = r1;
      DA[e] = make_double2(r2.x + ae * nph.x, r2.y + ae * nph.y);
    }
  }
  __syncthreads();
  // ---- fixed-point iterations 1..kmax (as k_helm_tiled), one barrier each
  const int lane = tid & 31;
  for (int it = 1; it <= kmax; ++it) {
    const double2 *X = (it & 1) ? XA : XB, *D = (it & 1) ? DA : DB;
    double2 *NX = (it & 1) ? XB : XA, *ND = (it & 1) ? DB : DA;
    const bool out = it == kout;
    unsigned long long mx[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < CF_EPT; ++j) {
      const int e = tid + j * NT, r = e / CF_S;
      if (e < n && act) {
        const double2 rp = q0[j], r1 = Q1[e], r2 = Q2[e], o0 = pv[j];
        const double e_ = re[r];
        const double4 cf = rcf[r];
        int lo, hi;
        const bool m0 = cf_unpack(cf.w, lo, hi);
        const double2 x = X[e], d = D[e];
        double2 xl = make_double2(0.0, 0.0), dl = xl, xh = xl, dh = xl;
        if (lo >= 0) {
          xl = X[lo * CF_S + sl];
          dl = D[lo * CF_S + sl];
        }
        if (hi >= 0) {
          xh = X[hi * CF_S + sl];
          dh = D[hi * CF_S + sl];
        }
        double2 lx = make_double2(-(cf.x * dl.x + cf.y * dh.x + cf.z * x.y),
                                  -(cf.x * dl.y + cf.y * dh.y - cf.z * x.x));
        double2 lc = make_double2(cf.x * xl.x + cf.y * xh.x - cf.z * d.y,
                                  cf.x * xl.y + cf.y * xh.y + cf.z * d.x);
        if (m0) {
          lx.y = 0.0;
          lc.y = 0.0;
        }
        const double2 rx = add2(r1, sc2(alpha, lx)), rd = add2(r2, sc2(alpha, lc));
        const double denom = 1.0 + aap * e_;
        const double rdn = 1.0 / denom;  // recomputed (fewer live registers): the prologue's bits
        const double2 ph = make_double2(ddiv_r(rp.x - apb * rd.x, denom, rdn),
                                        ddiv_r(rp.y - apb * rd.y, denom, rdn));
        const double ae = alpha * e_;
        const double2 de = make_double2(rd.x + ae * ph.x, rd.y + ae * ph.y);
        mx[0] = max(mx[0], sqmag_bits(ph.x, ph.y));
        mx[1] = max(mx[1], sqmag_bits(rx.x, rx.y));
        mx[2] = max(mx[2], sqmag_bits(de.x, de.y));
        mx[3] = max(mx[3], sqmag_bits(ph.x - o0.x, ph.y - o0.y));
        mx[4] = max(mx[4], sqmag_bits(rx.x - x.x, rx.y - x.y));
        mx[5] = max(mx[5], sqmag_bits(de.x - d.x, de.y - d.y));
        pv[j] = ph;
        NX[e] = rx;
        ND[e] = de;
        if (out) {
          const size_t i = (size_t)grow(r) * B + b;
          if (!fin) {
            st2(U0, i, ph);
            st2((it & 1) ? B1 : A1, i, rx);
            st2((it & 1) ? B2 : A2, i, de);
          } else if (dtnu != 0.0) {
            const double bh = rbh[r];
            st2(U0, i, sc2(bh, ph));
            st2(A1, i, sc2(bh, rx));
            st2(A2, i, sc2(bh, de));
          } else {
            st2(U0, i, ph);
            st2(A1, i, rx);
            st2(A2, i, de);
          }
        }
      }
      asm volatile("" ::: "memory");  // one element's loads in flight at a time (registers)
    }
    // per-slice maxima: the 8 lanes of one slice differ in bits 2..4.  Reduce-scatter
    // over those bits (each step keeps the half of the maxima selected by the lane
    // bit and sends the other half: 4 + 2 + 1 exchanges instead of 6 x 3), then the
    // lane holding maximum q of slice sl adds it: one shared atomic per warp
    if (fst && it <= CF_KS) {
      const bool b2 = lane & 4, b3 = lane & 8, b4 = lane & 16;
      unsigned long long a4[4], a2[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const unsigned long long h = i + 4 < 6 ? mx[i + 4] : 0ULL;
        a4[i] = max(b2 ? h : mx[i], __shfl_xor_sync(0xffffffffu, b2 ? mx[i] : h, 4));
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
        a2[i] = max(b3 ? a4[i + 2] : a4[i], __shfl_xor_sync(0xffffffffu, b3 ? a4[i] : a4[i + 2], 8));
      const unsigned long long v =
          max(b4 ? a2[1] : a2[0], __shfl_xor_sync(0xffffffffu, b4 ? a2[0] : a2[1], 16));
      const int q = (b2 ? 4 : 0) + (b3 ? 2 : 0) + (b4 ? 1 : 0);
      if (q < 6 && v) atomicMax(&sst[it - 1][lane & 3][q], v);
    }
    __syncthreads();
  }
  if (fst) {
    const int nk = min(kmax, CF_KS);
    for (int q = tid; q < nk * CF_S * 6; q += NT) {
      const int it = q / (CF_S * 6), ss = (q / 6) % CF_S, f = q % 6;
      const int bb = blockIdx.x * CF_S + ss;
      const unsigned long long v = sst[it][ss][f];
      if (bb < B && tgt[ss] != 0 && v) atomicMax(fst + ((size_t)bb * CF_KS + it) * 6 + f, v);
    }
  }
}

int cn_fused_ok(int M, int B) { return M + 2 <= CF_MAXROW && B >= 1; }  // M <= 262
int cn_fused_kmax() { return CF_KS; }

int cn_fused(int M, int B, const int *offsets, const double4 *cf, const double *eps,
             const double *phibar, Ptr3C x0, Ptr3C x1, Ptr3C x2, double s, double alpha,
             Ptr3 R, int write_r, double *U0, double *A1, double *A2, double *B1, double *B2,
             const int *target, int G, unsigned long long *fst, double dtnu, double halfq,
             cudaStream_t st, const int *Gp) {
  const int nrow = M + 2, n = nrow * CF_S;
  const int NT = std::min(CF_NTMAX, ((n + CF_EPT - 1) / CF_EPT + 31) / 32 * 32);
  const int smem = 6 * n * (int)sizeof(double2) + nrow * (int)(sizeof(double4) + 2 * sizeof(double));
  dim3 grid((B + CF_S - 1) / CF_S, M / 2 + 1);
  if (M == 256) {
    static int attr = 0;
    if (smem > attr) {
      SWE_CUDA(cudaFuncSetAttribute(k_cn_fused<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem));
      attr = smem;
    }
    k_cn_fused<256><<<grid, NT, smem, st>>>(M, B, offsets, cf, eps, phibar, x0, x1, x2, s, alpha, R,
                                            write_r, U0, A1, A2, B1, B2, target, G, fst, dtnu,
                                            halfq, Gp);
  } else {
    static int attr = 0;
    if (smem > attr) {
      SWE_CUDA(cudaFuncSetAttribute(k_cn_fused<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attr = smem;
    }
    k_cn_fused<0><<<grid, NT, smem, st>>>(M, B, offsets, cf, eps, phibar, x0, x1, x2, s, alpha, R,
                                          write_r, U0, A1, A2, B1, B2, target, G, fst, dtnu, halfq,
                                          Gp);
  }
  SWE_LAUNCH_CHECK();
  return OK;
}

// Per-slice decision after k_cn_fused (one block): first converged iteration k*
// of each slice from the recorded maxima (decide_slice's test, steppers.py:100-112),
// k* < G -> target2 = k* (recompute pass), none -> still active after G
// iterations.  Sets counter = active slices, loop = G and, in a graph, the WHILE
// node's condition; zeroes the maxima for the next call.
SWE_DEV bool cf_converged(const unsigned long long *q6, double tol) {
  double v[6];
  for (int q = 0; q < 6; ++q) v[q] = sqrt(__longlong_as_double((long long)q6[q]));
  double overall = fmax(fmax(v[0], v[1]), v[2]);
  if (isnan(v[0]) || isnan(v[1]) || isnan(v[2])) overall = nan("");
  overall = (overall > 1e-300 || isnan(overall)) ? overall : 1e-300;
  for (int f = 0; f < 3; ++f) {
    const double tiny = 1e-13 * overall;
    const double scale = (v[f] >= tiny || isnan(v[f])) ? v[f] : tiny;
    if (v[3 + f] > tol * scale) return false;
  }
  return true;
}
__global__ void k_cn_decide(int B, int G, unsigned long long *fst, int *flags, int *iters,
                            int *target2, int *counter, int *loop, double tol,
                            cudaGraphConditionalHandle h, int has_h, int max_iter, int *Gp) {
  __shared__ int cnt, kmx;
  const int Gcap = G;
  if (Gp) G = max(1, min(*Gp, G));  // the guess the first fused pass ran with
  if (threadIdx.x == 0) cnt = kmx = 0;
  __syncthreads();
  // a 16-lane group per slice: lane k tests iteration k + 1 (independent loads instead of
  // one thread's dependent chain over the iterations), the first converged one by ballot
  static_assert(CF_KS == 16, "one half-warp lane per recorded iteration");
  const int lane = threadIdx.x & 31, k = lane & 15, sh = lane & 16;
  int mine = 0, kmine = 0;
  for (int b0 = 0; b0 < B; b0 += blockDim.x / 16) {  // (uniform trip count: ballots below)
    const int b = b0 + threadIdx.x / 16;
    const bool live = b < B;
    unsigned long long *q = fst + (size_t)(live ? b : 0) * CF_KS * 6;
    const bool conv = live && k < G && cf_converged(q + k * 6, tol);
    const unsigned m = (__ballot_sync(0xffffffffu, conv) >> sh) & 0xffffu;
    if (live && k < G)
      for (int f = 0; f < 6; ++f) q[k * 6 + f] = 0ULL;
    if (live && k == 0) {
      const int ks = m ? __ffs(m) : 0;
      if (ks) {
        kmine = max(kmine, ks);
        flags[b] = 0;
        iters[b] = ks;
        target2[b] = ks < G ? ks : 0;  // recompute the final result at k*
      } else {
        flags[b] = 1;
        iters[b] = G;
        target2[b] = -G;  // pass 1 stored a final result: recompute the raw iterate G
        ++mine;
      }
    }
  }
  if (mine) atomicAdd(&cnt, mine);
  if (kmine) atomicMax(&kmx, kmine);
  __syncthreads();
  if (threadIdx.x == 0) {
    *counter = cnt;
    *loop = G;
    // next solve's guess: the largest first-converged iteration, or one more than
    // this guess while slices still continue past it (as the host path's iter_guess)
    if (Gp) *Gp = cnt ? min(Gcap, G + 1) : max(1, kmx);
    if (has_h) cudaGraphSetConditional(h, (cnt > 0 && G < max_iter) ? 1u : 0u);
  }
}

int cn_decide(int B, int G, unsigned long long *fst, int *flags, int *iters, int *target2,
              int *counter, int *loop, double tol, const cudaGraphConditionalHandle *h,
              int max_iter, cudaStream_t st, int *Gp) {
  k_cn_decide<<<1, 1024, 0, st>>>(B, G, fst, flags, iters, target2, counter, loop, tol,
                                  h ? *h : cudaGraphConditionalHandle(0), h != nullptr, max_iter, Gp);
  SWE_LAUNCH_CHECK();
  return OK;
}

// Fixed-point epilogue: slices whose iterate ended in the B buffers (odd iteration
// count) copy xi/delta back to A = u[1], u[2]; with dtnu != 0 the viscosity
// factor (dynamics.py:191-200) is applied to every slice on the way.
__global__ void k_cn_finish(int K, int B, Ptr3 u, const double *b1, const double *b2,
                            const int *iters, const double *nn1a2, double dtnu, double halfq,
                            const int *counter, int *fail, const int *skip) {
  if (fail && blockIdx.x == 0 && threadIdx.x == 0 && *counter > 0) *fail = 1;
  if (skip) {  // the common case: k_cn_fused finished every slice, nothing to do
    int todo = 0;
    for (int b = threadIdx.x; b < B; b += blockDim.x) todo |= skip[b] < 0;
    if (!__syncthreads_or(todo)) return;
  }
  FOR_KB(K, B) {
    const int k = (int)(_i / B), b = (int)(_i - (size_t)k * B);
    if (skip && skip[b] >= 0) continue;  // finished by k_cn_fused
    const bool odd = iters && (iters[b] & 1);
    if (dtnu != 0.0) {
      const double bh = 1.0 / (1.0 + dtnu * pow(nn1a2[k], halfq));
      st2(u.p[0], _i, sc2(bh, ld2(u.p[0], _i)));
      st2(u.p[1], _i, sc2(bh, ld2(odd ? b1 : u.p[1], _i)));
      st2(u.p[2], _i, sc2(bh, ld2(odd ? b2 : u.p[2], _i)));
    } else if (odd) {
      st2(u.p[1], _i, ld2(b1, _i));
      st2(u.p[2], _i, ld2(b2, _i));
    }
  }
}

// CUDA-graph fixed point: WHILE-node condition after each iteration (the host
// loop's `active > 0 && it < max_iter`, steppers.py:96-112, evaluated on device)
__global__ void k_loop_cond(cudaGraphConditionalHandle h, const int *counter, int *loop,
                            int max_iter) {
  const int it = ++*loop;
  cudaGraphSetConditional(h, (*counter > 0 && it < max_iter) ? 1u : 0u);
}

// per-slice convergence decision (steppers.py:100-112); resets stats
__global__ void k_decide(int B, double *stats, int *active, int *iters, int *counter, double tol) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (decide_slice(b, stats, active, iters, tol)) atomicAdd(counter, 1);
}

__global__ void k_fill_int(int *p, int n, int v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// y = a + s*(x1 (+ x2)) for three fields (add_tendency, dynamics.py:58-63)
__global__ void k_axpy3(int n, Ptr3C a, Ptr3C x1, Ptr3C x2, double s, Ptr3 y) {
  FOR_KB(n, 1) {
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      double2 t = ld2(x1.p[f], _i);
      if (x2.p[f]) t = add2(t, ld2(x2.p[f], _i));
      st2(y.p[f], _i, add2(ld2(a.p[f], _i), sc2(s, t)));
    }
  }
}

// d = curl - lap(ke) (dynamics.py:151), optionally + L_C (explicit Coriolis)
__global__ void k_tend_finish(int K, int B, double *kd, const double *ke, const double *lap,
                              double *kx, const double *lcx, const double *lcd) {
  FOR_KB(K, B) {
    const int k = (int)(_i / B);
    const double2 ke2 = ld2(ke, _i);
    const double l = lap[k];
    double2 d = ld2(kd, _i);
    d = make_double2(d.x - ke2.x * l, d.y - ke2.y * l);
    if (lcd) {
      d = add2(d, ld2(lcd, _i));
      st2(kx, _i, add2(ld2(kx, _i), ld2(lcx, _i)));
    }
    st2(kd, _i, d);
  }
}

// backward-Euler damping b(n) (dynamics.py:181-200), in place on three fields
__global__ void k_visc(int K, int B, Ptr3 u, const double *nn1a2, double dtnu, double halfq) {
  FOR_KB(K, B) {
    const int k = (int)(_i / B);
    const double bh = 1.0 / (1.0 + dtnu * pow(nn1a2[k], halfq));
#pragma unroll
    for (int f = 0; f < 3; ++f) st2(u.p[f], _i, sc2(bh, ld2(u.p[f], _i)));
  }
}

__global__ void k_copy3(int n, Ptr3C a, Ptr3 y) {
  FOR_KB(n, 1) {
#pragma unroll
    for (int f = 0; f < 3; ++f) st2(y.p[f], _i, ld2(a.p[f], _i));
  }
}

__global__ void k_phi0(int B, const double *phibar, double *pb, double *phi0) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) {
    pb[b] = phibar[b];
    // phi_prime subtracts phibar*SQRT2 from mode (0,0) (dynamics.py:20, :52-56);
    // its synthesis is that times P_00 = 1/sqrt(2) at every latitude
    phi0[b] = (phibar[b] * 1.4142135623730951) * (1.0 / sqrt(2.0));
  }
}

// residual |u - alpha*(L_G + L_C) u - rhs| per slice (steppers.py:113-118)
__global__ void k_resid(int K, int B, Ptr3C u, Ptr3C rhs, const double *lcx, const double *lcd,
                        double alpha, const double *eps, const double *phibar, double *res) {
  FOR_KB(K, B) {
    const int k = (int)(_i / B), b = (int)(_i - (size_t)k * B);
    const double2 ph = ld2(u.p[0], _i), xi = ld2(u.p[1], _i), de = ld2(u.p[2], _i);
    const double pb = phibar[b];
    const double2 lph = make_double2(-pb * de.x, -pb * de.y);
    const double2 lxi = ld2(lcx, _i);
    const double2 lde = add2(sc2(eps[k], ph), ld2(lcd, _i));
    double r = 0.0;
    const double2 v[3] = {ph, xi, de}, l[3] = {lph, lxi, lde};
    for (int f = 0; f < 3; ++f) {
      const double2 rr = ld2(rhs.p[f], _i);
      r = fmax(r, hypot(v[f].x - alpha * l[f].x - rr.x, v[f].y - alpha * l[f].y - rr.y));
    }
    atomic_max_nonneg(res + b, r);
  }
}

// boundary-layout state stats: max|c| over 3 fields and finiteness (dynamics.py:65-71)
__global__ void k_state_stats(const double2 *__restrict__ s, int B, int K, double *maxabs,
                              int *finite) {
  const int b = blockIdx.y;
  double mx = 0.0;
  int fin = 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 3 * K; i += gridDim.x * blockDim.x) {
    const double2 v = s[(size_t)b * 3 * K + i];
    if (!isfinite(v.x) || !isfinite(v.y)) fin = 0;
    const double h = hypot(v.x, v.y);
    mx = (isnan(h) || isnan(mx)) ? nan("") : fmax(mx, h);
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double w = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = (isnan(w) || isnan(mx)) ? nan("") : fmax(mx, w);
    fin &= __shfl_xor_sync(0xffffffffu, fin, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(maxabs + b, mx);
    if (!fin) atomicAnd(finite + b, 0);
  }
}

// truncate_pad (spharm.py:352-368): [nb][Ks] -> [nb][Kd]
__global__ void k_truncate(const double2 *__restrict__ src, double2 *__restrict__ dst, int nb,
                           int Ms, int Md, const int *offs_s, const int *offs_d) {
  const int Kd = (Md + 1) * (Md + 2) / 2, Ks = (Ms + 1) * (Ms + 2) / 2;
  const int mm = min(Ms, Md);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < (size_t)nb * Kd;
       i += (size_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / Kd), k = (int)(i - (size_t)b * Kd);
    // locate (m, n) of destination mode k
    int lo = 0, hi = Md;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (offs_d[mid] <= k) lo = mid; else hi = mid - 1;
    }
    const int m = lo, n = m + (k - offs_d[m]);
    double2 v = make_double2(0.0, 0.0);
    if (m <= mm && n <= mm) v = src[(size_t)b * Ks + offs_s[m] + (n - m)];
    dst[i] = v;
  }
}

// ---- host wrappers -----------------------------------------------------------
int lin_rhs(int K, int B, const double *const U[3], const double *lcx, const double *lcd,
            double alpha, const double *eps, const double *phibar, double *const R[3],
            cudaStream_t st) {
  k_lin_rhs<<<nblocks((size_t)K * B), 256, 0, st>>>(K, B, U[0], U[1], U[2], lcx, lcd, alpha, eps,
                                                    phibar, R[0], R[1], R[2]);
  SWE_LAUNCH_CHECK();
  return OK;
}

int lin_tend(int K, int B, const double *U0, const double *U2, const double *lcx,
             const double *lcd, const double *eps, const double *phibar, double *const T[3],
             cudaStream_t st) {
  k_lin_tend<<<nblocks((size_t)K * B), 256, 0, st>>>(K, B, U0, U2, lcx, lcd, eps, phibar, T[0],
                                                     T[1], T[2]);
  SWE_LAUNCH_CHECK();
  return OK;
}

int coriolis_spec(int K, int B, const CorOp &c, double *lcx, double *lcd, cudaStream_t st) {
  k_coriolis<<<nblocks((size_t)K * B), 256, 0, st>>>(K, B, c, lcx, lcd);
  SWE_LAUNCH_CHECK();
  return OK;
}

int helm(int K, int B, const double *const R[3], const double *lcx, const double *lcd,
         double alpha, const double *eps, const double *phibar, double *const U[3],
         const int *active, double *stats, cudaStream_t st, const CorOp *cor, int *iters,
         int *counter, double tol, unsigned *hdone) {
  int bx = 1;
  while (bx < B && bx < 32) bx <<= 1;
  // rows per block: at least a warp, at most 256 threads, and small enough that
  // small problems still spread over >= 2 blocks per SM
  int by = 256 / bx;
  while (by > 32 / bx && by > 1 && (size_t)((K + by - 1) / by) * ((B + bx - 1) / bx) < 296) by >>= 1;
  const int gx = (B + bx - 1) / bx;
  const int ybl = std::max(1, std::min((K + by - 1) / by, (148 * 8) / gx));
  dim3 grid(gx, ybl), blk(bx, by);
  CorOp c = cor ? *cor : CorOp{nullptr, nullptr, nullptr, nullptr};
  if (cor)
    k_helm<1><<<grid, blk, 0, st>>>(K, B, R[0], R[1], R[2], lcx, lcd, alpha, eps, phibar, U[0],
                                     U[1], U[2], active, stats, c, iters, counter, tol, hdone);
  else
    k_helm<4><<<grid, blk, 0, st>>>(K, B, R[0], R[1], R[2], lcx, lcd, alpha, eps, phibar, U[0],
                                     U[1], U[2], active, stats, c, iters, counter, tol, hdone);
  SWE_LAUNCH_CHECK();
  return OK;
}

int cn_start(int K, int B, Ptr3C x0, Ptr3C x1, Ptr3C x2, double s, double alpha,
             const double *eps, const double *phibar, const CorOp &c, Ptr3 R, Ptr3 dst,
             cudaStream_t st) {
  k_cn_start<<<nblocks((size_t)K * B), 256, 0, st>>>(K, B, x0, x1, x2, s, alpha, eps, phibar, c,
                                                     R, dst);
  SWE_LAUNCH_CHECK();
  return OK;
}

int cn_finish(int K, int B, Ptr3 u, const double *b1, const double *b2, const int *iters,
              const double *nn1a2, double dtnu, double halfq, cudaStream_t st,
              const int *counter, int *fail, const int *skip) {
  k_cn_finish<<<nblocks((size_t)K * B), 256, 0, st>>>(K, B, u, b1, b2, iters, nn1a2, dtnu, halfq,
                                                      counter, fail, skip);
  SWE_LAUNCH_CHECK();
  return OK;
}

int loop_cond(cudaGraphConditionalHandle h, const int *counter, int *loop, int max_iter,
              cudaStream_t st) {
  k_loop_cond<<<1, 1, 0, st>>>(h, counter, loop, max_iter);
  SWE_LAUNCH_CHECK();
  return OK;
}

// y[k] += g[k][col] for one batch-1 spectral field set (3 fields, [K][2]) from a
// batch-n set ([K][2n]) (serial coarse sweep forcing)
// one point of the serial sweep (B = 1): y += g[:, col] (when g is given, as
// add_col) and the result stored to dst in the boundary layout (as to_boundary):
// one launch per point instead of two
__global__ void k_sweep_point(int K, int n, int col, Ptr3 y, Ptr3C g, double2 *__restrict__ dst,
                              const int *__restrict__ perm) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x) {
    const int r = perm[k];
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      double2 a = ld2(y.p[f], r);
      if (g.p[0]) {
        a = add2(a, ld2(g.p[f], (size_t)r * n + col));
        st2(y.p[f], r, a);
      }
      dst[(size_t)f * K + k] = a;
    }
  }
}

int sweep_point(int K, int n, int col, Ptr3 y, Ptr3C g, double *dst, const int *perm,
                cudaStream_t st) {
  k_sweep_point<<<(K + 255) / 256, 256, 0, st>>>(K, n, col, y, g, reinterpret_cast<double2 *>(dst),
                                                 perm);
  SWE_LAUNCH_CHECK();
  return OK;
}

// copy the active count and the iteration counts to mapped host memory
__global__ void k_publish(int B, const int *counter, const int *iters, volatile int *pub) {
  for (int i = threadIdx.x; i <= B; i += blockDim.x) pub[i] = i == 0 ? *counter : iters[i - 1];
}

int publish(int B, const int *counter, const int *iters, int *pub, cudaStream_t st) {
  k_publish<<<1, 256, 0, st>>>(B, counter, iters, pub);
  SWE_LAUNCH_CHECK();
  return OK;
}

int decide(int B, double *stats, int *active, int *iters, int *counter, double tol,
           cudaStream_t st) {
  k_decide<<<(B + 127) / 128, 128, 0, st>>>(B, stats, active, iters, counter, tol);
  SWE_LAUNCH_CHECK();
  return OK;
}

int fill_int(int *p, int n, int v, cudaStream_t st) {
  k_fill_int<<<(n + 255) / 256, 256, 0, st>>>(p, n, v);
  SWE_LAUNCH_CHECK();
  return OK;
}

int axpy3(size_t n, Ptr3C a, Ptr3C x1, Ptr3C x2, double s, Ptr3 y, cudaStream_t st) {
  k_axpy3<<<nblocks(n), 256, 0, st>>>((int)n, a, x1, x2, s, y);
  SWE_LAUNCH_CHECK();
  return OK;
}

// k_tend_finish of K1 fused with the Heun midpoint MID = U* + s K1 (k_axpy3): the
// same two expressions, one pass
__global__ void k_finish_axpy(int K, int B, double *kd, const double *ke, const double *lap,
                              Ptr3C us, Ptr3C k1, double s, Ptr3 mid) {
  FOR_KB(K, B) {
    const int k = (int)(_i / B);
    const double2 ke2 = ld2(ke, _i);
    const double l = lap[k];
    double2 d = ld2(kd, _i);
    d = make_double2(d.x - ke2.x * l, d.y - ke2.y * l);
    st2(kd, _i, d);
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      const double2 t = f == 2 ? d : ld2(k1.p[f], _i);
      st2(mid.p[f], _i, add2(ld2(us.p[f], _i), sc2(s, t)));
    }
  }
}

int finish_axpy(int K, int B, double *kd, const double *ke, const double *lap, Ptr3C us, Ptr3C k1,
                double s, Ptr3 mid, cudaStream_t st) {
  k_finish_axpy<<<nblocks((size_t)K * B), 256, 0, st>>>(K, B, kd, ke, lap, us, k1, s, mid);
  SWE_LAUNCH_CHECK();
  return OK;
}

int tend_finish(int K, int B, double *kd, const double *ke, const double *lap, double *kx,
                const double *lcx, const double *lcd, cudaStream_t st) {
  k_tend_finish<<<nblocks((size_t)K * B), 256, 0, st>>>(K, B, kd, ke, lap, kx, lcx, lcd);
  SWE_LAUNCH_CHECK();
  return OK;
}

int visc(int K, int B, Ptr3 u, const double *nn1a2, double dtnu, double halfq, cudaStream_t st) {
  k_visc<<<nblocks((size_t)K * B), 256, 0, st>>>(K, B, u, nn1a2, dtnu, halfq);
  SWE_LAUNCH_CHECK();
  return OK;
}

int copy3(size_t n, Ptr3C a, Ptr3 y, cudaStream_t st) {
  k_copy3<<<nblocks(n), 256, 0, st>>>((int)n, a, y);
  SWE_LAUNCH_CHECK();
  return OK;
}

int set_phibar(int B, const double *phibar, double *pb, double *phi0, cudaStream_t st) {
  k_phi0<<<(B + 127) / 128, 128, 0, st>>>(B, phibar, pb, phi0);
  SWE_LAUNCH_CHECK();
  return OK;
}

int resid(int K, int B, Ptr3C u, Ptr3C rhs, const double *lcx, const double *lcd, double alpha,
          const double *eps, const double *phibar, double *res, cudaStream_t st) {
  k_resid<<<nblocks((size_t)K * B), 256, 0, st>>>(K, B, u, rhs, lcx, lcd, alpha, eps, phibar, res);
  SWE_LAUNCH_CHECK();
  return OK;
}

int state_stats(const double *s, int B, int K, double *maxabs, int *finite, cudaStream_t st) {
  SWE_CUDA(cudaMemsetAsync(maxabs, 0, sizeof(double) * B, st));
  k_fill_int<<<(B + 255) / 256, 256, 0, st>>>(finite, B, 1);
  dim3 grid(std::max(1, std::min(64, (3 * K + 255) / 256)), B);
  k_state_stats<<<grid, 256, 0, st>>>(reinterpret_cast<const double2 *>(s), B, K, maxabs, finite);
  SWE_LAUNCH_CHECK();
  return OK;
}

int truncate_pad(const double *src, double *dst, int nb, int Ms, int Md, const int *offs_s,
                 const int *offs_d, cudaStream_t st) {
  const size_t n = (size_t)nb * (Md + 1) * (Md + 2) / 2;
  k_truncate<<<nblocks(n), 256, 0, st>>>(reinterpret_cast<const double2 *>(src),
                                        reinterpret_cast<double2 *>(dst), nb, Ms, Md, offs_s,
                                        offs_d);
  SWE_LAUNCH_CHECK();
  return OK;
}

}  // namespace swe
