// Plan creation: Gaussian grid (host), Legendre tables (device), FFT plan.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>

#include "plan.cuh"

#include <cudaTypedefs.h>
#include "spectral.cuh"

namespace swe {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
const char *last_error() { return g_err; }

int cuda_fail(cudaError_t e, const char *what, const char *file, int line) {
  set_error("CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e), cudaGetErrorString(e), file,
            line, what);
  return E_CUDA;
}

// Gauss-Legendre nodes (decreasing) and weights; same Newton scheme and
// operation order as gauss_legendre (spharm.py:75-108), all nodes iterated
// together until every node has converged.
static int gauss_legendre(int n, std::vector<double> &x, std::vector<double> &w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  std::vector<double> pp(n, 0.0), pn(n), pnm1(n);
  for (int k = 0; k < n; ++k) x[k] = cos(M_PI * (k + 0.75) / (n + 0.5));
  bool done = false;
  for (int it = 0; it < 100 && !done; ++it) {
    done = true;
    for (int k = 0; k < n; ++k) {
      double p0 = 1.0, p1 = x[k];
      for (int j = 2; j <= n; ++j) {
        const double p2 = ((double)(2 * j - 1) * x[k] * p1 - (double)(j - 1) * p0) / (double)j;
        p0 = p1;
        p1 = p2;
      }
      pn[k] = p1;
      pnm1[k] = p0;
    }
    for (int k = 0; k < n; ++k) {
      pp[k] = (double)n * (x[k] * pn[k] - pnm1[k]) / (x[k] * x[k] - 1.0);
      const double dx = pn[k] / pp[k];
      x[k] = x[k] - dx;
      if (!(fabs(dx) <= 1e-15 * std::max(1.0, fabs(x[k])))) done = false;
    }
  }
  if (!done) {
    set_error("Gauss-Legendre Newton iteration did not converge for n=%d", n);
    return E_SHAPE;
  }
  std::vector<int> order(n);
  for (int k = 0; k < n; ++k) order[k] = k;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return x[a] > x[b]; });
  std::vector<double> xs(n), ws(n);
  for (int k = 0; k < n; ++k) {
    const int o = order[k];
    xs[k] = x[o];
    ws[k] = 2.0 / ((1.0 - x[o] * x[o]) * pp[o] * pp[o]);
  }
  x.swap(xs);
  w.swap(ws);
  return OK;
}

__device__ __forceinline__ double eps_mn(int m, int n) {
  if (n <= m) return 0.0;
  const double nn = (double)n * n - (double)m * m;
  return __dsqrt_rn(__ddiv_rn(nn, 4.0 * (double)n * n - 1.0));
}

// One thread per (order m, latitude pair p): P_mm by the diagonal recurrence,
// then the three-term recurrence in n (spharm.py:118-143) and
// H_mn = -n eps_{m,n+1} P_{m,n+1} + (n+1) eps_{mn} P_{m,n-1} (spharm.py:179-187).
// Explicit _rn intrinsics keep the reference's rounding (no FMA contraction).
__global__ void table_kernel(int M, int Jh, int Jp, const double *mu, const int *offsets,
                             double *P, double *H) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int m = blockIdx.y;
  if (p >= Jp) return;
  const int km = M + 1 - m, ne = (km + 1) >> 1;
  const int off = offsets[m];
  auto row = [&](int n) -> size_t {
    const int d = n - m;
    return (size_t)off + ((d & 1) ? ne + (d >> 1) : (d >> 1));
  };
  if (p >= Jh) {
    for (int n = m; n <= M; ++n) {
      P[row(n) * Jp + p] = 0.0;
      H[row(n) * Jp + p] = 0.0;
    }
    return;
  }
  const double x = mu[p];
  const double ct = __dsqrt_rn(fmax(__dsub_rn(1.0, __dmul_rn(x, x)), 0.0));
  double pmm = 1.0 / sqrt(2.0);
  for (int k = 1; k <= m; ++k)
    pmm = __dmul_rn(__dmul_rn(pmm, ct), __dsqrt_rn(__ddiv_rn(2.0 * k + 1.0, 2.0 * k)));
  // rolling window P_{n-1}, P_n, P_{n+1}
  double pm1 = 0.0;  // P_{m,n-1}
  double p0 = pmm;   // P_{m,n}
  double p1 = __dmul_rn(__dmul_rn(__dsqrt_rn(2.0 * m + 3.0), x), pmm);  // P_{m,n+1}
  for (int n = m; n <= M; ++n) {
    P[row(n) * Jp + p] = p0;
    double h = __dmul_rn(__dmul_rn(-(double)n, eps_mn(m, n + 1)), p1);
    if (n > m) h = __dadd_rn(h, __dmul_rn(__dmul_rn((double)(n + 1), eps_mn(m, n)), pm1));
    H[row(n) * Jp + p] = h;
    // advance: P_{m,n+2} = (mu P_{n+1} - eps_{n+1} P_n) / eps_{n+2}
    const int n2 = n + 2;
    const double nxt =
        __ddiv_rn(__dsub_rn(__dmul_rn(x, p1), __dmul_rn(eps_mn(m, n2 - 1), p0)), eps_mn(m, n2));
    pm1 = p0;
    p0 = p1;
    p1 = nxt;
  }
}

static void factorize(int N, int *radix, int *ns, int &nst) {
  std::vector<int> f;
  int n = N;
  while (n % 4 == 0) { f.push_back(4); n /= 4; }
  while (n % 2 == 0) { f.push_back(2); n /= 2; }
  for (int p = 3; p * p <= n; p += 2)
    while (n % p == 0) { f.push_back(p); n /= p; }
  if (n > 1) f.push_back(n);
  nst = (int)f.size();
  int acc = 1;
  for (int s = 0; s < nst; ++s) {
    radix[s] = f[s];
    ns[s] = acc;
    acc *= f[s];
  }
}

template <typename T>
static int upload(T **dst, const std::vector<T> &src) {
  SWE_CUDA(cudaMalloc(dst, src.size() * sizeof(T)));
  SWE_CUDA(cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
  return OK;
}

int plan_create(int M, double a, double omega, double gravity, int device, swe_plan **out) {
  if (M < 1) {
    set_error("truncation M must be >= 1");
    return E_SHAPE;
  }
  if (!(a > 0 && gravity > 0) || omega < 0) {
    set_error("radius and gravity must be positive, omega non-negative");
    return E_SHAPE;
  }
  SWE_CUDA(cudaSetDevice(device));
  swe_plan *pl = new swe_plan();
  pl->M = M;
  pl->J = (3 * M + 2) / 2;                 // ceil((3M+1)/2)   spharm.py:61-68
  pl->I = 3 * M + 1 + ((3 * M + 1) & 1);   // 3M+1 rounded up to even
  pl->Jh = (pl->J + 1) / 2;
  pl->Jp = (pl->Jh + AN_KP - 1) / AN_KP * AN_KP;
  pl->K = (M + 1) * (M + 2) / 2;
  pl->N2 = pl->I / 2;
  pl->device = device;
  pl->a = a;
  pl->omega = omega;
  pl->gravity = gravity;
  int rc = gauss_legendre(pl->J, pl->mu, pl->w);
  if (rc) { delete pl; return rc; }

  const int J = pl->J, K = pl->K, Jp = pl->Jp, Jh = pl->Jh;
  std::vector<int> offs(M + 2, 0);
  for (int m = 0; m <= M; ++m) offs[m + 1] = offs[m] + (M + 1 - m);
  pl->h_offsets = offs;
  // internal (device) spectral order = table row order: per m block the even n-m
  // modes, then the odd ones.  perm maps the reference's packed index to it.
  std::vector<double> lap(K), inv(K), eps(K);
  std::vector<int> perm(K);
  for (int m = 0; m <= M; ++m)
    for (int n = m; n <= M; ++n) {
      const int d = n - m, ne = (M + 2 - m) / 2;
      const int k = offs[m] + ((d & 1) ? ne + (d >> 1) : (d >> 1));
      perm[offs[m] + d] = k;
      const double nn1 = (double)n * (n + 1.0);
      lap[k] = -nn1 / (a * a);                      // spharm.py:195-197
      inv[k] = nn1 > 0 ? -(a * a) / nn1 : 0.0;      // spharm.py:198-200
      eps[k] = -lap[k];                             // n(n+1)/a^2 (steppers.py:67)
    }
  std::vector<double> coslv(J), iac(J), fc(J), wsq(J);
  for (int j = 0; j < J; ++j) {
    coslv[j] = sqrt(1.0 - pl->mu[j] * pl->mu[j]);
    iac[j] = 1.0 / (a * coslv[j]);
    fc[j] = 2.0 * omega * pl->mu[j];
    wsq[j] = pl->w[j] / (1.0 - pl->mu[j] * pl->mu[j]);
  }
  if ((rc = upload(&pl->offsets, offs)) || (rc = upload(&pl->perm, perm)) ||
      (rc = upload(&pl->lap_eig, lap)) ||
      (rc = upload(&pl->inv_lap, inv)) || (rc = upload(&pl->eps, eps)) ||
      (rc = upload(&pl->coslat, coslv)) || (rc = upload(&pl->inv_acos, iac)) ||
      (rc = upload(&pl->fcor, fc)) || (rc = upload(&pl->wq, pl->w)) ||
      (rc = upload(&pl->wsin2, wsq)))
    return rc;
  {
    std::vector<double> cs(Jp, 0.0);
    for (int p = 0; p < Jh; ++p) cs[p] = 2.0 * (wsq[p] / a) * (fc[p] / a);
    if ((rc = upload(&pl->cor_scale, cs))) return rc;
  }
  {
    // L_C(xi, delta) = (0, -div(fV), curl(fV)) with f = 2 Omega mu is tridiagonal in n
    // per order m (mu P_n = eps_{n+1} P_{n+1} + eps_n P_{n-1}, H_n = -n eps_{n+1} P_{n+1}
    // + (n+1) eps_n P_{n-1}, V = (psi, chi) from inverse Laplacians of (xi, delta)):
    //   div_n  = 2W [ (n+1)/n eps_n d_{n-1} + n/(n+1) eps_{n+1} d_{n+1} - i m/(n(n+1)) x_n ]
    //   curl_n = 2W [ (n+1)/n eps_n x_{n-1} + n/(n+1) eps_{n+1} x_{n+1} + i m/(n(n+1)) d_n ]
    // The pseudospectral evaluation (dynamics.py:129-135) equals this exactly: its
    // integrands are polynomials of degree <= 2M+2 < 2J, which Gauss quadrature
    // integrates exactly.  Modes n = 0 never reach V (inverse Laplacian), modes
    // n > M are truncated, and m = 0 uses real parts only (irfft/rfft).
    std::vector<int2> nb(K);
    std::vector<double4> cf(K);
    auto row = [&](int m, int n) {
      const int d = n - m, ne = (M + 2 - m) / 2;
      return offs[m] + ((d & 1) ? ne + (d >> 1) : (d >> 1));
    };
    auto epsh = [](int m, int n) {
      return n > m ? sqrt(((double)n * n - (double)m * m) / (4.0 * n * n - 1.0)) : 0.0;
    };
    const double w2 = 2.0 * omega;
    for (int m = 0; m <= M; ++m)
      for (int n = m; n <= M; ++n) {
        const int k = row(m, n);
        nb[k].x = (n - 1 >= m && n - 1 >= 1) ? row(m, n - 1) : -1;
        nb[k].y = n + 1 <= M ? row(m, n + 1) : -1;
        const double nn1 = (double)n * (n + 1.0);
        // absent neighbours (n-1 < m, n-1 = 0, n+1 > M) get a zero coefficient
        cf[k].x = nb[k].x >= 0 ? w2 * epsh(m, n) * ((n + 1.0) / n) : 0.0;
        cf[k].y = nb[k].y >= 0 ? w2 * epsh(m, n + 1) * (n / (n + 1.0)) : 0.0;
        cf[k].z = nn1 > 0 ? w2 * (m / nn1) : 0.0;
        cf[k].w = m == 0 ? 1.0 : 0.0;
      }
    if ((rc = upload(&pl->cor_nb, nb)) || (rc = upload(&pl->cor_cf, cf))) return rc;
    // k_helm_tiled work: each m-block in chunks of 64 consecutive n (32 even + 32 odd
    // rows of the parity-split order), largest m-blocks first
    std::vector<int2> tiles;
    for (int m = 0; m <= M; ++m)
      for (int c = 0; c < (M + 1 - m + 63) / 64; ++c) tiles.push_back(make_int2(m, c));
    pl->n_helm_tiles = (int)tiles.size();
    if ((rc = upload(&pl->zeros, std::vector<double>(1024, 0.0)))) return rc;
    // SETTLS: Gauss nodes and the ascending latitude list with pole ghosts
    // (semilag.py:33-40: -pi - lat[1], -pi - lat[0], lats..., pi - lat[-1], pi - lat[-2])
    std::vector<double> up(J), nodes(J + 4);
    for (int j = 0; j < J; ++j) up[j] = asin(pl->mu[J - 1 - j]);
    const double pi = 3.14159265358979323846;
    nodes[0] = -pi - up[1];
    nodes[1] = -pi - up[0];
    for (int j = 0; j < J; ++j) nodes[2 + j] = up[j];
    nodes[J + 2] = pi - up[J - 1];
    nodes[J + 3] = pi - up[J - 2];
    if ((rc = upload(&pl->mu_dev, pl->mu)) || (rc = upload(&pl->sl_nodes, nodes))) return rc;
    if ((rc = upload(&pl->helm_tiles, tiles))) return rc;
  }

  // Legendre tables on the device (north pairs only)
  const size_t tab = (size_t)K * Jp;
  pl->table_bytes = 2 * tab * sizeof(double);
  SWE_CUDA(cudaMalloc(&pl->P, tab * sizeof(double)));
  SWE_CUDA(cudaMalloc(&pl->H, tab * sizeof(double)));
  {
    double *dmu = nullptr;
    std::vector<double> mu_n(pl->mu.begin(), pl->mu.begin() + Jh);
    if ((rc = upload(&dmu, mu_n))) return rc;
    dim3 grid((Jp + 127) / 128, M + 1);
    table_kernel<<<grid, 128>>>(M, Jh, Jp, dmu, pl->offsets, pl->P, pl->H);
    SWE_LAUNCH_CHECK();
    SWE_CUDA(cudaDeviceSynchronize());
    SWE_CUDA(cudaFree(dmu));
  }

  // TMA tensor maps of the tables for the analysis GEMM: [K rows][Jp] fp64, box of
  // 16 latitude pairs (128 bytes) x 32 mode rows, 128-byte swizzle (the consumers
  // read the tile with the matching XOR); rows past K are zero-filled
  {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
      cudaDriverEntryPointQueryResult q;
      void *fn = nullptr;
      SWE_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
      if (q != cudaDriverEntryPointSuccess || !fn) {
        set_error("cuTensorMapEncodeTiled not available");
        return E_CUDA;
      }
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[2] = {(cuuint64_t)Jp, (cuuint64_t)K};
    const cuuint64_t strides[1] = {(cuuint64_t)Jp * sizeof(double)};
    const cuuint32_t box[2] = {16, 32}, estr[2] = {1, 1};
    double *tabs[2] = {pl->P, pl->H};
    for (int t = 0; t < 2; ++t) {
      const CUresult cr = encode(&pl->tmap[t], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, tabs[t], dims,
                                 strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d)", (int)cr);
        return E_CUDA;
      }
    }
  }

  // FFT: roots of unity in long double, rounded once
  factorize(pl->N2, pl->radix, pl->ns, pl->nst);
  if (pl->nst > FFT_MAXST) {
    set_error("FFT length %d has too many factors", pl->N2);
    return E_SHAPE;
  }
  {
    const int N2 = pl->N2, I = pl->I;
    std::vector<double2> tw(N2), twh(N2);
    for (int e = 0; e < N2; ++e) {
      const long double th = 2.0L * 3.141592653589793238462643383279502884L * e / N2;
      tw[e] = make_double2((double)cosl(th), (double)sinl(th));
      const long double th2 = 2.0L * 3.141592653589793238462643383279502884L * e / I;
      twh[e] = make_double2((double)cosl(th2), (double)sinl(th2));
    }
    if ((rc = upload(&pl->tw, tw)) || (rc = upload(&pl->twh, twh))) return rc;
    // slot maps (fft.cu): pos_z = spectral index -> slot, pos_g = grid pair -> slot
    std::vector<int> pos_z(N2), pos_g(N2);
    pl->pfa = 1;
    for (int s = 0; s < pl->nst; ++s)
      for (int t = s + 1; t < pl->nst; ++t) {
        int x = pl->radix[s], y = pl->radix[t];
        while (y) { const int r = x % y; x = y; y = r; }
        if (x != 1) pl->pfa = 0;
      }
    if (pl->pfa) {
      // Good-Thomas: slot p(i) = sum_s i_s * prod_{t<s} r_t;
      // spectral (Ruritanian) n = sum_s (N/r_s) i_s mod N; grid (CRT) i_s = n mod r_s
      std::vector<int> idx(pl->nst, 0);
      for (int p = 0; p < N2; ++p) {
        int rem = p;
        long long n = 0;
        for (int s = 0; s < pl->nst; ++s) {
          idx[s] = rem % pl->radix[s];
          rem /= pl->radix[s];
          n += (long long)(N2 / pl->radix[s]) * idx[s];
        }
        pos_z[(int)(n % N2)] = p;
      }
      for (int n = 0; n < N2; ++n) {
        int p = 0, mult = 1;
        for (int s = 0; s < pl->nst; ++s) {
          p += (n % pl->radix[s]) * mult;
          mult *= pl->radix[s];
        }
        pos_g[n] = p;
      }
    } else {
      // Cooley-Tukey: digit-reversed spectral slots, natural grid slots
      for (int i = 0; i < N2; ++i) {
        int rem = i, n = N2, mult = 1, res = 0;
        for (int s = pl->nst - 1; s >= 0; --s) {
          n /= pl->radix[s];
          const int q = rem / n;
          rem -= q * n;
          res += q * mult;
          mult *= pl->radix[s];
        }
        pos_z[res] = i;
        pos_g[i] = i;
      }
    }
    if ((rc = upload(&pl->fft_pos_z, pos_z)) || (rc = upload(&pl->fft_pos_g, pos_g))) return rc;
    pl->rgen = 0;
    for (int s = 0; s < pl->nst; ++s)
      if (!fft_small_radix(pl->radix[s])) pl->rgen = std::max(pl->rgen, pl->radix[s]);
  }

  // work items, heaviest order first
  {
    std::vector<int2> sy, an;
    const int ptiles = (Jh + SY_BM - 1) / SY_BM;
    for (int m = 0; m <= M; ++m)
      for (int t = 0; t < ptiles; ++t) sy.push_back(make_int2(m, t));
    for (int m = 0; m <= M; ++m) {
      const int ne = (M + 2 - m) / 2;
      const int rt = (ne + AN_BR - 1) / AN_BR;
      for (int t = 0; t < rt; ++t) an.push_back(make_int2(m, t));
    }
    std::vector<int2> sy3;
    const int pt3 = std::max(1, Jh / 64 + (Jh % 64 > 8 ? 1 : 0));
    for (int m = 0; m <= M; ++m)
      for (int t = 0; t < pt3; ++t) sy3.push_back(make_int2(m, t));
    pl->n_synth_items_v3 = (int)sy3.size();
    if ((rc = upload(&pl->synth_items_v3, sy3))) return rc;
    std::vector<int2> an2;
    for (int m = 0; m <= M; ++m) {
      const int ne = (M + 2 - m) / 2;
      for (int t = 0; t < (ne + V2_ABR - 1) / V2_ABR; ++t) an2.push_back(make_int2(m, t));
    }
    std::vector<int2> an3;
    for (int m = 0; m <= M; ++m) {
      const int ne = (M + 2 - m) / 2;
      for (int t = 0; t < (ne + V3_ABR - 1) / V3_ABR; ++t) an3.push_back(make_int2(m, t));
    }
    pl->n_synth_items = (int)sy.size();
    pl->n_anal_items = (int)an.size();
    pl->n_anal_items_v2 = (int)an2.size();
    pl->n_anal_items_v3 = (int)an3.size();
    if ((rc = upload(&pl->synth_items, sy)) || (rc = upload(&pl->anal_items, an)) ||
        (rc = upload(&pl->anal_items_v2, an2)) || (rc = upload(&pl->anal_items_v3, an3)))
      return rc;
  }
  *out = pl;
  return OK;
}

void graphs_clear(swe_plan *pl) {
  for (auto &g : pl->graphs) {  // entries seen once hold no graph yet
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
  }
  pl->graphs.clear();
}

void work_free(Work &w) {
  cudaFree(w.spec);
  cudaFree(w.half);
  cudaFree(w.fspec);
  cudaFree(w.stats);
  cudaFree(w.fstats);
  cudaFree(w.target2);
  cudaFree(w.flags);
  cudaFree(w.iters);
  cudaFree(w.counter);
  cudaFreeHost(w.h_counter);
  cudaFreeHost(w.h_iters);
  cudaFreeHost(w.h_pub);
  cudaFree(w.sched);
  cudaFree(w.loop);
  cudaFree(w.hdone);
  cudaFreeHost(w.h_bad);
  cudaFree(w.grids);
  cudaFree(w.sweep_g);
  cudaFreeHost(w.h_fail);
  cudaFree(w.d_fail);
  cudaFree(w.gguess);
  cudaFree(w.phi0);
  cudaFree(w.phibar);
  w = Work();
}

void plan_destroy(swe_plan *pl) {
  if (!pl) return;
  cudaSetDevice(pl->device);
  cudaDeviceSynchronize();
  graphs_clear(pl);
  for (auto &c : pl->cap)
    if (c) cudaStreamDestroy(c);
  work_free(pl->ws);
  cudaFree(pl->P);
  cudaFree(pl->H);
  cudaFree(pl->offsets);
  cudaFree(pl->perm);
  cudaFree(pl->lap_eig);
  cudaFree(pl->inv_lap);
  cudaFree(pl->eps);
  cudaFree(pl->coslat);
  cudaFree(pl->inv_acos);
  cudaFree(pl->fcor);
  cudaFree(pl->wq);
  cudaFree(pl->wsin2);
  cudaFree(pl->cor_scale);
  cudaFree(pl->cor_nb);
  cudaFree(pl->helm_tiles);
  cudaFree(pl->zeros);
  cudaFree(pl->mu_dev);
  cudaFree(pl->sl_nodes);
  cudaFree(pl->cor_cf);
  cudaFree(pl->tw);
  cudaFree(pl->twh);
  cudaFree(pl->fft_pos_z);
  cudaFree(pl->fft_pos_g);
  cudaFree(pl->synth_items);
  cudaFree(pl->synth_items_v3);
  cudaFree(pl->anal_items);
  cudaFree(pl->anal_items_v2);
  cudaFree(pl->anal_items_v3);
  delete pl;
}

int work_reserve(swe_plan *pl, int B) {
  Work &w = pl->ws;
  if (B <= w.cap) return OK;
  SWE_CUDA(cudaDeviceSynchronize());
  graphs_clear(pl);
  work_free(w);
  const size_t ld = 2 * (size_t)B;
  const size_t spec = (size_t)pl->K * ld, half = (size_t)(pl->M + 1) * 2 * pl->Jp * ld;
  SWE_CUDA(cudaMalloc(&w.spec, NSPEC * spec * sizeof(double)));
  SWE_CUDA(cudaMalloc(&w.half, NHALF * half * sizeof(double)));
  SWE_CUDA(cudaMalloc(&w.fspec, NF * half * sizeof(double)));
  SWE_CUDA(cudaMalloc(&w.stats, (size_t)B * 8 * sizeof(double)));
  SWE_CUDA(cudaMalloc(&w.fstats, (size_t)B * cn_fused_kmax() * 6 * sizeof(unsigned long long)));
  SWE_CUDA(cudaMemset(w.fstats, 0, (size_t)B * cn_fused_kmax() * 6 * sizeof(unsigned long long)));
  SWE_CUDA(cudaMalloc(&w.target2, (size_t)B * sizeof(int)));
  SWE_CUDA(cudaMalloc(&w.flags, (size_t)B * sizeof(int)));
  SWE_CUDA(cudaMalloc(&w.iters, (size_t)B * sizeof(int)));
  SWE_CUDA(cudaMalloc(&w.counter, sizeof(int)));
  SWE_CUDA(cudaMallocHost(&w.h_counter, sizeof(int)));
  SWE_CUDA(cudaMallocHost(&w.h_iters, (size_t)B * sizeof(int)));
  SWE_CUDA(cudaHostAlloc(&w.h_pub, (size_t)(B + 1) * sizeof(int), cudaHostAllocMapped));
  SWE_CUDA(cudaHostGetDevicePointer(&w.d_pub, w.h_pub, 0));
  SWE_CUDA(cudaMalloc(&w.loop, sizeof(int)));
  SWE_CUDA(cudaMalloc(&w.hdone, sizeof(unsigned)));
  SWE_CUDA(cudaHostAlloc(&w.h_bad, sizeof(int), cudaHostAllocMapped));
  SWE_CUDA(cudaHostGetDevicePointer(&w.d_bad, w.h_bad, 0));
  SWE_CUDA(cudaMemset(w.hdone, 0, sizeof(unsigned)));
  SWE_CUDA(cudaMallocHost(&w.h_fail, sizeof(int)));
  SWE_CUDA(cudaMalloc(&w.d_fail, sizeof(int)));
  SWE_CUDA(cudaMemset(w.d_fail, 0, sizeof(int)));  // swe_imex_step_async accumulates into it
  SWE_CUDA(cudaMalloc(&w.gguess, sizeof(int)));
  {
    const int one = 1;
    SWE_CUDA(cudaMemcpy(w.gguess, &one, sizeof(int), cudaMemcpyHostToDevice));
  }
  SWE_CUDA(cudaMalloc(&w.sched, 2 * sizeof(unsigned long long)));
  SWE_CUDA(cudaMemset(w.sched, 0, 2 * sizeof(unsigned long long)));
  SWE_CUDA(cudaMalloc(&w.phi0, (size_t)B * sizeof(double)));
  SWE_CUDA(cudaMalloc(&w.phibar, (size_t)B * sizeof(double)));
  w.cap = B;
  return OK;
}

}  // namespace swe
