// SL-SI-SETTLS building blocks (reference semilag.py:25-179, steppers.py:171-212):
// departure points along great circles with bicubic interpolation of the
// extrapolated wind, bicubic interpolation of grid fields at the departure
// points, and the small spectral/grid combinations of the step.  One thread
// per grid point; the Gaussian-grid latitude search is a binary search over
// the ascending node list with two ghost rows past each pole.
#include <algorithm>

#include "settls.cuh"
#include "spectral.cuh"

namespace swe {

namespace {

struct Stencil {
  int rows[4];   // ascending extended-row indices (0 .. J+3)
  int cols[4];
  double wt[4];  // latitude weights
  double wl[4];  // longitude weights
};

// extended ascending row e (0..J+3) -> (grid row north->south, longitude shift)
SWE_DEV void ext_row(int e, int J, int &row, bool &shift) {
  // ascending rows: a = e - 2 in 0..J-1 maps to grid row J-1-a
  if (e < 2) {            // ghosts below the south pole: asc rows 1, 0 shifted
    row = J - 1 - (1 - e);
    shift = true;
  } else if (e >= J + 2) {  // ghosts above the north pole: asc rows J-1, J-2 shifted
    row = e - (J + 2);
    shift = true;
  } else {
    row = J - 1 - (e - 2);
    shift = false;
  }
}

SWE_DEV Stencil stencil(const double *__restrict__ nodes, int next, int I, double lam,
                        double th) {
  Stencil s;
  const double two_pi = 6.283185307179586476925286766559;
  lam = fmod(lam, two_pi);
  if (lam < 0.0) lam += two_pi;
  const double dlon = two_pi / I;
  const double x = lam / dlon;
  const double fi = floor(x);
  const int i0 = (int)fi;
  const double t = x - fi;
  s.wl[0] = -t * (t - 1.0) * (t - 2.0) / 6.0;
  s.wl[1] = (t + 1.0) * (t - 1.0) * (t - 2.0) / 2.0;
  s.wl[2] = -(t + 1.0) * t * (t - 2.0) / 2.0;
  s.wl[3] = (t + 1.0) * t * (t - 1.0) / 6.0;
  for (int q = 0; q < 4; ++q) s.cols[q] = ((i0 + q - 1) % I + I) % I;
  // j = searchsorted(nodes, th) - 1 (left insertion point), clipped to [1, next-3]
  int lo = 0, hi = next;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (nodes[mid] < th) lo = mid + 1;
    else hi = mid;
  }
  int j = lo - 1;
  j = j < 1 ? 1 : (j > next - 3 ? next - 3 : j);
  double nd[4];
  for (int q = 0; q < 4; ++q) {
    s.rows[q] = j - 1 + q;
    nd[q] = nodes[j - 1 + q];
  }
  for (int k = 0; k < 4; ++k) {
    double num = 1.0, den = 1.0;
    for (int l = 0; l < 4; ++l) {
      if (l == k) continue;
      num = num * (th - nd[l]);
      den = den * (nd[k] - nd[l]);
    }
    s.wt[k] = num / den;
  }
  return s;
}

// bicubic value of grid g ([J][I], north->south) at a stencil
SWE_DEV double interp(const double *__restrict__ g, int J, int I, const Stencil &s) {
  double acc = 0.0;
  const int half = I / 2;
  for (int a = 0; a < 4; ++a) {
    int row;
    bool shift;
    ext_row(s.rows[a], J, row, shift);
    const double *gr = g + (size_t)row * I;
    double r = 0.0;
    for (int b = 0; b < 4; ++b) {
      const int c = shift ? (s.cols[b] - half + I) % I : s.cols[b];
      r += gr[c] * s.wt[a] * s.wl[b];
    }
    acc += r;
  }
  return acc;
}

struct V3 {
  double x, y, z;
};
SWE_DEV V3 v3(double x, double y, double z) { return V3{x, y, z}; }
SWE_DEV V3 add(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
SWE_DEV V3 mul(double s, V3 a) { return v3(s * a.x, s * a.y, s * a.z); }
SWE_DEV double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
SWE_DEV V3 cross(V3 a, V3 b) {
  return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}

// great-circle step of length |w| dt / a backward from xa along w (semilag.py:108-117)
SWE_DEV V3 back(V3 xa, V3 w, double dt, double a) {
  const double sp = sqrt(dot(w, w));
  const double sig = sp * dt / a;
  const V3 dir = sp > 0.0 ? mul(1.0 / sp, w) : v3(0.0, 0.0, 0.0);
  const V3 xd = add(mul(cos(sig), xa), mul(-sin(sig), dir));
  return mul(1.0 / sqrt(dot(xd, xd)), xd);
}

// parallel transport of v from src to dst (semilag.py:120-131)
SWE_DEV V3 transport(V3 v, V3 src, V3 dst) {
  const V3 k = cross(src, dst);
  const double s2 = dot(k, k), c = dot(src, dst);
  if (s2 < 1e-24) return v;
  return add(add(mul(c, v), cross(k, v)), mul(dot(k, v) * (1.0 - c) / s2, k));
}

SWE_DEV void lonlat(V3 xd, double &lam, double &th) {
  const double two_pi = 6.283185307179586476925286766559;
  lam = fmod(atan2(xd.y, xd.x), two_pi);
  if (lam < 0.0) lam += two_pi;
  th = asin(fmin(fmax(xd.z, -1.0), 1.0));
}

// unit vectors at grid point (row j, column i)
SWE_DEV void frame(const SetArgs &a, int j, int i, V3 &xa, V3 &el, V3 &et) {
  const double lam = 6.283185307179586476925286766559 * i / a.I;
  const double mu = a.mu[j], c = a.coslat[j];
  const double cl = cos(lam), sl = sin(lam);
  xa = v3(c * cl, c * sl, mu);
  el = v3(-sl, cl, 0.0);
  et = v3(-mu * cl, -mu * sl, c);
}

// extrapolated wind (Cartesian) at grid point (row, col) of slice b:
// 2 (u, v)(t_n) - (u, v)(t_{n-1}) in the local frame
SWE_DEV V3 vext(const SetArgs &a, int b, int row, int col) {
  const size_t o = ((size_t)b * a.J + row) * a.I + col;
  const double ue = a.ext_given ? a.up[o] : 2.0 * a.un[o] - a.up[o];
  const double ve = a.ext_given ? a.vp[o] : 2.0 * a.vn[o] - a.vp[o];
  V3 xa, el, et;
  frame(a, row, col, xa, el, et);
  return add(mul(ue, el), mul(ve, et));
}

SWE_DEV V3 interp_vext(const SetArgs &a, int b, const Stencil &s) {
  V3 acc = v3(0.0, 0.0, 0.0);
  const int half = a.I / 2;
  for (int q = 0; q < 4; ++q) {
    int row;
    bool shift;
    ext_row(s.rows[q], a.J, row, shift);
    V3 r = v3(0.0, 0.0, 0.0);
    for (int p = 0; p < 4; ++p) {
      const int c = shift ? (s.cols[p] - half + a.I) % a.I : s.cols[p];
      const V3 w = vext(a, b, row, c);
      const double f = s.wt[q] * s.wl[p];
      r = add(r, mul(f, w));
    }
    acc = add(acc, r);
  }
  return acc;
}

__global__ void k_departure(SetArgs a, int iterations, double dt, double *lam_out,
                            double *th_out, int *bad) {
  const size_t n = (size_t)a.B * a.J * a.I;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < n;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % a.I);
    const int j = (int)((idx / a.I) % a.J);
    const int b = (int)(idx / ((size_t)a.I * a.J));
    V3 xa, el, et;
    frame(a, j, i, xa, el, et);
    const V3 wa = add(mul(a.un[idx], el), mul(a.vn[idx], et));
    V3 xd = back(xa, wa, dt, a.radius);
    for (int it = 0; it < iterations; ++it) {
      double lam, th;
      lonlat(xd, lam, th);
      const Stencil s = stencil(a.nodes, a.J + 4, a.I, lam, th);
      V3 we = interp_vext(a, b, s);
      we = add(we, mul(-dot(we, xd), xd));
      const V3 w = mul(0.5, add(transport(we, xd, xa), wa));
      xd = back(xa, w, dt, a.radius);
    }
    double lam, th;
    lonlat(xd, lam, th);
    if (!isfinite(lam) || !isfinite(th)) *bad = 1;
    lam_out[idx] = lam;
    th_out[idx] = th;
  }
}

__global__ void k_interp(SetArgs a, const double *lam, const double *th, int nf, GridPtrs p) {
  const size_t n = (size_t)a.B * a.J * a.I;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < n;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int b = (int)(idx / ((size_t)a.I * a.J));
    const Stencil s = stencil(a.nodes, a.J + 4, a.I, lam[idx], th[idx]);
    for (int f = 0; f < nf; ++f)
      p.out[f][idx] = interp(p.in[f] + (size_t)b * a.J * a.I, a.J, a.I, s);
  }
}

// (phi - phibar) * delta on the grid: nonlinear_rest's product (dynamics.py:154-160);
// the phi_prime shift of mode (0,0) synthesises to phibar at every point
__global__ void k_phiprime_mul(int B, size_t per, const double *phi, const double *de,
                               const double *phibar, double *out) {
  const size_t n = (size_t)B * per;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < n;
       idx += (size_t)gridDim.x * blockDim.x)
    out[idx] = (phi[idx] - phibar[idx / per]) * de[idx];
}

// G = U + h (L U + 2 N_R(U) - N_R(prev)) for Phi; U + h L U for xi, delta
// (steppers.py:196-199, N_R has only a Phi component)
__global__ void k_settls_g(size_t n, Ptr3C u, Ptr3C l, const double2 *nru, const double2 *nrp,
                           double h, Ptr3 g) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const double2 *u0 = reinterpret_cast<const double2 *>(u.p[0]);
    const double2 *l0 = reinterpret_cast<const double2 *>(l.p[0]);
    const double2 a = l0[i], b = nru[i], c = nrp[i], x = u0[i];
    reinterpret_cast<double2 *>(g.p[0])[i] =
        make_double2(x.x + h * ((a.x + 2.0 * b.x) - c.x), x.y + h * ((a.y + 2.0 * b.y) - c.y));
    for (int f = 1; f < 3; ++f) {
      const double2 xf = reinterpret_cast<const double2 *>(u.p[f])[i];
      const double2 lf = reinterpret_cast<const double2 *>(l.p[f])[i];
      reinterpret_cast<double2 *>(g.p[f])[i] = make_double2(xf.x + h * lf.x, xf.y + h * lf.y);
    }
  }
}

// y += s x (complex)
__global__ void k_spec_axpy(size_t n, double2 *y, const double2 *x, double s) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    y[i] = make_double2(y[i].x + s * x[i].x, y[i].y + s * x[i].y);
}

static int nblk(size_t n) { return (int)std::min<size_t>((n + 255) / 256, 148 * 16); }

}  // namespace

int settls_g(int K, int B, double *const u[3], double *const l[3], const double *nru,
             const double *nrp, double h, double *const g[3], cudaStream_t st) {
  const size_t n = (size_t)K * B;
  Ptr3C uu = {{u[0], u[1], u[2]}}, ll = {{l[0], l[1], l[2]}};
  Ptr3 gg = {{g[0], g[1], g[2]}};
  k_settls_g<<<nblk(n), 256, 0, st>>>(n, uu, ll, reinterpret_cast<const double2 *>(nru),
                                      reinterpret_cast<const double2 *>(nrp), h, gg);
  SWE_LAUNCH_CHECK();
  return OK;
}

int spec_axpy(int K, int B, double *y, const double *x, double s, cudaStream_t st) {
  const size_t n = (size_t)K * B;
  k_spec_axpy<<<nblk(n), 256, 0, st>>>(n, reinterpret_cast<double2 *>(y),
                                       reinterpret_cast<const double2 *>(x), s);
  SWE_LAUNCH_CHECK();
  return OK;
}

int departure_points(const SetArgs &a, int iterations, double dt, double *lam, double *th,
                     int *bad, cudaStream_t st) {
  k_departure<<<nblk((size_t)a.B * a.J * a.I), 256, 0, st>>>(a, iterations, dt, lam, th, bad);
  SWE_LAUNCH_CHECK();
  return OK;
}

int interp_fields(const SetArgs &a, const double *lam, const double *th, int nf,
                  const GridPtrs &p, cudaStream_t st) {
  if (nf < 1 || nf > 4) {
    set_error("interp_fields: nf = %d outside 1..4", nf);
    return E_SHAPE;
  }
  k_interp<<<nblk((size_t)a.B * a.J * a.I), 256, 0, st>>>(a, lam, th, nf, p);
  SWE_LAUNCH_CHECK();
  return OK;
}

int phiprime_mul(int B, size_t per, const double *phi, const double *de, const double *phibar,
                 double *out, cudaStream_t st) {
  k_phiprime_mul<<<nblk((size_t)B * per), 256, 0, st>>>(B, per, phi, de, phibar, out);
  SWE_LAUNCH_CHECK();
  return OK;
}

}  // namespace swe
