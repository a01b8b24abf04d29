// Shared FFT device primitives (complex arithmetic, small-radix DFT kernels).
#pragma once

#include "common.cuh"

namespace swe {
namespace fftcore {

SWE_DEV double2 cm(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
SWE_DEV double2 twd(const double2 *tw, int e, double dir) {
  double2 w = __ldg(tw + e);
  w.y *= dir;
  return w;
}

// y_t = sum_q v_q exp(dir 2 pi i q t / R); cr/sr hold cos/sin(2 pi e / R) for
// e = 0..(R-1)/2 (v is clobbered)
template <int R>
SWE_DEV void dft(double2 (&v)[R], double dir, const double *cr, const double *sr, double2 (&y)[R]) {
  if constexpr (R == 2) {
    y[0] = make_double2(v[0].x + v[1].x, v[0].y + v[1].y);
    y[1] = make_double2(v[0].x - v[1].x, v[0].y - v[1].y);
  } else if constexpr (R == 4) {
    const double2 s02 = make_double2(v[0].x + v[2].x, v[0].y + v[2].y);
    const double2 d02 = make_double2(v[0].x - v[2].x, v[0].y - v[2].y);
    const double2 s13 = make_double2(v[1].x + v[3].x, v[1].y + v[3].y);
    const double2 d13 = make_double2(v[1].x - v[3].x, v[1].y - v[3].y);
    const double2 rot = make_double2(-dir * d13.y, dir * d13.x);  // i*dir*d13
    y[0] = make_double2(s02.x + s13.x, s02.y + s13.y);
    y[2] = make_double2(s02.x - s13.x, s02.y - s13.y);
    y[1] = make_double2(d02.x + rot.x, d02.y + rot.y);
    y[3] = make_double2(d02.x - rot.x, d02.y - rot.y);
  } else {
    constexpr int H = (R - 1) / 2;
    y[0] = v[0];
#pragma unroll
    for (int q = 1; q <= H; ++q) {
      const double2 p = v[q], m = v[R - q];
      v[q] = make_double2(p.x + m.x, p.y + m.y);
      v[R - q] = make_double2(p.x - m.x, p.y - m.y);
      y[0].x += v[q].x;
      y[0].y += v[q].y;
    }
#pragma unroll
    for (int t = 1; t <= H; ++t) {
      double re = v[0].x, im = v[0].y, sx = 0.0, sy = 0.0;
#pragma unroll
      for (int q = 1; q <= H; ++q) {
        const int e = (q * t) % R;
        const double c = e <= H ? cr[e] : cr[R - e];
        const double s = e <= H ? sr[e] : -sr[R - e];
        re += v[q].x * c;
        im += v[q].y * c;
        sx += v[R - q].x * s;
        sy += v[R - q].y * s;
      }
      y[t] = make_double2(re - dir * sy, im + dir * sx);
      y[R - t] = make_double2(re + dir * sy, im - dir * sx);
    }
  }
}

// dft, optionally times exp(dir 2 pi i t kt / N2), stored to dst[t*stride]
template <int R>
SWE_DEV void dft_store(double2 (&v)[R], double dir, const double *cr, const double *sr,
                       double2 *dst, int stride, const double2 *tw, int kt) {
  double2 y[R];
  dft<R>(v, dir, cr, sr, y);
#pragma unroll
  for (int t = 0; t < R; ++t) dst[t * stride] = (kt && t) ? cm(y[t], twd(tw, t * kt, dir)) : y[t];
}

}  // namespace fftcore
}  // namespace swe
