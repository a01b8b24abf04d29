// Legendre GEMMs, warp-specialised persistent variant (the hot path for
// batches of >= 32 slices).
//
// Same contraction as legendre.cu / legendre_v2.cu.  Structure for the sm_100a
// DMMA issue model (each DMMA.8x8x4 holds its warp 16 cycles; 1 DMMA per 16
// cycles per SM sub-partition saturates the FP64 tensor pipe):
//   * warp 0 is the producer: its lanes stream table rows and spectral rows
//     into shared memory with TMA bulk copies (cp.async.bulk ... complete_tx)
//     and arrive on a per-stage "full" mbarrier; rows are padded in shared
//     memory so fragment loads are bank-conflict free;
//   * 8 consumer warps only wait on "full", load fragments and issue DMMAs,
//     then arrive on the stage's "empty" mbarrier (no CTA-wide barriers);
//   * the grid is persistent (one CTA per SM); work units (order m, row tile,
//     column tile, output) are strided over CTAs heaviest first, and the
//     producer runs ahead into the next unit while consumers store results.
// Synthesis: CTA tile 64 latitude pairs x BN columns, consumer warp = one
//   parity class (E/O) x 32 pairs x 64 columns, 16 modes per parity per stage.
// Analysis: CTA tile 64 even + 64 odd modes x BN columns, consumer warp = one
//   parity x 32 modes x 64 columns, 16 latitude pairs per stage; it reads the
//   folded F+/F- rows written by the FFT stage.
#include "legendre.cuh"

namespace swe {

namespace {

// 3 warpgroups: warpgroup 0 = producer (warp 0; warps 1-3 exit), warpgroups 1-2 =
// 8 consumer warps.  setmaxnreg moves registers from the producer warpgroup to the
// consumers (compiled budget 65536/384 = 168 per thread -> 56 / 224).
constexpr int V3_BN = 128, V3_NC = 8, V3_NT = 384, V3_CW0 = 4;
constexpr int S3_KT = 16, S3_NS = 4, S3_LDA = 72 + 4, S3_LDB = V3_BN + 4;
// latitude-pair tiles are 64 wide; a remainder of <= 8 pairs (Jh = 193 at M=256)
// joins the last tile as a fifth 8-row fragment of its upper-half warps instead
// of costing a whole extra work unit (plan.cu synth_items_v3)
constexpr int S3_TW = 64, S3_XTRA = 8;
constexpr int A3_KP = 16, A3_NS = 4, A3_LDA = A3_KP + 4, A3_LDB = V3_BN + 4;
// interleaved F+- rows ([slice][F+, F-] complex, LegTerm::f_il): 2 x 128 doubles per
// pair row, padded to 258 (= 2 mod 16 eight-byte banks: conflict-free B fragments)
constexpr int A3_LDBI = 2 * V3_BN + 2;
constexpr int A3_BR = V3_ABR;  // analysis modes per parity per unit
constexpr int A3_RW = A3_BR / 2, A3_FR = A3_RW / 8;  // rows / 8-row fragments per consumer warp

struct alignas(128) Synth3Stage {
  double A[2 * S3_KT][S3_LDA];
  double B[2 * S3_KT][S3_LDB];
  double S[2 * S3_KT];
  int unit;  // work unit this stage belongs to (first stage of a unit), -1: no more work
};
struct Synth3Smem {
  Synth3Stage st[S3_NS];
  unsigned long long full[S3_NS], empty[S3_NS];
  int next;  // unit handed from producer warp 0 to warp 1
};
// analysis table tile: 2 x 32 mode rows (E, O) x 16 latitude pairs, written by two
// TMA tensor loads with the 128-byte swizzle: the 16-byte chunk c of row r sits at
// chunk c ^ (r & 7) (conflict-free fragment reads without padding)
struct alignas(1024) Anal3Stage {
  double A[2 * A3_BR][A3_KP];
  double F[2][A3_KP][A3_LDB];
  int unit;
};
struct alignas(1024) Anal3Smem {
  Anal3Stage st[A3_NS];
  unsigned long long full[A3_NS], empty[A3_NS];
  int next;  // unit handed from producer thread 0 to the producer warpgroup
};

SWE_DEV unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

SWE_DEV void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
SWE_DEV void mbar_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
SWE_DEV void mbar_arrive_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
SWE_DEV void mbar_wait(unsigned long long *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
SWE_DEV void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// arrive on `bar` once all of this thread's prior cp.async copies have landed
SWE_DEV void cp_async_arrive(unsigned long long *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
// TMA tensor tile (2D) global -> shared, completion counted on `bar` in bytes
SWE_DEV void tma2d(void *dst, const CUtensorMap *tm, int c0, int c1, unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// TMA bulk copy global -> shared, completion counted on `bar` in bytes
SWE_DEV void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

SWE_DEV void regs_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory"); }
SWE_DEV void regs_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory"); }

SWE_DEV double flip_sign(double x, unsigned long long mask) {
  return __longlong_as_double(__double_as_longlong(x) ^ (long long)mask);
}

struct Unit {
  int m, tile, c0, out;
};
SWE_DEV Unit decode(const LegArgs &a, int u, int ncol, int tile_w) {
  Unit x;
  x.out = u % a.nout;
  const int r = u / a.nout;
  const int col = r % ncol;
  const int2 it = a.items[r / ncol];
  x.m = it.x;
  x.tile = it.y * tile_w;
  x.c0 = col * V3_BN;
  return x;
}

// Dynamic work distribution: units are claimed from a device counter
// (sched[0]); every CTA draws one ticket past the end and then checks in on
// sched[1]; the last CTA to check in resets both, so the next launch (stream
// ordered, or the next replay of a CUDA graph) starts from zero without a memset.
SWE_DEV int claim(const LegArgs &a) {
  return (int)atomicAdd(a.sched, 1ULL);
}
SWE_DEV void sched_done(const LegArgs &a) {
  if (atomicAdd(a.sched + 1, 1ULL) == gridDim.x - 1) {
    a.sched[0] = 0;
    a.sched[1] = 0;
  }
}

}  // namespace

__global__ void __launch_bounds__(V3_NT, 1) leg_synth_v3(const __grid_constant__ LegArgs args) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Synth3Smem &sm = *reinterpret_cast<Synth3Smem *>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int M = args.M, Jp = args.Jp, ld = args.ld, Jh = args.Jh;
  const int ncol = (ld + V3_BN - 1) / V3_BN;
  const int nunits = args.nitems * ncol * args.nout;
  if (tid == 0) {
    for (int s = 0; s < S3_NS; ++s) {
      mbar_init(&sm.full[s], 64);  // both producer warps' lanes
      mbar_init(&sm.empty[s], V3_NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp < V3_CW0) {
    // ------------------------------------------------------------ producer
    regs_dec();
    // two producer warps: warp 0 streams the table rows (A), warp 1 the spectral
    // rows (B); each lane issues one bulk copy per stage and arrives with its bytes
    if (warp >= 2) return;
    int it = 0;
    const int r = lane, par = r >> 4;
    while (true) {
      // warp 0 lane 0 claims the unit; named barrier 1 hands it to warp 1
      asm volatile("bar.sync 1, 64;\n" ::: "memory");
      if (warp == 0 && lane == 0) sm.next = claim(args);
      asm volatile("bar.sync 1, 64;\n" ::: "memory");
      const int u = sm.next;
      if (u >= nunits) {  // terminal stage: tells the consumers to stop
        const int s = it % S3_NS;
        mbar_wait(&sm.empty[s], ((it / S3_NS) & 1) ^ 1);
        if (warp == 0 && lane == 0) {
          sm.st[s].unit = -1;
          sched_done(args);
        }
        mbar_arrive(&sm.full[s]);
        break;
      }
      const Unit x = decode(args, u, ncol, 64);
      const LegOut &o = args.out[x.out];
      const int km = M + 1 - x.m, ne = (km + 1) >> 1, no = km >> 1;
      const int off = args.offsets[x.m];
      const int nch_t = (ne + S3_KT - 1) / S3_KT;
      const bool wide = x.tile + S3_TW + S3_XTRA >= Jh;
      const unsigned abytes = (unsigned)min(wide ? S3_TW + S3_XTRA : S3_TW, Jp - x.tile) * 8u;
      const int bcols = min(V3_BN, ld - x.c0);
      // stage c = (term, chunk cc), chunk fastest (counters instead of divisions)
      for (int c = 0, term = 0, cc = 0; c < nch_t * o.nterms; ++c, ++it, cc = cc + 1 == nch_t ? 0 : cc + 1, term += cc == 0) {
        const int s = it % S3_NS;
        mbar_wait(&sm.empty[s], ((it / S3_NS) & 1) ^ 1);
        const int tt = cc * S3_KT + (r & 15);
        const LegTerm &T = o.t[term];
        Synth3Stage &S = sm.st[s];
        const bool v = tt < (par ? no : ne);
        const int k = off + (par ? ne : 0) + tt;
        // rows past the m-block: scale 0 and A/B rows copied from a zero block (shared
        // memory left by an earlier kernel may hold non-finite values, 0 * NaN = NaN)
        if (warp == 0) {
          if (lane == 0) S.unit = u;  // published by lane 0's arrive (release)
          S.S[r] = v ? T.sign * (T.scale ? T.scale[k] : 1.0) * (T.times_im ? (double)x.m : 1.0) : 0.0;
          mbar_arrive_tx(&sm.full[s], abytes);
          bulk_g2s(&S.A[r][0], v ? T.tab + (size_t)k * Jp + x.tile : args.zeros, abytes,
                   &sm.full[s]);
        } else {
          mbar_arrive_tx(&sm.full[s], (unsigned)bcols * 8u);
          bulk_g2s(&S.B[r][0], v ? T.src + (size_t)k * ld + x.c0 : args.zeros,
                   (unsigned)bcols * 8u, &sm.full[s]);
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  regs_inc();
  const int cw = warp - V3_CW0, g = lane >> 2, t = lane & 3;
  const int wpar = cw & 1, wph = (cw >> 1) & 1, wch = cw >> 2;
  int it = 0;
  while (true) {
    {
      const int s = it % S3_NS;
      mbar_wait(&sm.full[s], (it / S3_NS) & 1);
    }
    const int u = sm.st[it % S3_NS].unit;
    if (u < 0) break;
    const Unit x = decode(args, u, ncol, 64);
    const LegOut &o = args.out[x.out];
    const int km = M + 1 - x.m, ne = (km + 1) >> 1, no = km >> 1;
    const int nch_t = (ne + S3_KT - 1) / S3_KT;
    const int pw0 = x.tile + wph * 32;
    const bool wide = x.tile + S3_TW + S3_XTRA >= Jh;  // carries the remainder pairs
    const int tend = wide ? Jh : x.tile + S3_TW;
    const int nfr = max(0, min(4, (tend - pw0 + 7) >> 3));
    // remainder fragment (pairs tile+64 .. tile+71) of a wide tile, split over the
    // four warps of this parity by 32-column quarter so the unit stays balanced
    const int xq = wph * 2 + wch;  // this warp's column quarter of the remainder
    const bool xtra = wide && x.tile + S3_TW < Jh;
    // column fragments holding real columns (small batches: a column's sums do not
    // depend on the others, so skipping empty fragments changes no result)
    const int bcols = min(V3_BN, ld - x.c0);
    const bool wcols = bcols > wch * 64;  // this warp's 64 columns hold real ones
    const bool xcols = bcols > xq * 32;
    double acc[4][8][2], acx[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) acx[j][0] = acx[j][1] = 0.0;
    // the remainder path is a separate instantiation, so ordinary units keep the
    // lean register allocation of the plain 4 x 8 fragment loop
    auto mainloop = [&](auto xt_tag, auto nj_tag) {
      constexpr bool XT = decltype(xt_tag)::value;
      constexpr int NJ = decltype(nj_tag)::value;  // column fragments computed (8, 4, 2)
      for (int c = 0, term = 0, cc = 0; c < nch_t * o.nterms; ++c, ++it, cc = cc + 1 == nch_t ? 0 : cc + 1, term += cc == 0) {
        const int s = it % S3_NS;
        if (c > 0) mbar_wait(&sm.full[s], (it / S3_NS) & 1);
        // small batches: warps whose columns are all padding skip the stage (a
        // column's sums do not depend on the others: no result changes)
        if ((nfr > 0 || XT) && (wcols || (XT && xcols))) {
          const Synth3Stage &S = sm.st[s];
          const LegTerm &T = o.t[term];
          const int rpar = wpar ^ T.flip;
          const int tim = T.times_im;
          const unsigned long long bmask = (tim && !(g & 1)) ? 0x8000000000000000ULL : 0ULL;
          const double *Ab = &S.A[rpar * S3_KT + t][wph * 32 + g];
          const double *Bb = &S.B[rpar * S3_KT + t][wch * 64 + (g ^ tim)];
          const double *Sb = &S.S[rpar * S3_KT + t];
          double a[2][4], b[2][8];
          auto frag = [&](int kk, int q) {
            const double sc = Sb[kk * 4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[q][i] = Ab[kk * 4 * S3_LDA + i * 8] * sc;
#pragma unroll
            for (int j = 0; j < NJ; ++j) b[q][j] = flip_sign(Bb[kk * 4 * S3_LDB + j * 8], bmask);
          };
          // NKK k-steps of 4 modes: the last chunk of an order runs only those holding
          // modes of this warp's parity (the rest are zero rows: no sum changes)
          auto steps = [&](auto nkk_tag) {
            constexpr int NKK = decltype(nkk_tag)::value;
            frag(0, 0);
#pragma unroll
            for (int kk = 0; kk < NKK; ++kk) {
              const int q = kk & 1;
              if (kk + 1 < NKK) frag(kk + 1, q ^ 1);
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (i < nfr) {
#pragma unroll
                  for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], a[q][i], b[q][j]);
                }
              if constexpr (XT) {
                const double *Ax = &S.A[rpar * S3_KT + t][S3_TW + g];
                const double *Bx = &S.B[rpar * S3_KT + t][xq * 32 + (g ^ tim)];
                const double ax = Ax[kk * 4 * S3_LDA] * Sb[kk * 4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  dmma(acx[j][0], acx[j][1], ax, flip_sign(Bx[kk * 4 * S3_LDB + j * 8], bmask));
              }
            }
          };
          const int rem = (rpar ? no : ne) - cc * S3_KT;
          if (rem >= S3_KT - 3) steps(std::integral_constant<int, 4>{});
          else if (rem > 8) steps(std::integral_constant<int, 3>{});
          else if (rem > 4) steps(std::integral_constant<int, 2>{});
          else if (rem > 0) steps(std::integral_constant<int, 1>{});
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);
      }
    };
    // narrow batches (<= 16 / 32 real columns in the tile) compute only the fragments
    // that hold them: a column's sums never depend on the others
    using N8 = std::integral_constant<int, 8>;
    using N4 = std::integral_constant<int, 4>;
    using N2 = std::integral_constant<int, 2>;
    if (xtra) mainloop(std::true_type{}, N8{});
    else if (bcols <= 16) mainloop(std::false_type{}, N2{});
    else if (bcols <= 32) mainloop(std::false_type{}, N4{});
    else mainloop(std::false_type{}, N8{});
    if (o.layout == 0) {
      // E or O plane of [m][2][Jp][ld]
      double *dst = o.dst + ((size_t)x.m * 2 + wpar) * Jp * ld;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int p = pw0 + i * 8 + g;
        if (p >= tend) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int col = x.c0 + wch * 64 + j * 8 + 2 * t;
          if (col < ld)
            *reinterpret_cast<double2 *>(dst + (size_t)p * ld + col) =
                make_double2(acc[i][j][0], x.m ? acc[i][j][1] : 0.0);  // Im of m = 0 is dropped
        }
      }
      const int px = x.tile + S3_TW + g;
      if (xtra && px < Jh) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int col = x.c0 + xq * 32 + j * 8 + 2 * t;
          if (col < ld)
            *reinterpret_cast<double2 *>(dst + (size_t)px * ld + col) =
                make_double2(acx[j][0], x.m ? acx[j][1] : 0.0);
        }
      }
    } else {
      // pair-major [Jh][M+1][ld/2][E,O]: E and O of one (pair, slice, m) share a
      // 32-byte sector, written by the two parity warps of this unit
      double2 *dst = reinterpret_cast<double2 *>(o.dst);
      const int nsl = ld >> 1;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int p = pw0 + i * 8 + g;
        if (p >= tend) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int col = x.c0 + wch * 64 + j * 8 + 2 * t;
          if (col < ld)
            dst[(((size_t)p * (M + 1) + x.m) * nsl + (col >> 1)) * 2 + wpar] =
                make_double2(acc[i][j][0], x.m ? acc[i][j][1] : 0.0);
        }
      }
      const int px = x.tile + S3_TW + g;
      if (xtra && px < Jh) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int col = x.c0 + xq * 32 + j * 8 + 2 * t;
          if (col < ld)
            dst[(((size_t)px * (M + 1) + x.m) * nsl + (col >> 1)) * 2 + wpar] =
                make_double2(acx[j][0], x.m ? acx[j][1] : 0.0);
        }
      }
    }
  }
}

__global__ void __launch_bounds__(V3_NT, 1) leg_anal_v3(const __grid_constant__ LegArgs args) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // the 128-byte swizzle needs 1024-byte aligned tiles
  Anal3Smem &sm = *reinterpret_cast<Anal3Smem *>(smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int M = args.M, Jp = args.Jp, ld = args.ld, Jh = args.Jh;
  const int ncol = (ld + V3_BN - 1) / V3_BN;
  const int nunits = args.nitems * ncol * args.nout;
  const int nch_t = Jp / A3_KP;
  if (tid == 0) {
    for (int s = 0; s < A3_NS; ++s) {
      mbar_init(&sm.full[s], 129);  // every producer thread (cp.async) + thread 0's unit store
      mbar_init(&sm.empty[s], V3_NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp < V3_CW0) {
    regs_dec();
    // the producer warpgroup (128 threads) streams each stage: the table tile
    // (2 x 32 modes x 16 pairs) as two TMA tensor tiles, the F+/F- rows (2 x 16 pairs
    // x 128 columns) as 32 bulk copies; every thread arrives on "full" (thread 0
    // after the expect_tx, the others at once: cp.async.mbarrier.arrive.noinc)
    const int ptid = tid;  // 0..127
    int it = 0;
    while (true) {
      // thread 0 claims the next unit and hands it to the warpgroup (named barrier 1)
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (ptid == 0) sm.next = claim(args);
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      const int u = sm.next;
      if (u >= nunits) {  // terminal stage: tells the consumers to stop
        const int s = it % A3_NS;
        mbar_wait(&sm.empty[s], ((it / A3_NS) & 1) ^ 1);
        if (ptid == 0) {
          sm.st[s].unit = -1;
          sched_done(args);
          mbar_arrive(&sm.full[s]);
        }
        cp_async_arrive(&sm.full[s]);
        break;
      }
      const Unit x = decode(args, u, ncol, A3_BR);
      const LegOut &o = args.out[x.out];
      const int km = M + 1 - x.m, ne = (km + 1) >> 1, no = km >> 1;
      const int off = args.offsets[x.m];
      for (int c = 0, term = 0, cc = 0; c < nch_t * o.nterms; ++c, ++it, cc = cc + 1 == nch_t ? 0 : cc + 1, term += cc == 0) {
        const int s = it % A3_NS;
        mbar_wait(&sm.empty[s], ((it / A3_NS) & 1) ^ 1);
        const int q0 = cc * A3_KP;
        const LegTerm &T = o.t[term];
        Anal3Stage &S = sm.st[s];
        // table rows off + tile.. (E) and off + ne + tile.. (O): rows past the
        // parity block only feed output rows that are never stored; rows past K
        // are zero-filled by the TMA unit
        // F+/F- rows (2 x 16 pairs, up to 1 KB each) as 32 bulk copies (TMA) instead
        // of 2048 16-byte cp.async requests; pairs >= Jh come from the zero block
        const double *fb = T.src + (size_t)x.m * 2 * Jp * ld + x.c0;
        const unsigned fbytes = (unsigned)min(V3_BN, ld - x.c0) * 8u;
        if (ptid == 0) {
          mbar_expect_tx(&sm.full[s], 2u * A3_KP * fbytes + (unsigned)sizeof(S.A));
          const CUtensorMap *tm = &args.tmap[T.flip];
          tma2d(&S.A[0][0], tm, q0, off + x.tile, &sm.full[s]);
          tma2d(&S.A[A3_BR][0], tm, q0, off + ne + x.tile, &sm.full[s]);
        }
        if (T.f_il) {
          // one row of 2 x fbytes (F+ and F- of every slice) per pair
          if (ptid < A3_KP) {
            const int p = q0 + ptid;
            double *Fi = &S.F[0][0][0] + (size_t)ptid * A3_LDBI;
            bulk_g2s(Fi, p < Jh ? T.src + ((size_t)x.m * Jp + p) * 2 * ld + 2 * x.c0 : args.zeros,
                     2 * fbytes, &sm.full[s]);
          }
        } else if (ptid < 2 * A3_KP) {
          const int hs = ptid / A3_KP, pr = ptid % A3_KP, p = q0 + pr;
          bulk_g2s(&S.F[hs][pr][0],
                   p < Jh ? fb + ((size_t)(hs ^ T.swap_pm) * Jp + p) * ld : args.zeros, fbytes,
                   &sm.full[s]);
        }
        if (ptid == 0) {
          S.unit = u;
          mbar_arrive(&sm.full[s]);  // release: publishes S.unit (after the expect_tx)
        }
        cp_async_arrive(&sm.full[s]);
      }
    }
    return;
  }

  regs_inc();
  const int cw = warp - V3_CW0, g = lane >> 2, t = lane & 3;
  const int gr = ((g & 3) << 1) | (g >> 2);  // tile row of fragment row g
  const int wpar = cw & 1, wrq = (cw >> 1) & 1, wch = cw >> 2;
  int it = 0;
  while (true) {
    mbar_wait(&sm.full[it % A3_NS], (it / A3_NS) & 1);
    const int u = sm.st[it % A3_NS].unit;
    if (u < 0) break;
    const Unit x = decode(args, u, ncol, A3_BR);
    const LegOut &o = args.out[x.out];
    const int km = M + 1 - x.m, ne = (km + 1) >> 1, no = km >> 1;
    const int nrow = (wpar ? no : ne) - (x.tile + wrq * A3_RW);
    const int nfr = max(0, min(A3_FR, (nrow + 7) >> 3));
    double acc[A3_FR][8][2];
#pragma unroll
    for (int i = 0; i < A3_FR; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    // small batches: a warp whose 64 columns (planes: wch*64..; interleaved rows:
    // slices wch*32..) are all padding skips the stages (see leg_synth_v3)
    const bool wcols = min(V3_BN, ld - x.c0) > wch * 64;
    // the unit's F layout as a compile-time switch (interleaved rows or planes)
    auto mainloop = [&](auto ilc, auto nj_tag) {
    constexpr bool IL = decltype(ilc)::value;
    constexpr int NJ = decltype(nj_tag)::value;  // column fragments computed (8, 4, 2)
    for (int c = 0, term = 0, cc = 0; c < nch_t * o.nterms; ++c, ++it, cc = cc + 1 == nch_t ? 0 : cc + 1, term += cc == 0) {
      const int s = it % A3_NS;
      if (c > 0) mbar_wait(&sm.full[s], (it / A3_NS) & 1);
      if (nfr > 0 && wcols) {
        const Anal3Stage &S = sm.st[s];
        const LegTerm &T = o.t[term];
        const int tim = T.times_im;
        const int fsel = wpar ^ T.flip;
        const unsigned long long bmask = (tim && !(g & 1)) ? 0x8000000000000000ULL : 0ULL;
        const double asc = T.sign * (tim ? (double)x.m : 1.0);
        // per-pair scale of this lane's k row for each k-step (read-only, L1-cached)
        double ps[A3_KP / 4];
        const int q0 = cc * A3_KP;
#pragma unroll
        for (int kk = 0; kk < A3_KP / 4; ++kk)
          ps[kk] = T.pscale ? __ldg(T.pscale + q0 + kk * 4 + t) : 1.0;
        // fragment row g reads tile row wpar*32 + wrq*16 + i*8 + gr, gr = the even rows
        // for lanes 0-15 and the odd ones for 16-31 (a half-warp's 64-bit loads then
        // hit 8 distinct 16-byte chunks); k index kk*4 + t sits in chunk
        // (2 kk + t/2) ^ gr, element t & 1
        const double *Ab = &S.A[wpar * A3_BR + wrq * A3_RW + gr][t & 1];
        // B column n = wch*64 + j*8 + g' (g' = g ^ tim: re/im swap for i m X).  Planes:
        // slice n/2 of plane fsel.  Interleaved rows: DMMA j's 8 columns are slices
        // wch*32 + (j/2)*8 + (j&1) + 2 (g'/2), so a half-warp's 64-bit loads fall on 16
        // distinct banks (row stride 258 = 2 mod 16); the epilogue stores the same map
        const int gp = g ^ tim;
        const double *Bb =
            IL ? &S.F[0][0][0] + t * A3_LDBI + (wch * 32 + 2 * (gp >> 1)) * 4 + fsel * 2 + (gp & 1)
               : &S.F[fsel][t][wch * 64 + gp];
        constexpr int kst = IL ? 4 * A3_LDBI : 4 * A3_LDB;
        double a[2][A3_FR], b[2][8];
        auto frag = [&](int kk, int q) {
          const int cs = ((2 * kk + (t >> 1)) ^ gr) << 1;
#pragma unroll
          for (int i = 0; i < A3_FR; ++i) a[q][i] = Ab[i * 8 * A3_KP + cs] * (asc * ps[kk]);
#pragma unroll
          for (int j = 0; j < NJ; ++j)
            b[q][j] = flip_sign(Bb[kk * kst + (IL ? (j >> 1) * 32 + (j & 1) * 4 : j * 8)], bmask);
        };
        // NKK k-steps of 4 pairs: the last chunk runs only those holding pairs < Jh
        // (pairs past Jh are zero rows: no sum changes)
        auto steps = [&](auto nkk_tag) {
          constexpr int NKK = decltype(nkk_tag)::value;
          frag(0, 0);
#pragma unroll
          for (int kk = 0; kk < NKK; ++kk) {
            const int q = kk & 1;
            if (kk + 1 < NKK) frag(kk + 1, q ^ 1);
#pragma unroll
            for (int i = 0; i < A3_FR; ++i)
              if (i < nfr) {
#pragma unroll
                for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], a[q][i], b[q][j]);
              }
          }
        };
        const int rem = Jh - q0;
        if (rem >= A3_KP - 3) steps(std::integral_constant<int, 4>{});
        else if (rem > 8) steps(std::integral_constant<int, 3>{});
        else if (rem > 4) steps(std::integral_constant<int, 2>{});
        else if (rem > 0) steps(std::integral_constant<int, 1>{});
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
    }
    };
    const int il = o.t[0].f_il;
    // narrow batches: only the fragments holding real columns (planes: columns
    // j*8..; interleaved rows: j = 0, 1 hold slices 0..7, j < 4 slices 0..15)
    using N8 = std::integral_constant<int, 8>;
    using N4 = std::integral_constant<int, 4>;
    using N2 = std::integral_constant<int, 2>;
    const int bc = min(V3_BN, ld - x.c0);
    if (il) {
      if (bc <= 16) mainloop(std::true_type{}, N2{});
      else if (bc <= 32) mainloop(std::true_type{}, N4{});
      else mainloop(std::true_type{}, N8{});
    } else {
      if (bc <= 16) mainloop(std::false_type{}, N2{});
      else if (bc <= 32) mainloop(std::false_type{}, N4{});
      else mainloop(std::false_type{}, N8{});
    }
    const int nt = wpar ? no : ne;
    const int off = args.offsets[x.m];
#pragma unroll
    for (int i = 0; i < A3_FR; ++i) {
      const int tt = x.tile + wrq * A3_RW + i * 8 + gr;
      if (tt >= nt) continue;
      const size_t k = (size_t)off + (wpar ? ne : 0) + tt;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int col = il ? x.c0 + 2 * (wch * 32 + (j >> 1) * 8 + (j & 1) + 2 * t)
                           : x.c0 + wch * 64 + j * 8 + 2 * t;
        if (col < ld)
          *reinterpret_cast<double2 *>(o.dst + k * ld + col) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
    }
  }
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

int leg_synth_v3_launch(const LegArgs &a, cudaStream_t st) {
  static bool attr = false;
  const int smem = (int)sizeof(Synth3Smem);
  if (!attr) {
    SWE_CUDA(cudaFuncSetAttribute(leg_synth_v3, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  const int units = a.nitems * ((a.ld + V3_BN - 1) / V3_BN) * a.nout;
  const int grid = std::min(units, num_sms());
  leg_synth_v3<<<grid, V3_NT, smem, st>>>(a);
  SWE_LAUNCH_CHECK();
  return OK;
}

int leg_anal_v3_launch(const LegArgs &a, cudaStream_t st) {
  static bool attr = false;
  const int smem = (int)sizeof(Anal3Smem) + 1024;  // + alignment slack (1024-byte tiles)
  if (!attr) {
    SWE_CUDA(cudaFuncSetAttribute(leg_anal_v3, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  const int units = a.nitems * ((a.ld + V3_BN - 1) / V3_BN) * a.nout;
  const int grid = std::min(units, num_sms());
  leg_anal_v3<<<grid, V3_NT, smem, st>>>(a);
  SWE_LAUNCH_CHECK();
  return OK;
}

}  // namespace swe
