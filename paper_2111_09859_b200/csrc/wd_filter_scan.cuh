// Fast-arithmetic implicit filter sweep (SolveConfig.arith="fast"): the
// tridiagonal system of operators.py:305-352 (10th-order filter, reduced
// order near the ends, identity end rows; cyclic by Sherman-Morrison on
// periodic axes, oracle/wd.py:cyclic_apply) solved as a SEGMENTED AFFINE
// SCAN in shared memory instead of one sequential recurrence per line.
//
// Why: the exact sweep (wd_filter_sweep.cuh) must follow dgtsv's row order,
// so each line is one 2 x n-step dependency chain and the input is read
// twice.  The filter matrix is field independent, so both recurrences of
// the LU solve
//     y_r = rhs_r - f_{r-1} y_{r-1}          x_r = y_r / d_r - g_r x_{r+1}
// are affine maps with precomputed coefficients.  A CTA stages 16 whole
// lines in shared memory (one HBM read), splits every line into 16
// segments of m <= 32 rows (256 threads = 16 lines x 16 segments) and
//   1. computes the right-hand side and the local forward recurrence of
//      its segment from zero (registers),
//   2. gets the true carry-in y_{r0-1} from the segment ends of the
//      preceding segments (c = Yend_t + P_end(t) c, <= 15 FMAs), fixes its
//      rows with y_r = y'_r + P_r c, P_r = prod(-f) from the segment start,
//   3. does the same for the back substitution with Q_r = prod(-g) to the
//      segment end,
// and writes the line once (one HBM write).  Same linear system, round-off
// level differences; the multipliers |f|, |g| < 1 (diagonally dominant
// filter matrix), so the scan is stable.  HBM traffic: 2 words per node
// (+1 for the fused convergence reduction) versus 3 for the exact sweep.
//
// Layout: the tile carries 5 ghost rows per side (periodic: wrapped rows,
// otherwise zeros), so the 11-point window never branches on the line end.
// Axes 0/1 (row stride != 1): [row][line], lines = 16 consecutive k, each
// row one 128-byte segment in HBM, staged with 16-byte cp.async.  Axis 2
// (contiguous lines): [line][row] with an odd line stride (bank-conflict
// free), lines = 16 consecutive j.  Tables (shared memory, broadcast reads):
// (f_{r-1}, h_r), (P_r, g_r), 1/d_r, (Q_r, z_r) -- one 16-byte load per
// phase and row.  With n = 16 m (m = 32 at 512^3) the rows of a segment are
// compile-time: the reduced-order rows at the line ends get compile-time
// coefficients and only rows 0-4 / m-5..m-1 of y' stay in registers, the
// rest go back into the tile behind the window (rows no other thread reads).
#pragma once

#include <cuda.h>  // CUtensorMap (the encoder is resolved at run time, no libcuda link)

#include "wd_filter_sweep.cuh"
#include "wd_fused.cuh"

namespace wd {

// Tensor maps of the sweep's input for the TMA tile loads (strided axes,
// full-segment tiles): `main` moves n / 2 rows x 16 lines per copy, `ghost`
// the 5 wrapped rows of a periodic line.
struct ScanTma {
  CUtensorMap main, ghost;
};

__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WD_MBAR_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra WD_MBAR_DONE;\n"
      "bra WD_MBAR_WAIT;\n"
      "WD_MBAR_DONE:\n"
      "}\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}
// 2-D / 3-D tile loads: box of the tensor map at (c0, c1[, c2]) -> dst,
// completion (bytes) signalled on `bar`
__device__ __forceinline__ void tma_load_2d(double* dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(double* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

struct ScanArgs {
  const double* in;
  double* out;
  int axis;
  int n0, n1, n2;
  long long s0;
  int per;
  ScanDev T;
  FilterCoef fc;
  const double* A;  // nullptr -> no convergence reduction
  Status* st;
  const double* fixc;    // FIX: [3][n1 n2] coefficient planes (see SweepArgs)
  const double* fixrow;  // FIX: [3][n0] per-plane factors
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = ok ? 8 : 0;  // 0 -> zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(sz));
}
// 16 bytes, the first `bytes` (0, 8, 16) copied, the rest zero filled
__device__ __forceinline__ void cp_async16(double* dst, const double* src, int bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// full-order (10th) right-hand side, window w[0..10] centred at w[5], FMA form
__device__ __forceinline__ double fs_rhs5(const double* w, const FilterCoef& fc) {
  const double* c = fc.hc + 30;
  double v = c[5] * (w[10] + w[0]);
  v = fma(c[4], w[9] + w[1], v);
  v = fma(c[3], w[8] + w[2], v);
  v = fma(c[2], w[7] + w[3], v);
  v = fma(c[1], w[6] + w[4], v);
  return fma(c[0], w[5], v);
}
// reduced order h (compile time in the full-segment path)
__device__ __forceinline__ double fs_rhs_c(const double* w, int H, const FilterCoef& fc) {
  if (H == 0) return w[5];
  double v = fc.hc[H * 6] * w[5];
#pragma unroll
  for (int k = 1; k <= 5; ++k)
    if (k <= H) v = fma(fc.hc[H * 6 + k], w[5 + k] + w[5 - k], v);
  return v;
}
__device__ __forceinline__ double fs_rhsh(const double* w, int h, const double* hc) {
  if (h == 0) return w[5];
  const double* c = hc + h * 6;
  double v = c[0] * w[5];
#pragma unroll
  for (int k = 1; k <= 5; ++k)
    if (k <= h) v = fma(c[k], w[5 + k] + w[5 - k], v);
  return v;
}

// MM > 0: every segment has exactly MM rows (n = 16 MM); MM = 0: any n <= 512.
// RED: fused convergence reduction against a.A (separate instantiation, so
// the plain sweeps carry no predicated reduction code).
// TMA (strided axes, full-segment tiles, inner length a multiple of 16): the
// tile is loaded by one elected thread with cp.async.bulk.tensor (two copies
// of n / 2 rows x 128 bytes + the wrapped ghost rows) completing on two
// mbarriers, one per half of the rows, so the segments of the first half
// start their right-hand sides while the second half is still in flight;
// the other instantiations stage with per-thread cp.async.
// FIX (AX2 && RED only): out = x + c0 W_i + c1 Qp_i - c2 z_i with the
// per-line coefficients c(j, k) and the per-plane factors of plane i: the
// correction of the slab-decomposed axis-0 filter, which commutes with the j
// and k sweeps (all linear), applied here instead of in a pass of its own.
template <bool AX2, int MM, bool RED, bool TMA, bool FIX = false>
#ifndef WD_SCAN_TG
#define WD_SCAN_TG 0  // 1: factor tables read from global memory (L1) instead of shared
#endif
#ifndef WD_SCAN_PF
#define WD_SCAN_PF 1  // L2 prefetch of A and the next tile, stride-1 lines
                      // (A/B: filter along k 0.83 -> 0.70 ms at 512^3; on
                      // the strided axes it measured neutral to slower)
#endif
#ifndef WD_SCAN_MINB
#define WD_SCAN_MINB 2
#endif
__global__ void __launch_bounds__(FS_T, WD_SCAN_MINB)
    k_filter_scan(ScanArgs a, const __grid_constant__ ScanTma tm) {
  if (a.st->state != WD_STATE_RUNNING) return;
  extern __shared__ __align__(128) double fs_smem[];
  constexpr bool kTma = TMA && !AX2 && MM > 0;
  __shared__ __align__(8) unsigned long long tbar[2];
  // full-segment tiles: n = FS_S * MM at compile time (scan dispatch, wd_fused.cu)
  const int n = MM > 0 ? FS_S * MM : a.T.n, m = MM > 0 ? MM : a.T.m, per = a.per;
  // tables: T1 (fm, h), T2 (P, g), T4 (Q, z) as double2; T3 rinv
  const double* tb = WD_SCAN_TG ? a.T.tab : fs_smem;
  const double2* T1 = reinterpret_cast<const double2*>(tb);
  const double2* T2 = T1 + n;
  const double2* T4 = T2 + n;
  const double* T3 = tb + 6 * n;
  constexpr int tabn = WD_SCAN_TG ? 0 : 1;  // tables in shared memory?
  double* shc = fs_smem + tabn * 7 * n;  // FilterCoef (dynamic h: generic path)
  double* tile = fs_smem + ((tabn * 7 * n + 36 + 15) & ~15);  // 128-byte aligned (TMA / cp.async)
  const int NR = n + 2 * FS_G;
  const int LS = NR | 1;  // AX2 line stride (odd)
  const int tsz = AX2 ? FS_L * LS : NR * FS_L;
  double* Yend = tile + tsz;
  double* Xst = Yend + FS_T;
  double* Hs = Xst + FS_T;
  if (!WD_SCAN_TG)
    for (int t = threadIdx.x; t < 7 * n; t += FS_T) fs_smem[t] = a.T.tab[t];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 36; ++k) shc[k] = a.fc.hc[k];
  }

  const int tid = threadIdx.x, l = tid % FS_L, s = tid / FS_L;
  const int r0 = s * m;
  const int cnt = max(0, min(m, n - r0));
  const int nseg = (n + m - 1) / m;
  int inner_n;
  long long outer_n, rstride, lstride;
  if (a.axis == 0) {
    inner_n = a.n2; outer_n = a.n1; rstride = a.s0; lstride = 1;
  } else if (a.axis == 1) {
    inner_n = a.n2; outer_n = a.n0; rstride = a.n2; lstride = 1;
  } else {
    inner_n = a.n1; outer_n = a.n0; rstride = 1; lstride = a.n2;
  }
  const int nb = (inner_n + FS_L - 1) / FS_L;
  const long long groups = outer_n * nb;
  const double rden = 1.0 / a.T.denom;
  const bool vec16 = !AX2 && (rstride % 2 == 0);  // 16-byte rows (base parity per tile)

  long long t_outer = 0;  // tile coordinates of the last tile_of (TMA)
  int t_inner0 = 0;
  auto tile_of = [&](long long q, long long& base, int& nl) {
    const long long outer = q / nb;
    const int inner0 = (int)(q - outer * nb) * FS_L;
    t_outer = outer;
    t_inner0 = inner0;
    nl = min(FS_L, inner_n - inner0);
    if (a.axis == 0) base = outer * a.n2 + inner0;
    else if (a.axis == 1) base = outer * a.s0 + inner0;
    else base = outer * a.s0 + (long long)inner0 * a.n2;
  };
  // stage rows -5 .. n+4 of the tile's lines (cp.async; ghosts wrapped or 0)
  auto load = [&](long long base, int nl) {
    const double* in = a.in + base;
    if (AX2) {
      // main rows: consecutive threads -> consecutive rows of one line
      const double* src = in + tid;
      double* dst = tile + FS_G + tid;
      for (int ll = 0; ll < nl; ++ll) {
        for (int r = 0; r + tid < n; r += FS_T) cp_async8(dst + r, src + r, true);
        src += lstride;
        dst += LS;
      }
      if (tid < 2 * FS_G * FS_L) {  // ghosts: 10 rows x 16 lines
        const int ll = tid / (2 * FS_G), gq = tid - ll * 2 * FS_G;
        const int rr = gq < FS_G ? gq : n + gq;  // tile row
        const int r = per ? (gq < FS_G ? n - FS_G + gq : gq - FS_G) : 0;
        cp_async8(tile + ll * LS + rr, in + (long long)ll * lstride + r, per && ll < nl);
      }
    } else if (vec16 && (base % 2 == 0)) {
      const int c = tid & 7;  // line pair
      const int bytes = 2 * c < nl ? (2 * c + 1 < nl ? 16 : 8) : 0;
      const double* src = in + 2 * c;
      if (tid < 2 * FS_G * 8) {
        const int gq = tid >> 3;
        const int rr = gq < FS_G ? gq : n + gq;
        const int r = per ? (gq < FS_G ? n - FS_G + gq : gq - FS_G) : 0;
        cp_async16(tile + rr * FS_L + 2 * c, src + (long long)r * rstride, per ? bytes : 0);
      }
      const long long step = (FS_T / 8) * rstride;
      src += (long long)(tid >> 3) * rstride;
      double* dst = tile + (FS_G + (tid >> 3)) * FS_L + 2 * c;
      for (int r = tid >> 3; r < n; r += FS_T / 8) {
        cp_async16(dst, src, bytes);
        src += step;
        dst += (FS_T / 8) * FS_L;
      }
    } else {
      const bool ok = l < nl;
      const double* src = in + l;
      if (s < 2 * FS_G) {
        const int rr = s < FS_G ? s : n + s;
        const int r = per ? (s < FS_G ? n - FS_G + s : s - FS_G) : 0;
        cp_async8(tile + rr * FS_L + l, src + (long long)r * rstride, per && ok);
      }
      const long long step = FS_S * rstride;
      src += (long long)s * rstride;
      double* dst = tile + (FS_G + s) * FS_L + l;
      for (int r = s; r < n; r += FS_S) {
        cp_async8(dst, src, ok);
        src += step;
        dst += FS_S * FS_L;
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  // TMA: thread 0 arms the two mbarriers with the bytes of their half and
  // issues the copies; tile rows [0, 5) / [n + 5, n + 10) are the ghosts
  auto load_tma = [&]() {
    if (tid != 0) return;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // tile last written by threads
    const unsigned half = (unsigned)(n / 2) * FS_L * 8u, gh = per ? FS_G * FS_L * 8u : 0u;
    mbar_expect_tx(&tbar[0], half + gh);
    mbar_expect_tx(&tbar[1], half + gh);
    if (a.axis == 0) {
      const int c0 = (int)(t_outer * a.n2 + t_inner0);
      if (per) tma_load_2d(tile, &tm.ghost, c0, n - FS_G, &tbar[0]);
      tma_load_2d(tile + FS_G * FS_L, &tm.main, c0, 0, &tbar[0]);
      tma_load_2d(tile + (FS_G + n / 2) * FS_L, &tm.main, c0, n / 2, &tbar[1]);
      if (per) tma_load_2d(tile + (FS_G + n) * FS_L, &tm.ghost, c0, 0, &tbar[1]);
    } else {
      const int c2 = (int)t_outer;
      if (per) tma_load_3d(tile, &tm.ghost, t_inner0, n - FS_G, c2, &tbar[0]);
      tma_load_3d(tile + FS_G * FS_L, &tm.main, t_inner0, 0, c2, &tbar[0]);
      tma_load_3d(tile + (FS_G + n / 2) * FS_L, &tm.main, t_inner0, n / 2, c2, &tbar[1]);
      if (per) tma_load_3d(tile + (FS_G + n) * FS_L, &tm.ghost, t_inner0, 0, c2, &tbar[1]);
    }
  };
  if (kTma) {
    if (tid == 0) {
      mbar_init(&tbar[0], 1);
      mbar_init(&tbar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (!per)  // wall lines: zero ghosts, written once (no copy ever lands there)
      for (int t = tid; t < 2 * FS_G * FS_L; t += FS_T)
        tile[(t < FS_G * FS_L ? 0 : n * FS_L) + t] = 0.0;
    __syncthreads();
  }
  unsigned tphase = 0;
  double md = 0.0, ma = 0.0;
  int bad = 0;
  long long q = blockIdx.x;
  long long base = 0;
  int nl = 0;
  if (q < groups) {
    tile_of(q, base, nl);
    if (kTma) load_tma();
    else load(base, nl);
  }
  const int RS = AX2 ? 1 : FS_L;
  double* tl = tile + (AX2 ? l * LS : l) + (r0 + FS_G) * RS;  // row r0 of my line
  for (; q < groups; q += gridDim.x) {
    if (kTma) {
      // a segment's window spans tile rows [r0, r0 + m + 10): wait for the
      // half (or halves) it touches only
      if (r0 < n / 2 + FS_G) mbar_wait(&tbar[0], tphase);
      if (r0 + m + 2 * FS_G > n / 2 + FS_G) mbar_wait(&tbar[1], tphase);
      tphase ^= 1u;
    } else {
      cp_async_wait_all();
      __syncthreads();
    }
#if WD_SCAN_PF
    // full-segment tiles: pull the convergence operand of this tile and the
    // input rows of the next one into L2 while this tile is solved, so the
    // store-phase loads of A and the next cp.async fill see L2 latency
    if (MM > 0 && AX2) {
      auto pf = [](const double* p) { asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p)); };
      long long nb2 = 0;
      int nl2 = 0;
      const bool nxt = q + gridDim.x < groups;
      if (nxt) tile_of(q + gridDim.x, nb2, nl2);
#pragma unroll
      for (int k = tid; k < FS_L * (FS_NMAX / 16); k += FS_T) {
        // AX2: 16 lines x (n / 16) 128-byte pieces; else n rows x 128 bytes
        const int ll = AX2 ? k / (n / 16) : 0, pc = AX2 ? k % (n / 16) : k;
        const long long off = AX2 ? ll * lstride + pc * 16 : (long long)pc * rstride;
        if (AX2 ? ll < nl : pc < n) {
          if (RED) pf(a.A + base + off);
        }
        if (nxt && (AX2 ? ll < nl2 : pc < n)) pf(a.in + nb2 + off);
      }
    }
#endif
    // ---- 1. right-hand side + local forward recurrence (from zero)
    double yv[MM > 0 ? 10 : FS_M];  // MM > 0: rows 0-4 and MM-5..MM-1 only
    double hs = 0.0, yp = 0.0;
    {
      double ww[(MM > 0 ? MM : FS_M) + 10];
#pragma unroll
      for (int k = 0; k < 10; ++k) ww[k] = tl[(k - 5) * RS];
      if constexpr (MM > 0) {
        const bool first = !per && s == 0;          // rows 0..4: h = row
        const bool last = !per && s == FS_S - 1;    // rows MM-5..MM-1: h = MM-1-row
        double dq[6];
#pragma unroll
        for (int rr = 0; rr < MM; ++rr) {
          ww[rr + 10] = tl[(rr + 5) * RS];
          double rhs;
          if (rr < 5 && first) rhs = fs_rhs_c(ww + rr, rr, a.fc);
          else if (rr >= MM - 5 && last) rhs = fs_rhs_c(ww + rr, MM - 1 - rr, a.fc);
          else rhs = fs_rhs5(ww + rr, a.fc);
          const double2 t1 = T1[r0 + rr];
          yp = fma(-t1.x, yp, rhs);
          if (per) hs = fma(t1.y, rhs, hs);
          if (rr < 5) yv[rr] = yp;
          else if (rr >= MM - 5) yv[rr - MM + 10] = yp;
          else dq[rr % 6] = yp;
          const int qd = rr - 5;  // row whose input the window no longer needs
          if (qd >= 5 && qd < MM - 5) tl[qd * RS] = dq[qd % 6];
        }
      } else {
#pragma unroll
        for (int rr = 0; rr < FS_M; ++rr) {
          if (rr < cnt) {
            ww[rr + 10] = tl[(rr + 5) * RS];
            const int r = r0 + rr;
            const int hh = per ? 5 : min(min(r, n - 1 - r), 5);
            const double rhs = hh == 5 ? fs_rhs5(ww + rr, a.fc) : fs_rhsh(ww + rr, hh, shc);
            const double2 t1 = T1[r];
            yp = fma(-t1.x, yp, rhs);
            yv[rr] = yp;
            if (per) hs = fma(t1.y, rhs, hs);
          }
        }
      }
    }
    Yend[tid] = yp;
    Hs[tid] = hs;
    __syncthreads();
    // generic path, axes 0/1: the staged input is consumed and the output
    // leaves from registers -> prefetch the next tile now
    long long nbase = 0;
    int nnl = 0;
    if (MM == 0 && !AX2 && q + gridDim.x < groups) {
      tile_of(q + gridDim.x, nbase, nnl);
      load(nbase, nnl);
    }
    // ---- 2. forward carry, fix-up, local back substitution
    double c = 0.0;
    for (int t = 0; t < s; ++t) c = fma(T2[t * m + m - 1].x, c, Yend[t * FS_L + l]);
    double xn = 0.0;
    if constexpr (MM > 0) {
#pragma unroll
      for (int rr = MM - 1; rr >= 0; --rr) {
        const bool reg = rr < 5 || rr >= MM - 5;
        const int ri = rr < 5 ? rr : rr - MM + 10;
        const double yl = reg ? yv[ri] : tl[rr * RS];
        const double2 t2 = T2[r0 + rr];
        const double y = fma(t2.x, c, yl);
        xn = fma(-t2.y, xn, y * T3[r0 + rr]);
        if (reg) yv[ri] = xn;
        else tl[rr * RS] = xn;
      }
    } else {
#pragma unroll
      for (int rr = FS_M - 1; rr >= 0; --rr) {
        if (rr < cnt) {
          const int r = r0 + rr;
          const double2 t2 = T2[r];
          const double y = fma(t2.x, c, yv[rr]);
          xn = fma(-t2.y, xn, y * T3[r]);
          yv[rr] = xn;
        }
      }
    }
    Xst[tid] = xn;
    __syncthreads();
    // ---- 3. backward carry, fix-up, cyclic correction
    double c2 = 0.0;
    for (int t = nseg - 1; t > s; --t) c2 = fma(T4[t * m].x, c2, Xst[t * FS_L + l]);
    double f = 0.0;
    if (per) {
      double hsum = 0.0;
      for (int t = 0; t < nseg; ++t) hsum += Hs[t * FS_L + l];
      f = hsum * rden;
    }
    auto xfin = [&](int rr, double xl) {  // x' + Q c2 - f z
      const double2 t4 = T4[r0 + rr];
      double x = fma(t4.x, c2, xl);
      if (per) x = fma(-f, t4.y, x);
      return x;
    };
    // FIX: the plane's factors and the tile's offset inside a coefficient plane
    double fxW = 0.0, fxQ = 0.0, fxZ = 0.0;
    long long fxoff = 0;
    if (FIX) {
      const long long oc = q / nb;  // plane i of this tile (axis 2: outer = i)
      fxW = a.fixrow[oc];
      fxQ = a.fixrow[a.n0 + oc];
      fxZ = a.fixrow[2 * a.n0 + oc];
      fxoff = base - oc * a.s0;
    }
    const long long fxN = (long long)a.n1 * a.n2;
    auto fixed = [&](double x, long long off2) {  // off2: offset inside the plane
      if (!FIX) return x;
      const double* pc = a.fixc + off2;
      x = fma(__ldg(pc), fxW, x);
      x = fma(__ldg(pc + fxN), fxQ, x);
      return fma(-__ldg(pc + 2 * fxN), fxZ, x);
    };
    // ---- 4. store (+ convergence reduction against A)
    auto emit = [&](double* po, const double* pa, double x) {
      __stcs(po, x);
      if (RED) {
        if (!isfinite(x)) bad = 1;
        ma = fmax(ma, fabs(x));
        md = fmax(md, fabs(x - __ldcs(pa)));
      }
    };
    if (!AX2) {
      if (l < nl) {
        const long long b = base + l + (long long)r0 * rstride;
        double* po = a.out + b;
        const double* pa = RED ? a.A + b : nullptr;
        if constexpr (MM > 0) {
#pragma unroll
          for (int rr = 0; rr < MM; ++rr) {
            const bool reg = rr < 5 || rr >= MM - 5;
            const int ri = rr < 5 ? rr : rr - MM + 10;
            emit(po, pa, xfin(rr, reg ? yv[ri] : tl[rr * RS]));
            po += rstride;
            if (RED) pa += rstride;
          }
        } else {
#pragma unroll
          for (int rr = 0; rr < FS_M; ++rr) {
            if (rr < cnt) {
              emit(po, pa, xfin(rr, yv[rr]));
              po += rstride;
              if (RED) pa += rstride;
            }
          }
        }
      }
      if (MM == 0) {
        base = nbase;
        nl = nnl;
      } else if (q + gridDim.x < groups) {
        // the threads' writes into the tile (y', x') are ordered before the
        // next copy of the async proxy
        if (kTma) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();  // every thread done with the tile
        tile_of(q + gridDim.x, base, nl);
        if (kTma) load_tma();
        else load(base, nl);
      }
    } else {
      if constexpr (MM > 0) {
#pragma unroll
        for (int rr = 0; rr < MM; ++rr) {
          const bool reg = rr < 5 || rr >= MM - 5;
          const int ri = rr < 5 ? rr : rr - MM + 10;
          tl[rr] = xfin(rr, reg ? yv[ri] : tl[rr]);
        }
      } else {
#pragma unroll
        for (int rr = 0; rr < FS_M; ++rr)
          if (rr < cnt) tl[rr] = xfin(rr, yv[rr]);
      }
      __syncthreads();
      {
        double* po = a.out + base + tid;
        const double* pa = RED ? a.A + base + tid : nullptr;
        const double* pt = tile + FS_G + tid;
        if (MM > 0 && !RED) {
          for (int ll = 0; ll < nl; ++ll) {
#pragma unroll
            for (int r = 0; r < FS_S * MM; r += FS_T) __stcs(po + r, pt[r]);
            po += lstride;
            pt += LS;
          }
        } else if (MM > 0) {
          // batches of 4 lines: 8 independent loads of A in flight per thread
          for (int l0 = 0; l0 < nl; l0 += 4) {
            constexpr int KK = MM > 0 ? FS_S * MM / FS_T : 1;
            double av[4][KK];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int k = 0; k < KK; ++k)
                av[u][k] = l0 + u < nl ? __ldcs(pa + u * lstride + k * FS_T) : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (l0 + u < nl) {
#pragma unroll
                for (int k = 0; k < KK; ++k) {
                  const double x = fixed(pt[u * LS + k * FS_T],
                                         fxoff + (l0 + u) * lstride + tid + k * FS_T);
                  __stcs(po + u * lstride + k * FS_T, x);
                  if (!isfinite(x)) bad = 1;
                  ma = fmax(ma, fabs(x));
                  md = fmax(md, fabs(x - av[u][k]));
                }
              }
            }
            po += 4 * lstride;
            pa += 4 * lstride;
            pt += 4 * LS;
          }
        } else {
          for (int ll = 0; ll < nl; ++ll) {
            for (int r = 0; r + tid < n; r += FS_T)
              emit(po + r, pa + r, fixed(pt[r], fxoff + ll * lstride + tid + r));
            po += lstride;
            if (RED) pa += lstride;
            pt += LS;
          }
        }
      }
      if (q + gridDim.x < groups) {
        __syncthreads();  // tile fully read before it is overwritten
        tile_of(q + gridDim.x, base, nl);
        load(base, nl);
      }
    }
  }
  if (RED) {
    md = warp_max(md);
    ma = warp_max(ma);
    bad = __any_sync(0xffffffffu, bad);
    if ((tid & 31) == 0) {
      atomicMax(&a.st->max_delta_bits, (unsigned long long)__double_as_longlong(md));
      atomicMax(&a.st->max_abs_bits, (unsigned long long)__double_as_longlong(ma));
      if (bad) atomicOr(&a.st->nonfinite, 1);
    }
  }
}

inline size_t scan_smem(int n) {
  const int NR = n + 2 * FS_G;
  const size_t tile = (size_t)FS_L * (size_t)(NR | 1);  // >= NR * FS_L
  return ((((size_t)(WD_SCAN_TG ? 0 : 7) * n + 36 + 15) & ~(size_t)15) + tile + 3 * FS_T) *
         sizeof(double);
}

}  // namespace wd
