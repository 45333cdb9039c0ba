// Fast-arithmetic compact first derivative (SolveConfig.arith="fast",
// generic path): the C4/C6 system of operators.py:94-148 (closures of
// operators.py:136-145; cyclic on periodic axes, oracle/wd.py:cyclic_apply)
// solved as the segmented affine scan of wd_filter_scan.cuh, with the
// derivative epilogue (Epi: D, c*D or acc + c*D) fused into the store.
//
// Why: the exact line solve follows dgtsv's row order and interchanges, so
// one derivative pass is a right-hand-side kernel plus a forward and a back
// sweep through HBM (rhs write + read, y write + read: ~8 field transfers
// with the epilogue operands).  Here a CTA stages 16 whole lines in shared
// memory, computes the right-hand side from the staged rows, solves, and
// applies the epilogue on the way out: 1 read of the input + the epilogue
// operands + 1 write (2-4 field transfers per pass).
//
// The factor is the no-pivoting LU (Thomas) of the same matrix
// (compact_factor_fast, wd_capi.cu): swap-free, which the scan form needs;
// its multipliers stay bounded (|l| <= 3.2 at the closure rows, -> 0.38 in
// the interior), so round-off stays at the level of the exact solve.
// Results differ from dgtsv's in the last bits (tests/test_gpu_deriv_scan.py).
//
// Lines: stride-1 axes ("AX2") stage [line][row] (odd line stride: bank
// conflict free), 16 consecutive lines; strided axes stage [row][line], 16
// consecutive lines (inner index), each tile row one 128-byte run in HBM.
// 256 threads = 16 lines x 16 segments of m <= 32 rows, n in [12, 512].
#pragma once

#include "wd_filter_scan.cuh"

namespace wd {

constexpr int DS_G = 2;  // ghost rows per side (C6 reach)

struct DScanArgs {
  const double* in;
  double* out;
  long long N;   // nodes
  long long sa;  // stride of the axis (1 -> AX2)
  int per;
  int scheme;  // WD_C4 / WD_C6
  ScanDev T;
  Epi epi;
  const Status* st;
};

// Tile shapes: NL lines x NS = TT / NL segments, TT threads.
//   n <= 512:          16 lines x 16 segments, 256 threads, 2 CTAs / SM;
//   512 < n <= 1024:   stride-1 lines 8 x 32 / 256 threads with the factor
//                      tables read through L1 (2 CTAs / SM); strided lines
//                      16 x 32 / 512 threads (1 CTA / SM), so every tile row
//                      is a 128-byte run in HBM rather than 64 bytes.
struct DScanShape {
  int NL, TT;
};
inline DScanShape dscan_shape(int n, bool ax2) {
  if (n <= FS_NMAX) return {16, 256};
  return ax2 ? DScanShape{8, 256} : DScanShape{16, 512};
}
inline int dscan_segments(int n) { return n <= FS_NMAX ? 16 : 32; }
inline size_t dscan_smem(int n, DScanShape sh) {
  const int NR = n + 2 * DS_G;
  const bool tg = sh.NL == 8;
  const size_t tab = tg ? 0 : (size_t)((7 * n + 3) & ~3);
  return (tab + (size_t)sh.NL * (size_t)(NR | 1) + 3 * (size_t)sh.TT) * sizeof(double);
}

// MM > 0: every segment has exactly MM rows (n = 16 MM, compile-time row
// loops without guards: the register window is renamed, not moved); MM = 0:
// any n in [12, NS * 32].  PER / C6: periodic axis, scheme C6 (else C4).
template <bool AX2, int MM, bool PER, bool C6, int NL, int TT>
__global__ void __launch_bounds__(TT, TT == 256 ? 2 : 1) k_deriv_scan(DScanArgs a) {
  if (a.st && a.st->state != WD_STATE_RUNNING) return;
  extern __shared__ double ds_smem[];
  constexpr int NS = TT / NL;
  constexpr bool TG = NL == 8;            // tables from global (L1)
  constexpr int UM = MM > 0 ? MM : FS_M;  // unrolled rows per segment
  // full-segment tiles: n = NS * MM is a compile-time constant (dscan_pick),
  // which folds the tile / table offsets and the row bounds
  // (not the 512-thread n = 1024 tiles: at their 128-register cap the extra
  // constant propagation spills and measured 774 -> 808 us per pass)
  const int n = (MM > 0 && TT == 256) ? (TT / NL) * MM : a.T.n, m = MM > 0 ? MM : a.T.m;
  constexpr bool per = PER;
  const double* tb = TG ? a.T.tab : ds_smem;
  const double2* T1 = reinterpret_cast<const double2*>(tb);  // (fm, h)
  const double2* T2 = T1 + n;                                // (P, g)
  const double2* T4 = T2 + n;                                // (Q, z)
  const double* T3 = tb + 6 * n;                             // 1/d
  double* tile = ds_smem + (TG ? 0 : ((7 * n + 3) & ~3));
  const int NR = n + 2 * DS_G;
  const int LS = NR | 1;
  double* Yend = tile + (AX2 ? NL * LS : NR * NL);
  double* Xst = Yend + TT;
  double* Hs = Xst + TT;
  if (!TG)
    for (int t = threadIdx.x; t < 7 * n; t += TT) ds_smem[t] = a.T.tab[t];

  const int tid = threadIdx.x, l = tid % NL, s = tid / NL;
  const int r0 = s * m;
  const int cnt = MM > 0 ? MM : max(0, min(m, n - r0));
  const int nseg = (n + m - 1) / m;
  const long long sa = a.sa;
  // lines: AX2 -> q * n (L = N / n lines); strided -> outer * n * sa + inner
  const long long inner_n = AX2 ? a.N / n : sa;
  const long long outer_n = AX2 ? 1 : a.N / (n * sa);
  const long long nb = (inner_n + NL - 1) / NL;
  const long long groups = outer_n * nb;
  const double rden = 1.0 / a.T.denom;
  const int RS = AX2 ? 1 : NL;
  const long long lstride = AX2 ? n : 1;

  auto tile_of = [&](long long q, long long& base, int& nl) {
    const long long outer = q / nb;
    const long long inner0 = (q - outer * nb) * NL;
    nl = (int)min((long long)NL, inner_n - inner0);
    base = AX2 ? inner0 * n : outer * n * sa + inner0;
  };
  // rows -2 .. n+1 of the tile's lines (ghosts wrapped when periodic, else 0)
  auto load = [&](long long base, int nl) {
    const double* in = a.in + base;
    if (AX2) {
      for (int ll = 0; ll < nl; ++ll) {
        const double* src = in + ll * lstride;
        double* dst = tile + ll * LS + DS_G;
        for (int r = tid; r < n; r += TT) cp_async8(dst + r, src + r, true);
      }
      if (tid < 2 * DS_G * NL) {
        const int ll = tid / (2 * DS_G), gq = tid - ll * 2 * DS_G;
        const int rr = gq < DS_G ? gq : n + gq;  // tile row
        const int r = per ? (gq < DS_G ? n - DS_G + gq : gq - DS_G) : 0;
        cp_async8(tile + ll * LS + rr, in + ll * lstride + r, per && ll < nl);
      }
    } else {
      const bool ok = l < nl;
      const double* src = in + l;
      if (s < 2 * DS_G) {
        const int rr = s < DS_G ? s : n + s;
        const int r = per ? (s < DS_G ? n - DS_G + s : s - DS_G) : 0;
        cp_async8(tile + rr * NL + l, src + (long long)r * sa, per && ok);
      }
      for (int r = s; r < n; r += NS)
        cp_async8(tile + (DS_G + r) * NL + l, src + (long long)r * sa, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  long long q = blockIdx.x, base = 0;
  int nl = 0;
  if (q < groups) {
    tile_of(q, base, nl);
    load(base, nl);
  }
  // row r0 of my line in the tile
  double* tl = tile + (AX2 ? l * LS : l) + (r0 + DS_G) * RS;
  for (; q < groups; q += gridDim.x) {
    cp_async_wait_all();
    __syncthreads();
    // ---- 1. right-hand side (compact_rhs_at) + local forward recurrence
    double yv[UM];
    double yp = 0.0, hs = 0.0;
    {
      // closure rows (operators.py:136-145) once per thread, outside the
      // unrolled body (it would otherwise carry 2 divisions per row: ~15k
      // SASS instructions, instruction-cache bound)
      const double* c0 = tl - r0 * RS;  // row 0 of the line
      double rc0 = 0.0, rcn = 0.0;
      if (!per && s == 0)
        rc0 = (-17.0 * c0[0] + 9.0 * c0[RS] + 9.0 * c0[2 * RS] - c0[3 * RS]) / 6.0;
      if (!per && r0 + cnt == n && cnt > 0)
        rcn = (17.0 * c0[(n - 1) * RS] - 9.0 * c0[(n - 2) * RS] - 9.0 * c0[(n - 3) * RS] +
               c0[(n - 4) * RS]) / 6.0;
      double w0 = tl[-2 * RS], w1 = tl[-RS], w2 = tl[0], w3 = tl[RS];
#pragma unroll
      for (int rr = 0; rr < UM; ++rr) {
        if (MM > 0 || rr < cnt) {
          const double w4 = tl[(rr + 2) * RS];
          const int r = r0 + rr;
          const double d1 = w3 - w1;
          double rhs = C6 ? fma(C6_CB, w4 - w0, C6_CA * d1) : C4_CA * d1;
          if (!PER && (MM == 0 || rr <= 1 || rr >= UM - 2)) {
            rhs = (C6 && (r == 1 || r == n - 2)) ? 0.75 * d1 : rhs;
            rhs = r == 0 ? rc0 : rhs;
            rhs = r == n - 1 ? rcn : rhs;
          }
          const double2 t1 = T1[r];
          yp = fma(-t1.x, yp, rhs);
          if (per) hs = fma(t1.y, rhs, hs);
          yv[rr] = yp;
          w0 = w1;
          w1 = w2;
          w2 = w3;
          w3 = w4;
        }
      }
    }
    Yend[tid] = yp;
    Hs[tid] = hs;
    __syncthreads();
    // strided axes: the staged input is consumed and the output leaves from
    // registers -> the next tile's rows are in flight from here on
    long long nbase = 0;
    int nnl = 0;
    if (!AX2 && q + gridDim.x < groups) {
      tile_of(q + gridDim.x, nbase, nnl);
      load(nbase, nnl);
    }
    // ---- 2. forward carry, fix-up, local back substitution
    double c = 0.0;
    for (int t = 0; t < s; ++t) c = fma(T2[t * m + m - 1].x, c, Yend[t * NL + l]);
    double xn = 0.0;
#pragma unroll
    for (int rr = UM - 1; rr >= 0; --rr) {
      if (MM > 0 || rr < cnt) {
        const int r = r0 + rr;
        const double2 t2 = T2[r];
        const double y = fma(t2.x, c, yv[rr]);
        xn = fma(-t2.y, xn, y * T3[r]);
        yv[rr] = xn;
      }
    }
    Xst[tid] = xn;
    __syncthreads();
    // ---- 3. backward carry, fix-up, cyclic correction
    double c2 = 0.0;
    for (int t = nseg - 1; t > s; --t) c2 = fma(T4[t * m].x, c2, Xst[t * NL + l]);
    double f = 0.0;
    if (per) {
      double hsum = 0.0;
      for (int t = 0; t < nseg; ++t) hsum += Hs[t * NL + l];
      f = hsum * rden;
    }
    // epilogue operands (acc, c) are fetched 8 rows / 4 lines at a time so
    // their HBM latencies overlap instead of serialising on the store loop
    const Epi& e = a.epi;
    const bool need_acc = e.mode == 2, need_c = e.mode != 0 && e.cfield != nullptr;
    // coefficient stored once per line of the last axis (Epi::ccomp): on the
    // strided axes the tile's 16 lines share one value per row
    const bool kc = e.cdiv > 1;
    auto fin = [&](double x, double av, double cv) {
      if (e.mode == 0) return x;
      const double t = cv * x;
      return e.mode == 1 ? t : av + t;
    };
    if (!AX2) {
      if (l < nl) {
        const long long b = base + l + (long long)r0 * sa;
        const double* pa = e.acc + b;
        const long long csa = kc ? sa / e.cdiv : sa;
        const double* pc = kc ? e.ccomp + b / e.cdiv : e.cfield + b;
        double* po = a.out + b;
#pragma unroll
        for (int rb = 0; rb < UM; rb += 8) {
          double av[8], cv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const bool ok = MM > 0 || rb + u < cnt;
            av[u] = ok && need_acc ? pa[u * sa] : 0.0;
            cv[u] = ok && need_c ? pc[u * csa] : e.cscal;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int rr = rb + u;
            if (MM > 0 || rr < cnt) {
              const double2 t4 = T4[r0 + rr];
              double x = fma(t4.x, c2, yv[rr]);
              if (per) x = fma(-f, t4.y, x);
              __stcs(po + u * sa, fin(x, av[u], cv[u]));
            }
          }
          pa += 8 * sa;
          pc += 8 * csa;
          po += 8 * sa;
        }
      }
      base = nbase;
      nl = nnl;
    } else {
#pragma unroll
      for (int rr = 0; rr < UM; ++rr) {
        if (MM > 0 || rr < cnt) {
          const double2 t4 = T4[r0 + rr];
          double x = fma(t4.x, c2, yv[rr]);
          if (per) x = fma(-f, t4.y, x);
          tl[rr] = x;
        }
      }
      __syncthreads();
      // rows per thread and line (exact for full segments), lines per batch
      constexpr int KR = MM > 0 ? (NS * MM + TT - 1) / TT : NS * FS_M / TT;
      constexpr int LB = 8 / KR;
      const long long cline = kc ? base / n : 0;  // first line of the tile
      for (int l0 = 0; l0 < nl; l0 += LB) {
        double av[LB][KR], cv[LB][KR];
#pragma unroll
        for (int u = 0; u < LB; ++u)
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            const int r = tid + k * TT;
            const bool ok = l0 + u < nl && r < n;
            const long long idx = base + (l0 + u) * lstride + r;
            av[u][k] = ok && need_acc ? e.acc[idx] : 0.0;
            // stride-1 lines are lines of the last axis: one value per line
            cv[u][k] = ok && need_c ? (kc ? e.ccomp[cline + l0 + u] : e.cfield[idx]) : e.cscal;
          }
#pragma unroll
        for (int u = 0; u < LB; ++u)
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            const int r = tid + k * TT;
            if (l0 + u < nl && r < n) {
              const long long idx = base + (l0 + u) * lstride + r;
              __stcs(a.out + idx, fin(tile[(l0 + u) * LS + DS_G + r], av[u][k], cv[u][k]));
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
}

}  // namespace wd

namespace wd {

using DScanFn = void (*)(DScanArgs);
template <bool AX2, int MM, int NL, int TT>
inline DScanFn dscan_pick4(bool per, bool c6) {
  if (per)
    return c6 ? k_deriv_scan<AX2, MM, true, true, NL, TT> : k_deriv_scan<AX2, MM, true, false, NL, TT>;
  return c6 ? k_deriv_scan<AX2, MM, false, true, NL, TT> : k_deriv_scan<AX2, MM, false, false, NL, TT>;
}
template <bool AX2>
inline DScanFn dscan_pick(int n, bool per, bool c6) {
  constexpr int NLB = AX2 ? 8 : 16, TTB = AX2 ? 256 : 512;  // n > 512
  if (n == 512) return dscan_pick4<AX2, 32, 16, 256>(per, c6);
  if (n == 256) return dscan_pick4<AX2, 16, 16, 256>(per, c6);
  if (n <= FS_NMAX) return dscan_pick4<AX2, 0, 16, 256>(per, c6);
  if (n == 2 * FS_NMAX) return dscan_pick4<AX2, 32, NLB, TTB>(per, c6);
  return dscan_pick4<AX2, 0, NLB, TTB>(per, c6);
}
// the instantiation for a line length / stride / periodicity / scheme; its
// dynamic shared-memory limit is raised on every call (cheap, host only)
inline DScanFn dscan_kernel(int n, bool ax2, bool per, bool c6) {
  const DScanFn f = ax2 ? dscan_pick<true>(n, per, c6) : dscan_pick<false>(n, per, c6);
  cudaFuncSetAttribute((const void*)f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)dscan_smem(n, dscan_shape(n, ax2)));
  return f;
}

}  // namespace wd
