// Generic line solves (compact first derivative, operators.py:130-148, and
// implicit filter, operators.py:305-352) for the generic path, in two
// kernels:
//
//   k_line_rhs    every node in parallel: the right-hand side row
//                 (compact_rhs_at / the filter row of half-order h) into a
//                 scratch field;
//   k_line_solve  a warp owns 32 lines (lane = line) and runs LAPACK dgtsv
//                 in its exact elimination order, row interchanges included
//                 (tri_solve_line, wd_kernels.cuh), restated as a carried
//                 row state: before step i the carry is the current row i
//                 of the eliminated system; step i with b = rhs[i+1] gives
//                   no swap: y_i = carry,  carry' = b - f_i * carry
//                   swap:    y_i = b,      carry' = carry - f_i * b
//                 and y_{n-1} = the final carry (y overwrites the scratch
//                 in place); back substitution
//                   x_i = ((y_i - du_i x_{i+1}) - du2_i x_{i+2}) / d_i
//                 (the quotient as the correctly rounded reciprocal
//                 product), periodic lines adding the Sherman-Morrison
//                 correction x - (h.rhs / denom) z (oracle/wd.py:
//                 cyclic_apply, h.rhs accumulated in row order).
//
// The recurrences are latency chains; everything that is not on the chain
// (stencils, boundary closures, pin tests, index arithmetic) runs in the
// fully parallel first kernel, so the solve issues ~10 instructions per row
// and the factor lives in shared memory.  Results are written through the
// derivative epilogue (JOB 0) or with the pinned-node restore (JOB 1).
#pragma once

#include "wd_kernels.cuh"

namespace wd {

#ifndef WD_LS_U
#define WD_LS_U 8
#endif
#ifndef WD_LS_MINB
#define WD_LS_MINB 1
#endif
#ifndef WD_LT_EPI
#define WD_LT_EPI 1
#endif
constexpr int LS_WARPS = 4;        // warps per CTA of k_line_solve
constexpr int LS_U = WD_LS_U;      // rows per unrolled group
constexpr int LS_MINB = WD_LS_MINB;  // resident CTAs per SM asked of ptxas
constexpr bool LT_EPI = WD_LT_EPI != 0;  // k_line_solve_t: epilogue operands via cp.async tiles

__device__ __forceinline__ double ls_div(double s, double d, double r) {
  const double q0 = s * r;
  const double e = fma(-q0, d, s);
  return fma(e, r, q0);
}

template <int JOB>
static __global__ void k_line_rhs(const double* __restrict__ in, double* __restrict__ rhs,
                                  AxisGeom ag, int per, double off, int scheme, FilterCoef fc,
                                  const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  const long long sa = ag.sa;
  const int n = ag.n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < ag.N;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = ag.coord(idx);
    double r;
    constexpr int H = JOB == 0 ? 2 : 5;  // stencil reach
    if (i >= H && i < n - H && sa == 1) {
      // stride-1 interior: compile-time offsets (same expressions)
      const double* q = in + idx;
      if (JOB == 0) {
        if (scheme == WD_C4) r = C4_CA * (q[1] - q[-1]);
        else r = C6_CA * (q[1] - q[-1]) + C6_CB * (q[2] - q[-2]);
      } else {
        const double* c = fc.hc + 30;
        r = c[0] * q[0];
#pragma unroll
        for (int k = 1; k <= 5; ++k) r = r + c[k] * (q[k] + q[-k]);
      }
      rhs[idx] = r;
      continue;
    }
    if (i >= H && i < n - H) {
      // interior row (no wrap, no closure, full order): the same
      // expressions as compact_rhs_at / the h = 5 filter row
      const double* q = in + idx;
      if (JOB == 0) {
        if (scheme == WD_C4) r = C4_CA * (q[sa] - q[-sa]);
        else r = C6_CA * (q[sa] - q[-sa]) + C6_CB * (q[2 * sa] - q[-2 * sa]);
      } else {
        const double* c = fc.hc + 30;
        r = c[0] * q[0];
#pragma unroll
        for (int k = 1; k <= 5; ++k) r = r + c[k] * (q[k * sa] + q[-k * sa]);
      }
      rhs[idx] = r;
      continue;
    }
    Line w{in + (idx - (long long)i * sa), sa, n, per, off};
    if (JOB == 0) {
      r = compact_rhs_at(w, i, n, scheme, per);
    } else {
      const int h = per ? 5 : ((i == 0 || i == n - 1) ? 0 : min(min(i, n - 1 - i), 5));
      if (h == 0) {
        r = w(i);
      } else {
        const double* c = fc.hc + h * 6;
        r = c[0] * w(i);
        for (int k = 1; k <= h; ++k) r = r + c[k] * (w(i + k) + w(i - k));
      }
    }
    rhs[idx] = r;
  }
}

// Strided axes: one thread per segment of RS consecutive rows of a line, the
// input window (RS + 2H rows) loaded once into registers, so every input
// row is read ~(RS + 2H) / RS times instead of 2H + 1 (the per-node kernel
// above read the axis-0 field 3.3x from DRAM at 1024x512x256, ncu).
// Threads with consecutive ids own consecutive lines (coalesced rows).
// Same expressions as k_line_rhs (bitwise equal).
constexpr int RS_ROWS = 16;

template <int JOB>
static __global__ void k_line_rhs_seg(const double* __restrict__ in, double* __restrict__ rhs,
                                      long long N, long long sa, int n, int per, double off,
                                      int scheme, FilterCoef fc, const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  constexpr int H = JOB == 0 ? 2 : 5;
  const int nseg = (n + RS_ROWS - 1) / RS_ROWS;
  const long long total = (N / n) * nseg;
  const bool small = N <= 0xffffffffLL;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long u, rest;
    int seg;
    if (small) {
      const unsigned ut = (unsigned)t, usa = (unsigned)sa;
      const unsigned r32 = ut / usa;
      u = ut - r32 * usa;
      const unsigned o32 = r32 / (unsigned)nseg;
      seg = (int)(r32 - o32 * (unsigned)nseg);
      rest = o32;
    } else {
      u = t % sa;
      const long long r64 = t / sa;
      seg = (int)(r64 % nseg);
      rest = r64 / nseg;
    }
    const long long base = rest * (long long)n * sa + u;  // row 0 of the line
    const int i0 = seg * RS_ROWS;
    if (i0 >= H && i0 + RS_ROWS + H <= n) {
      double v[RS_ROWS + 2 * H];
      const double* q = in + base + (long long)(i0 - H) * sa;
#pragma unroll
      for (int k = 0; k < RS_ROWS + 2 * H; ++k) v[k] = q[k * sa];
      double* o = rhs + base + (long long)i0 * sa;
#pragma unroll
      for (int r = 0; r < RS_ROWS; ++r) {
        const double* c = v + r + H;
        double x;
        if (JOB == 0) {
          if (scheme == WD_C4) x = C4_CA * (c[1] - c[-1]);
          else x = C6_CA * (c[1] - c[-1]) + C6_CB * (c[2] - c[-2]);
        } else {
          const double* hc = fc.hc + 30;
          x = hc[0] * c[0];
#pragma unroll
          for (int k = 1; k <= 5; ++k) x = x + hc[k] * (c[k] + c[-k]);
        }
        o[r * sa] = x;
      }
      continue;
    }
    const Line w{in + base, sa, n, per, off};
    for (int r = 0; r < RS_ROWS; ++r) {
      const int i = i0 + r;
      if (i >= n) break;
      double x;
      if (JOB == 0) {
        x = compact_rhs_at(w, i, n, scheme, per);
      } else {
        const int h = per ? 5 : ((i == 0 || i == n - 1) ? 0 : min(min(i, n - 1 - i), 5));
        if (h == 0) {
          x = w(i);
        } else {
          const double* c = fc.hc + h * 6;
          x = c[0] * w(i);
          for (int k = 1; k <= h; ++k) x = x + c[k] * (w(i + k) + w(i - k));
        }
      }
      rhs[base + (long long)i * sa] = x;
    }
  }
}

template <int JOB>
static __global__ void __launch_bounds__(LS_WARPS * 32, LS_MINB)
    k_line_solve(const double* __restrict__ in, double* y, double* out, Geom g, int axis,
                 int n, long long sa, TriDev T, Epi epi, const uint8_t* pin, int use_geom_pin,
                 const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  // factor rows: fact, swap, du, du2, d, rinv, z, h; then one flag per
  // forward group (any row interchange in the group)
  extern __shared__ double ls_f[];
  const long long L = g.N / n;
  double* sfact = ls_f;
  double* sswap = sfact + n;
  double* sdu = sswap + n;
  double* sdu2 = sdu + n;
  double* sd = sdu2 + n;
  double* srinv = sd + n;
  double* sz = srinv + n;
  double* sh = sz + n;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    sfact[t] = t < n - 1 ? T.fact[t] : 0.0;
    sswap[t] = t < n - 1 ? T.swap[t] : 0.0;
    sdu[t] = t < n - 1 ? T.du[t] : 0.0;
    sdu2[t] = t < n - 2 ? T.du2[t] : 0.0;
    sd[t] = T.d[t];
    srinv[t] = T.rinv[t];
    sz[t] = T.cyclic ? T.z[t] : 0.0;
    sh[t] = T.cyclic ? T.h[t] : 0.0;
  }
  int* gswap = reinterpret_cast<int*>(sh + n);
  for (int k = threadIdx.x; k * LS_U < n; k += blockDim.x) {
    int any = 0;
    for (int s2 = 0; s2 < LS_U; ++s2) {
      const int t = k * LS_U + s2;
      if (t < n - 1 && T.swap[t] != 0.0) any = 1;
    }
    gswap[k] = any;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long nwarps = (long long)gridDim.x * LS_WARPS;
  for (long long grp = (long long)blockIdx.x * LS_WARPS + wib; grp * 32 < L; grp += nwarps) {
    const long long q = grp * 32 + lane;
    if (q >= L) continue;  // no warp-collective operations below
    const long long base = line_base(g, axis, q);
    double* yl = y + base;
    // pinned nodes of this line (JOB 1): whole line on a wall face of
    // another axis, the ends on this axis' wall faces, the solid mask
    bool line_pin = false, pin_lo = false, pin_hi = false;
    if (JOB == 1 && use_geom_pin) {
      int c[kMaxDim];
      node_coords(g, base, c);
#pragma unroll
      for (int b = 0; b < kMaxDim; ++b) {
        if (b >= g.nd || b == axis) continue;
        if (c[b] == 0 && g.face[2 * b] == WD_FACE_WALL) line_pin = true;
        if (c[b] == g.n[b] - 1 && g.face[2 * b + 1] == WD_FACE_WALL) line_pin = true;
      }
      pin_lo = pick(g.face, 2 * axis) == WD_FACE_WALL;
      pin_hi = pick(g.face, 2 * axis + 1) == WD_FACE_WALL;
    }
    // ---------------- forward elimination (y in place of the rhs)
    // Software-pipelined: the loads of group k+1 are issued before the
    // recurrence of group k runs (warps issue in order, so a load consumed
    // right away would stall the chain for a full memory latency).
    double carry = yl[0];
    double hs = 0.0;
    if (T.cyclic) hs = hs + sh[0] * carry;
    const int nf = (n - 1) / LS_U;  // full forward groups (steps 0 .. nf*U-1)
    auto fload = [&](int k, double (&b)[LS_U]) {
#pragma unroll
      for (int s = 0; s < LS_U; ++s) b[s] = yl[(long long)(k * LS_U + s + 1) * sa];
    };
    auto fproc = [&](int k, const double (&b)[LS_U]) {
      if (!gswap[k]) {  // no interchange in this group (CTA-uniform branch)
#pragma unroll
        for (int s = 0; s < LS_U; ++s) {
          const int i = k * LS_U + s;
          const double yv = carry;
          carry = b[s] - sfact[i] * carry;
          if (T.cyclic) hs = hs + sh[i + 1] * b[s];
          yl[(long long)i * sa] = yv;
        }
        return;
      }
#pragma unroll
      for (int s = 0; s < LS_U; ++s) {
        const int i = k * LS_U + s;
        const double f = sfact[i];
        double yv;
        if (sswap[i] != 0.0) {
          yv = b[s];
          carry = carry - f * b[s];
        } else {
          yv = carry;
          carry = b[s] - f * carry;
        }
        if (T.cyclic) hs = hs + sh[i + 1] * b[s];
        yl[(long long)i * sa] = yv;
      }
    };
    {
      double bA[LS_U], bB[LS_U];
      if (nf > 0) fload(0, bA);
      for (int k = 0; k < nf; k += 2) {
        if (k + 1 < nf) fload(k + 1, bB);
        fproc(k, bA);
        if (k + 1 >= nf) break;
        if (k + 2 < nf) fload(k + 2, bA);
        fproc(k + 1, bB);
      }
    }
    for (int i = nf * LS_U; i < n - 1; ++i) {
      const double bv = yl[(long long)(i + 1) * sa];
      const double f = sfact[i];
      double yv;
      if (sswap[i] != 0.0) {
        yv = bv;
        carry = carry - f * bv;
      } else {
        yv = carry;
        carry = bv - f * carry;
      }
      if (T.cyclic) hs = hs + sh[i + 1] * bv;
      yl[(long long)i * sa] = yv;
    }
    yl[(long long)(n - 1) * sa] = carry;
    const double fcor = T.cyclic ? hs / T.denom : 0.0;
    // ---------------- back substitution + output (pipelined the same way;
    // the epilogue's per-node operands are fetched with the group's y)
    const bool need_acc = JOB == 0 && epi.mode == 2;
    const bool need_c = JOB == 0 && epi.mode != 0 && epi.cfield != nullptr;
    auto emit = [&](int r, double x, double accv, double cv) {
      const double xv = T.cyclic ? x - fcor * sz[r] : x;
      const long long idx = base + (long long)r * sa;
      if (JOB == 0) {
        double o = xv;
        if (epi.mode != 0) {
          const double t = (epi.cfield ? cv : epi.cscal) * xv;
          o = epi.mode == 1 ? t : accv + t;
        }
        out[idx] = o;
      } else {
        bool p;
        if (use_geom_pin)
          p = line_pin || (r == 0 && pin_lo) || (r == n - 1 && pin_hi) ||
              (g.mask != nullptr && g.mask[idx] != 0);
        else
          p = pin != nullptr && pin[idx] != 0;
        // branch, not a select: an unconditional load of in[idx] would
        // stall the in-order warp for a memory latency on every row
        if (p) out[idx] = in[idx];
        else out[idx] = xv;
      }
    };
    auto eload = [&](int r, double& accv, double& cv) {
      const long long idx = base + (long long)r * sa;
      accv = need_acc ? epi.acc[idx] : 0.0;
      cv = need_c ? epi.cfield[idx] : 0.0;
    };
    double x1, x2;
    {
      double a0, c0;
      eload(n - 1, a0, c0);
      x1 = ls_div(carry, sd[n - 1], srinv[n - 1]);
      emit(n - 1, x1, a0, c0);
      x2 = x1;
      eload(n - 2, a0, c0);
      x1 = ls_div(yl[(long long)(n - 2) * sa] - sdu[n - 2] * x2, sd[n - 2], srinv[n - 2]);
      emit(n - 2, x1, a0, c0);
    }
    // rows n-3 .. 0 in groups of U going down: group k covers rows
    // n-3-kU .. n-3-kU-U+1
    const int nbk = (n - 2) / LS_U;
    auto bload = [&](int k, double (&yv)[LS_U], double (&av)[LS_U], double (&cv)[LS_U]) {
#pragma unroll
      for (int s = 0; s < LS_U; ++s) {
        const int rr = n - 3 - k * LS_U - s;
        yv[s] = yl[(long long)rr * sa];
        eload(rr, av[s], cv[s]);
      }
    };
    auto bproc = [&](int k, const double (&yv)[LS_U], const double (&av)[LS_U],
                     const double (&cv)[LS_U]) {
#pragma unroll
      for (int s = 0; s < LS_U; ++s) {
        const int rr = n - 3 - k * LS_U - s;
        const double x = ls_div((yv[s] - sdu[rr] * x1) - sdu2[rr] * x2, sd[rr], srinv[rr]);
        x2 = x1;
        x1 = x;
        emit(rr, x, av[s], cv[s]);
      }
    };
    {
      double yA[LS_U], aA[LS_U], cA[LS_U], yB[LS_U], aB[LS_U], cB[LS_U];
      if (nbk > 0) bload(0, yA, aA, cA);
      for (int k = 0; k < nbk; k += 2) {
        if (k + 1 < nbk) bload(k + 1, yB, aB, cB);
        bproc(k, yA, aA, cA);
        if (k + 1 >= nbk) break;
        if (k + 2 < nbk) bload(k + 2, yA, aA, cA);
        bproc(k + 1, yB, aB, cB);
      }
    }
    for (int r = n - 3 - nbk * LS_U; r >= 0; --r) {
      double av, cv;
      eload(r, av, cv);
      const double x =
          ls_div((yl[(long long)r * sa] - sdu[r] * x1) - sdu2[r] * x2, sd[r], srinv[r]);
      x2 = x1;
      x1 = x;
      emit(r, x, av, cv);
    }
  }
}

// ---------------------------------------------------------------------
// FEW LONG LINES (2-D grids: BASELINE configs 1-3 have 101-1025 lines of
// 101-1025 rows).  The dgtsv recurrences are one dependency chain per line,
// and the warp-per-32-lines kernels above leave all but a handful of warps
// of the GPU empty while every step of the chain waits on a global or
// transposed-tile access (C3's axis-0 filter: 384 us for 513 lines).  Here a
// CTA owns FL lines: all its threads evaluate the right-hand sides into
// shared memory (field reads hit L2), then ONE thread per line -- lane 0 of
// its own warp, so the chains of a CTA sit on different schedulers -- runs
// the forward / backward recurrences out of shared memory with the factor
// rows prefetched in batches (off the chain), then all threads apply the
// cyclic correction, the epilogue / pinned-node restore and store.  Same
// expressions in the same order as k_line_rhs + k_line_solve (bitwise
// equal; tests/test_gpu_parity.py), one launch instead of two.
constexpr int LF_T = 256;   // threads per CTA
constexpr int LF_MAXL = 4;  // lines per CTA (one chain thread per warp)
constexpr int LF_U = 8;     // chain steps per prefetched batch

template <int JOB, class L>
__device__ __forceinline__ double line_rhs_at(const L& w, int i, int n, int scheme, int per,
                                              const FilterCoef& fc) {
  if (JOB == 0) return compact_rhs_at(w, i, n, scheme, per);
  const int h = per ? 5 : ((i == 0 || i == n - 1) ? 0 : min(min(i, n - 1 - i), 5));
  if (h == 0) return w(i);
  const double* c = fc.hc + h * 6;
  double r = c[0] * w(i);
  for (int k = 1; k <= h; ++k) r = r + c[k] * (w(i + k) + w(i - k));
  return r;
}

template <int JOB>
__device__ __forceinline__ void line_few_body(const double* __restrict__ in, double* out,
                                              const Geom& g, int axis, int n, long long sa,
                                              int per, double off, int scheme, const TriDev& T,
                                              const Epi& epi, const FilterCoef& fc,
                                              const uint8_t* pin, int use_geom_pin, int fl,
                                              int block_id) {
  extern __shared__ double lf_s[];  // [fl][n] right-hand sides -> y -> x, hs[LF_MAXL], factor rows
  const long long L = g.N / n;
  const long long q0 = (long long)block_id * fl;
  if (q0 >= L) return;
  const int nl = (int)min((long long)fl, L - q0);
  double* fcors = lf_s + (size_t)fl * n;
  // factor rows in shared memory: every operand of the chains is then an
  // LDS issued a batch ahead (global / L1 latency per batch was the bound)
  double* sfact = fcors + LF_MAXL;
  double* sswap = sfact + n;
  double* sdu = sswap + n;
  double* sdu2 = sdu + n;
  double* sd = sdu2 + n;
  double* srinv = sd + n;
  double* sh = srinv + n;
  for (int t = threadIdx.x; t < n; t += LF_T) {
    sfact[t] = t < n - 1 ? T.fact[t] : 0.0;
    sswap[t] = t < n - 1 ? T.swap[t] : 0.0;
    sdu[t] = t < n - 1 ? T.du[t] : 0.0;
    sdu2[t] = t < n - 2 ? T.du2[t] : 0.0;
    sd[t] = T.d[t];
    srinv[t] = T.rinv[t];
    sh[t] = T.cyclic ? T.h[t] : 0.0;
  }
  // ---- A. right-hand sides.  Strided lines: a thread owns a run of
  // consecutive rows of one line and slides a register window over them (one
  // L2 load per row instead of the stencil's 5 / 11); the rows whose stencil
  // leaves the line (closures, reduced filter orders, periodic wrap) and
  // contiguous lines take the per-row evaluation.  Same expressions.
  const int total = nl * n;
  constexpr int HW = JOB == 0 ? 2 : 5;  // stencil reach
  if (sa != 1 && n >= 4 * (2 * HW + 1)) {
    const int tpl = LF_T / nl;                  // threads per line
    const int ll = threadIdx.x / tpl, part = threadIdx.x - ll * tpl;
    if (ll < nl) {
      const int rows = (n + tpl - 1) / tpl;
      const int i0 = part * rows, i1 = min(n, i0 + rows);
      const long long base = line_base(g, axis, q0 + ll);
      Line w{in + base, sa, n, per, off};
      const double* q = in + base;
      double* dst = lf_s + (size_t)ll * n;
      const double* fcc = fc.hc + 30;
      int i = i0;
      // head rows near the line start
      for (; i < i1 && i < HW; ++i) dst[i] = line_rhs_at<JOB>(w, i, n, scheme, per, fc);
      if (i < i1 && i < n - HW) {
        double win[2 * HW + 1];  // w(i - HW) .. w(i + HW)
#pragma unroll
        for (int k = 0; k < 2 * HW; ++k) win[k + 1] = q[(long long)(i - HW + k) * sa];
        for (; i < i1 && i < n - HW; ++i) {
#pragma unroll
          for (int k = 0; k < 2 * HW; ++k) win[k] = win[k + 1];
          win[2 * HW] = q[(long long)(i + HW) * sa];
          double r;
          if (JOB == 0) {
            // compact interior rows (compact_rhs_at): C6 rows 1 / n-2 use the
            // C4 relation on non-periodic lines
            const double d1 = win[HW + 1] - win[HW - 1];
            if (scheme == WD_C4) r = C4_CA * d1;
            else if (!per && (i == 1 || i == n - 2)) r = 0.75 * d1;
            else r = C6_CA * d1 + C6_CB * (win[HW + 2] - win[HW - 2]);
          } else {
            r = fcc[0] * win[HW];
#pragma unroll
            for (int k = 1; k <= 5; ++k) r = r + fcc[k] * (win[HW + k] + win[HW - k]);
          }
          dst[i] = r;
        }
      }
      for (; i < i1; ++i) dst[i] = line_rhs_at<JOB>(w, i, n, scheme, per, fc);
    }
  } else {
    for (int t = threadIdx.x; t < total; t += LF_T) {
      const int ll = sa == 1 ? t / n : t % nl;
      const int i = sa == 1 ? t - ll * n : t / nl;
      const long long base = line_base(g, axis, q0 + ll);
      Line w{in + base, sa, n, per, off};
      lf_s[(size_t)ll * n + i] = line_rhs_at<JOB>(w, i, n, scheme, per, fc);
    }
  }
  __syncthreads();
  // ---- B. one chain per line: lane 0 of warp ll
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0 && wib < nl) {
    double* x = lf_s + (size_t)wib * n;
    if (n == 1) {
      x[0] = x[0] / T.d[0];
      fcors[wib] = 0.0;
    } else {
      const bool cyc = T.cyclic != 0;
      double carry = x[0];
      double hs = 0.0;
      if (cyc) hs = hs + sh[0] * carry;
      // forward elimination, software pipelined: batch k + 1 is loaded
      // before the recurrence of batch k runs
      const int nf = (n - 1) / LF_U;
      auto fload = [&](int k, double (&b)[LF_U], double (&f)[LF_U], double (&sw)[LF_U],
                       double (&hv)[LF_U]) {
#pragma unroll
        for (int u = 0; u < LF_U; ++u) {
          const int i = k * LF_U + u;
          b[u] = x[i + 1];
          f[u] = sfact[i];
          sw[u] = sswap[i];
          hv[u] = cyc ? sh[i + 1] : 0.0;
        }
      };
      auto fproc = [&](int k, const double (&b)[LF_U], const double (&f)[LF_U],
                       const double (&sw)[LF_U], const double (&hv)[LF_U]) {
        bool any = false;
#pragma unroll
        for (int u = 0; u < LF_U; ++u) any |= sw[u] != 0.0;
        if (!any) {  // no row interchange in the batch: branch-free chain
#pragma unroll
          for (int u = 0; u < LF_U; ++u) {
            x[k * LF_U + u] = carry;
            carry = b[u] - f[u] * carry;
            if (cyc) hs = hs + hv[u] * b[u];
          }
          return;
        }
#pragma unroll
        for (int u = 0; u < LF_U; ++u) {
          double yv;
          if (sw[u] != 0.0) {
            yv = b[u];
            carry = carry - f[u] * b[u];
          } else {
            yv = carry;
            carry = b[u] - f[u] * carry;
          }
          if (cyc) hs = hs + hv[u] * b[u];
          x[k * LF_U + u] = yv;
        }
      };
      {
        double bA[LF_U], fA[LF_U], sA[LF_U], hA[LF_U], bB[LF_U], fB[LF_U], sB[LF_U], hB[LF_U];
        if (nf > 0) fload(0, bA, fA, sA, hA);
        for (int k = 0; k < nf; k += 2) {
          if (k + 1 < nf) fload(k + 1, bB, fB, sB, hB);
          fproc(k, bA, fA, sA, hA);
          if (k + 1 >= nf) break;
          if (k + 2 < nf) fload(k + 2, bA, fA, sA, hA);
          fproc(k + 1, bB, fB, sB, hB);
        }
      }
      for (int i = nf * LF_U; i < n - 1; ++i) {
        const double bv = x[i + 1], f = sfact[i];
        double yv;
        if (sswap[i] != 0.0) {
          yv = bv;
          carry = carry - f * bv;
        } else {
          yv = carry;
          carry = bv - f * carry;
        }
        if (cyc) hs = hs + sh[i + 1] * bv;
        x[i] = yv;
      }
      fcors[wib] = cyc ? hs / T.denom : 0.0;
      double x1 = ls_div(carry, sd[n - 1], srinv[n - 1]);
      x[n - 1] = x1;
      double x2 = x1;
      x1 = ls_div(x[n - 2] - sdu[n - 2] * x2, sd[n - 2], srinv[n - 2]);
      x[n - 2] = x1;
      // back substitution: rows n-3 .. 0, batch k covers rows n-3-kU .. n-3-kU-U+1
      const int nbk = (n - 2) / LF_U;
      auto bload = [&](int k, double (&yv)[LF_U], double (&du)[LF_U], double (&du2)[LF_U],
                       double (&dd)[LF_U], double (&ri)[LF_U]) {
#pragma unroll
        for (int u = 0; u < LF_U; ++u) {
          const int r = n - 3 - k * LF_U - u;
          yv[u] = x[r];
          du[u] = sdu[r];
          du2[u] = sdu2[r];
          dd[u] = sd[r];
          ri[u] = srinv[r];
        }
      };
      auto bproc = [&](int k, const double (&yv)[LF_U], const double (&du)[LF_U],
                       const double (&du2)[LF_U], const double (&dd)[LF_U],
                       const double (&ri)[LF_U]) {
#pragma unroll
        for (int u = 0; u < LF_U; ++u) {
          const double xv = ls_div((yv[u] - du[u] * x1) - du2[u] * x2, dd[u], ri[u]);
          x2 = x1;
          x1 = xv;
          x[n - 3 - k * LF_U - u] = xv;
        }
      };
      {
        double yA[LF_U], aA[LF_U], cA[LF_U], dA[LF_U], rA[LF_U];
        double yB[LF_U], aB[LF_U], cB[LF_U], dB[LF_U], rB[LF_U];
        if (nbk > 0) bload(0, yA, aA, cA, dA, rA);
        for (int k = 0; k < nbk; k += 2) {
          if (k + 1 < nbk) bload(k + 1, yB, aB, cB, dB, rB);
          bproc(k, yA, aA, cA, dA, rA);
          if (k + 1 >= nbk) break;
          if (k + 2 < nbk) bload(k + 2, yA, aA, cA, dA, rA);
          bproc(k + 1, yB, aB, cB, dB, rB);
        }
      }
      for (int r = n - 3 - nbk * LF_U; r >= 0; --r) {
        const double xv = ls_div((x[r] - sdu[r] * x1) - sdu2[r] * x2, sd[r], srinv[r]);
        x2 = x1;
        x1 = xv;
        x[r] = xv;
      }
    }
  }
  __syncthreads();
  // ---- C. cyclic correction, epilogue / pinned-node restore, store
  for (int t = threadIdx.x; t < total; t += LF_T) {
    const int ll = sa == 1 ? t / n : t % nl;
    const int i = sa == 1 ? t - ll * n : t / nl;
    const long long base = line_base(g, axis, q0 + ll);
    const long long idx = base + (long long)i * sa;
    const double xs = lf_s[(size_t)ll * n + i];
    const double xv = T.cyclic ? xs - fcors[ll] * T.z[i] : xs;
    if (JOB == 0) {
      out[idx] = epi.apply(xv, idx);
    } else {
      bool p;
      if (use_geom_pin) {
        int c[kMaxDim];
        node_coords(g, idx, c);
        p = is_pinned(g, idx, c);
      } else {
        p = pin != nullptr && pin[idx] != 0;
      }
      out[idx] = p ? in[idx] : xv;
    }
  }
}

template <int JOB>
static __global__ void __launch_bounds__(LF_T)
    k_line_few(const double* __restrict__ in, double* out, Geom g, int axis, int n, long long sa,
               int per, double off, int scheme, TriDev T, Epi epi, FilterCoef fc,
               const uint8_t* pin, int use_geom_pin, int fl, const Status* st) {
  pdl_trigger();
  pdl_wait();
  if (st && st->state != WD_STATE_RUNNING) return;
  line_few_body<JOB>(in, out, g, axis, n, sa, per, off, scheme, T, epi, fc, pin, use_geom_pin, fl,
                     blockIdx.x);
}

// Several independent compact-derivative passes in one launch (blockIdx.y =
// pass): the axes of a gradient, or the terms of a divergence, whose chains
// then run side by side instead of one launch after another.  Plain
// epilogue (out = D); k_div_combine sums divergence terms afterwards.
struct LineFewJobs {
  const double* in[4];
  double* out[4];
  int axis[4];
  TriDev T[4];
  int count;
};
static __global__ void __launch_bounds__(LF_T)
    k_line_few_multi(LineFewJobs jobs, Geom g, int scheme, int fl, const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  const int j = blockIdx.y;  // select chains, not indexing: the struct stays in param space
  const int axis = pick(jobs.axis, j);
  const int n = pick(g.n, axis);
  const Epi plain{0, nullptr, nullptr, 0.0};
  FilterCoef fc;  // unused by JOB 0
  const TriDev T = pick(jobs.T, j);
  line_few_body<0>(pick(jobs.in, j), pick(jobs.out, j), g, axis, n, pick(g.s, axis),
                   pick(g.per, axis), 0.0, scheme, T, plain, fc, nullptr, 0, fl, blockIdx.x);
}

__host__ __forceinline__ size_t line_few_smem(int n, int fl) {
  return ((size_t)fl * n + LF_MAXL + (size_t)7 * n) * sizeof(double);
}

__host__ __forceinline__ size_t line_solve_smem(int n) {
  return (size_t)8 * n * sizeof(double) + (size_t)((n + LS_U - 1) / LS_U) * sizeof(int);
}
constexpr size_t kLineSolveMaxSmem = 200 * 1024;

// Contiguous lines (the last axis, stride 1): the same recurrences, with every
// global access transposed through per-warp shared tiles of 32 rows x 32
// lines.  With lane = line and stride-1 lines, a direct access by the warp
// touches 32 scattered sectors per row (8 of 32 bytes used, partial-sector
// stores); staged, each tile row is one 256-byte run of one line.  Tiles are
// filled with cp.async (no registers, the next chunk's rows in flight while
// the current chunk's recurrence runs): y double-buffered, and the epilogue
// operands (acc, c) of the back substitution issued one chunk ahead.  The
// right-hand side stays in k_line_rhs: evaluated inside this latency-bound
// chain (one resident CTA per SM) it made every axis slower (measured).
// Arithmetic and its order are those of k_line_solve (bitwise equal).
constexpr int LT_P = 33;                     // padded tile row (doubles)
#ifndef WD_LT_R
#define WD_LT_R 32
#endif
constexpr int LT_R = WD_LT_R;                // rows per chunk (<= 32)
constexpr int LT_TILE = LT_R * LT_P;         // doubles per tile
constexpr int LT_WARP = (LT_EPI ? 4 : 2) * LT_TILE + 64;  // y[2], (acc, c), fcor[32], line pin[32]

__host__ __forceinline__ size_t line_solve_t_smem(int n) {
  return line_solve_smem(n) + (size_t)LS_WARPS * LT_WARP * sizeof(double) + 16;
}

__device__ __forceinline__ void lt_cp8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void lt_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void lt_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

#ifndef WD_LT_MINB
#define WD_LT_MINB 1
#endif
template <int JOB>
static __global__ void __launch_bounds__(LS_WARPS * 32, WD_LT_MINB)
    k_line_solve_t(const double* __restrict__ in, double* y, double* out, Geom g, int axis, int n,
                   long long sa, TriDev T, Epi epi, const uint8_t* pin, int use_geom_pin,
                   const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  extern __shared__ double ls_f[];
  const long long L = g.N / n;
  const bool contig = sa == 1;
  double* sfact = ls_f;
  double* sswap = sfact + n;
  double* sdu = sswap + n;
  double* sdu2 = sdu + n;
  double* sd = sdu2 + n;
  double* srinv = sd + n;
  double* sz = srinv + n;
  double* sh = sz + n;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    sfact[t] = t < n - 1 ? T.fact[t] : 0.0;
    sswap[t] = t < n - 1 ? T.swap[t] : 0.0;
    sdu[t] = t < n - 1 ? T.du[t] : 0.0;
    sdu2[t] = t < n - 2 ? T.du2[t] : 0.0;
    sd[t] = T.d[t];
    srinv[t] = T.rinv[t];
    sz[t] = T.cyclic ? T.z[t] : 0.0;
    sh[t] = T.cyclic ? T.h[t] : 0.0;
  }
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* wbase = sh + n + 2 + wib * LT_WARP;
  double* ta = wbase + 2 * LT_TILE;
  double* tc = wbase + 3 * LT_TILE;
  double* sfc = wbase + (LT_EPI ? 4 : 2) * LT_TILE;
  double* slp = sfc + 32;
  __syncthreads();
  const bool need_acc = JOB == 0 && epi.mode == 2;
  const bool need_c = JOB == 0 && epi.mode != 0 && epi.cfield != nullptr;
  const bool pin_lo = JOB == 1 && use_geom_pin && pick(g.face, 2 * axis) == WD_FACE_WALL;
  const bool pin_hi = JOB == 1 && use_geom_pin && pick(g.face, 2 * axis + 1) == WD_FACE_WALL;
  const long long nwarps = (long long)gridDim.x * LS_WARPS;
  for (long long grp = (long long)blockIdx.x * LS_WARPS + wib; grp * 32 < L; grp += nwarps) {
    const long long q0 = grp * 32;
    const int nl = (int)min(32LL, L - q0);
    const bool act = lane < nl;
    // contiguous lines: line j starts at b0 + j n; strided: this lane's line
    const long long b0 = contig ? q0 * n : 0;
    const long long mybase =
        contig ? b0 + (long long)lane * n : line_base(g, axis, q0 + (act ? lane : 0));
    double* yb = y + b0;
    // rows [r, r + cnt) of the block's lines -> tile[row - r][line]
    auto fetch = [&](double* tile, const double* src, int r, int cnt) {
      if (contig) {
        if (lane < cnt) {
          const double* s0 = src + b0 + r + lane;
#pragma unroll 8
          for (int j = 0; j < nl; ++j) lt_cp8(tile + lane * LT_P + j, s0 + (long long)j * n);
        }
      } else if (act) {
        const double* s0 = src + mybase + (long long)r * sa;
#pragma unroll 8
        for (int t = 0; t < cnt; ++t) lt_cp8(tile + t * LT_P + lane, s0 + (long long)t * sa);
      }
    };
    if (JOB == 1 && use_geom_pin) {
      bool lp = false;
      if (act) {
        int c[kMaxDim];
        node_coords(g, mybase, c);
#pragma unroll
        for (int b = 0; b < kMaxDim; ++b) {
          if (b >= g.nd || b == axis) continue;
          if (c[b] == 0 && g.face[2 * b] == WD_FACE_WALL) lp = true;
          if (c[b] == g.n[b] - 1 && g.face[2 * b + 1] == WD_FACE_WALL) lp = true;
        }
      }
      slp[lane] = lp ? 1.0 : 0.0;
    }
    // ---------------- forward elimination: chunk k = steps [r0, r0 + cnt),
    // b = rhs rows r0 + 1 .. r0 + cnt in tile slots 0 .. cnt-1, y rows
    // r0 .. r0 + cnt - 1 left in the same slots
    double carry = act ? y[mybase] : 0.0;
    double hs = 0.0;
    if (T.cyclic) hs = hs + sh[0] * carry;
    fetch(wbase, y, 1, min(LT_R, n - 1));
    lt_commit();
    for (int r0 = 0, k = 0; r0 < n - 1; r0 += LT_R, ++k) {
      const int cnt = min(LT_R, n - 1 - r0);
      double* cur = wbase + (k & 1) * LT_TILE;
      lt_wait<0>();
      __syncwarp();
      if (r0 + LT_R < n - 1)
        fetch(wbase + ((k + 1) & 1) * LT_TILE, y, r0 + LT_R + 1, min(LT_R, n - 1 - (r0 + LT_R)));
      lt_commit();
      auto step = [&](int t) {
        const int i = r0 + t;
        const double b = cur[t * LT_P + lane];
        const double f = sfact[i];
        double yv;
        if (sswap[i] != 0.0) {
          yv = b;
          carry = carry - f * b;
        } else {
          yv = carry;
          carry = b - f * carry;
        }
        if (T.cyclic) hs = hs + sh[i + 1] * b;
        cur[t * LT_P + lane] = yv;
      };
      // no row interchange in the chunk (every row but 1 and n-2 of the
      // compact matrices): branch-free body, the carry update as in the
      // no-swap case of step()
      bool anysw = false;
      for (int t = 0; t < cnt; ++t) anysw |= sswap[r0 + t] != 0.0;
      if (cnt == LT_R && !anysw && !T.cyclic) {
#pragma unroll 8
        for (int t = 0; t < LT_R; ++t) {
          const double b = cur[t * LT_P + lane];
          const double yv = carry;
          carry = b - sfact[r0 + t] * carry;
          cur[t * LT_P + lane] = yv;
        }
      } else if (cnt == LT_R) {
#pragma unroll 8
        for (int t = 0; t < LT_R; ++t) step(t);
      } else {
        for (int t = 0; t < cnt; ++t) step(t);
      }
      __syncwarp();
      if (contig) {
        if (lane < cnt) {
          double* d0 = yb + r0 + lane;
#pragma unroll 8
          for (int j = 0; j < nl; ++j) d0[(long long)j * n] = cur[lane * LT_P + j];
        }
      } else if (act) {
        double* d0 = y + mybase + (long long)r0 * sa;
#pragma unroll 8
        for (int t = 0; t < cnt; ++t) d0[(long long)t * sa] = cur[t * LT_P + lane];
      }
      __syncwarp();
    }
    lt_wait<0>();
    if (act) y[mybase + (long long)(n - 1) * sa] = carry;
    sfc[lane] = T.cyclic ? hs / T.denom : 0.0;
    __syncwarp();
    // ---------------- back substitution, chunks [r0, rt) going down.  Copy
    // groups in flight: y of the next chunk (double buffer) and the epilogue
    // operands of the current one, so wait_group 1 releases the older.
    double x1 = 0.0, x2 = 0.0;
    auto fetch_epi = [&](int r0, int cnt) {
      if (LT_EPI && need_acc) fetch(ta, epi.acc, r0, cnt);
      if (LT_EPI && need_c) fetch(tc, epi.cfield, r0, cnt);
    };
    {
      const int r0 = max(0, n - LT_R);
      fetch(wbase, y, r0, n - r0);
      lt_commit();
      fetch_epi(r0, n - r0);
      lt_commit();
    }
    for (int rt = n, k = 0; rt > 0; rt -= LT_R, ++k) {
      const int r0 = max(0, rt - LT_R);
      const int cnt = rt - r0;
      double* cur = wbase + (k & 1) * LT_TILE;
      lt_wait<1>();  // y of this chunk
      __syncwarp();
      if (r0 > 0) {
        const int r0n = max(0, r0 - LT_R);
        fetch(wbase + ((k + 1) & 1) * LT_TILE, y, r0n, r0 - r0n);
      }
      lt_commit();
      int r = rt - 1;
      if (r == n - 1) {  // the last two rows first, then a branch-free unrolled body
        const double x = ls_div(cur[(r - r0) * LT_P + lane], sd[n - 1], srinv[n - 1]);
        x2 = x1;
        x1 = x;
        cur[(r - r0) * LT_P + lane] = x;
        --r;
      }
      if (r == n - 2 && r >= r0) {
        const double x = ls_div(cur[(r - r0) * LT_P + lane] - sdu[n - 2] * x1, sd[n - 2],
                                srinv[n - 2]);
        x2 = x1;
        x1 = x;
        cur[(r - r0) * LT_P + lane] = x;
        --r;
      }
#pragma unroll 8
      for (; r >= r0; --r) {
        const int t = r - r0;
        const double x = ls_div((cur[t * LT_P + lane] - sdu[r] * x1) - sdu2[r] * x2, sd[r], srinv[r]);
        x2 = x1;
        x1 = x;
        cur[t * LT_P + lane] = x;
      }
      lt_wait<1>();  // epilogue operands of this chunk
      __syncwarp();
      // node (line j, row r) from tile slot tj
      auto emit = [&](int j, int r, int tj, long long idx) {
        const double x = cur[tj];
        const double xv = T.cyclic ? x - sfc[j] * sz[r] : x;
        if (JOB == 0) {
          double o = xv;
          if (epi.mode != 0) {
            const double cv = need_c ? (LT_EPI ? tc[tj] : epi.cfield[idx]) : epi.cscal;
            const double tt = cv * xv;
            o = epi.mode == 1 ? tt : (need_acc ? (LT_EPI ? ta[tj] : epi.acc[idx]) : 0.0) + tt;
          }
          out[idx] = o;
        } else {
          bool p;
          if (use_geom_pin)
            p = slp[j] != 0.0 || (r == 0 && pin_lo) || (r == n - 1 && pin_hi) ||
                (g.mask != nullptr && g.mask[idx] != 0);
          else
            p = pin != nullptr && pin[idx] != 0;
          out[idx] = p ? in[idx] : xv;
        }
      };
      if (contig) {
        if (lane < cnt) {
          const int r = r0 + lane;
#pragma unroll 4
          for (int j = 0; j < nl; ++j) emit(j, r, lane * LT_P + j, b0 + (long long)j * n + r);
        }
      } else if (act) {
#pragma unroll 4
        for (int t = 0; t < cnt; ++t)
          emit(lane, r0 + t, t * LT_P + lane, mybase + (long long)(r0 + t) * sa);
      }
      __syncwarp();
      if (r0 > 0) {
        const int r0n = max(0, r0 - LT_R);
        fetch_epi(r0n, r0 - r0n);
      }
      lt_commit();
    }
    lt_wait<0>();
    __syncwarp();
  }
}

}  // namespace wd
