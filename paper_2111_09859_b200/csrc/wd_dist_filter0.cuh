// Partitioned axis-0 filter of the slab-decomposed fast path (wd_dist.cuh,
// SolveConfig.arith = "fast"): ONE kernel over the rank's rows, ONE all_gather
// of three doubles per line, one pointwise fix-up.
//
// The axis-0 lines are split over the P ranks (rank q owns global rows
// [lo, hi) = [q nl, (q + 1) nl)).  The implicit filter (operators.py:305-352,
// cyclic by Sherman-Morrison, oracle/wd.py:cyclic_apply) is the LU solve
//     y_i = rhs_i - fm_i y_{i-1},   x_i = y_i / d_i - g_i x_{i+1},
//     x <- x - (h . rhs / denom) z,
// whose recurrences are affine in their carries.  With y', x' the rank-local
// solves started from zero carries,
//     x_r = x'_r + cf W_r + cb Qp_r - f z_r,
// where cf = y_{lo-1} and cb = x_{hi} are the true carries, Pp_r =
// prod_{t=lo..r}(-fm_t), W the backward solve of Pp_r / d_r from zero and
// Qp_r = prod_{t=r..hi-1}(-g_t) -- all field independent (host tables).  The
// carries follow from every rank's (y'_{hi-1}, x'_{lo}, partial h.rhs):
//     cf(0) = 0,      cf(q+1) = Yend(q) + Pblk(q) cf(q),
//     cb(P-1) = 0,    cb(q-1) = Xfirst(q) + cf(q) Wfirst(q) + cb(q) Qblk(q).
// k_f0_local: a CTA stages 16 lines x (nl + 10) rows (5 ghost rows per side
// straight from the slab's ghost planes) with cp.async, splits each line's
// rows into S segments of MM rows and solves both recurrences as the
// segmented affine scan of wd_filter_scan.cuh (the next tile's load is in
// flight during the carry / back-substitution / store phases); 2 fp64 words
// per node of HBM traffic, like the single-GPU sweep.  k_f0_fix applies the
// correction in place (2 words).  The previous three-phase version moved 7
// words and needed two all_gathers and a second pass over the ghost planes.
// Same linear system as the single-GPU scan filter; round-off-level
// differences (tests/test_gpu_dist.py).
#pragma once

#include "wd_filter_scan.cuh"

namespace wd {

constexpr int F0_L = 16;     // lines per CTA (128-byte rows)
constexpr int F0_SMAX = 32;  // segments per line (threads = F0_L * S <= 512)

struct F0Tables {
  // local tables, nl entries each: fm, h, Pseg, g, rinv, Qseg | W, Qp, z
  const double* tab = nullptr;
  const double* blk = nullptr;  // per rank q: Pblk, Qblk, Wfirst
  int P = 1, rank = 0, nl = 0;
  int m = 0, S = 0;             // rows per segment, segments per line
  double rden = 0.0;            // 1 / cyclic Sherman-Morrison denominator
};

struct F0Args {
  const double* in;  // ghosted slab (nl + 2G, n1, n2), ghosts filled
  double* out;       // x': interior layout (nl, n1, n2)
  double* mine;      // [3][lines]: y'_{hi-1}, x'_{lo}, sum h rhs
  int n1, n2, G;
  F0Tables T;
  FilterCoef fc;
  const Status* st;
};

// MM > 0: every segment has exactly MM rows, all of y' in registers;
// MM = 0: runtime m <= 32 rows per segment (any nl), y' kept in shared memory.
template <int MM>
__global__ void __launch_bounds__(F0_L* F0_SMAX) k_f0_local(F0Args a) {
  if (a.st && a.st->state != WD_STATE_RUNNING) return;
  extern __shared__ double f0_smem[];
  const int nl = a.T.nl, S = a.T.S, m = MM > 0 ? MM : a.T.m;
  const int NT = F0_L * S;
  const double* fm = f0_smem;
  const double* hh = fm + nl;
  const double* Ps = hh + nl;
  const double* gg = Ps + nl;
  const double* ri = gg + nl;
  const double* Qs = ri + nl;
  double* tile = f0_smem + ((6 * nl + 3) & ~3);
  const int NR = nl + 2 * FS_G;
  double* Yend = tile + NR * F0_L;
  double* Xst = Yend + F0_L * F0_SMAX;
  double* Hs = Xst + F0_L * F0_SMAX;
  double* ysm = Hs + F0_L * F0_SMAX;  // MM == 0 only: (nl, F0_L)
  const int tid = threadIdx.x;
  for (int t = tid; t < 6 * nl; t += NT) f0_smem[t] = a.T.tab[t];

  const int l = tid % F0_L, s = tid / F0_L;
  const int r0 = s * m;
  const int cnt = max(0, min(m, nl - r0));
  const long long s0 = (long long)a.n1 * a.n2;
  const long long lines = s0;
  const int nb = (a.n2 + F0_L - 1) / F0_L;
  const long long groups = (long long)a.n1 * nb;
  const bool vec16 = (a.n2 % 2) == 0;  // F0_L even -> every tile base is even

  auto tile_of = [&](long long q, long long& base, int& nlines) {
    const long long j = q / nb;
    const int k0 = (int)(q - j * nb) * F0_L;
    nlines = min(F0_L, a.n2 - k0);
    base = j * a.n2 + k0;
  };
  // rows -5 .. nl+4 of the tile's lines: ghosts are real neighbour rows
  auto load = [&](long long base, int nlines) {
    const double* in = a.in + (long long)(a.G - FS_G) * s0 + base;
    if (vec16) {
      const int c = tid & 7;
      const int bytes = 2 * c < nlines ? (2 * c + 1 < nlines ? 16 : 8) : 0;
      for (int r = tid >> 3; r < NR; r += NT / 8)
        cp_async16(tile + r * F0_L + 2 * c, in + (long long)r * s0 + 2 * c, bytes);
    } else {
      for (int r = s; r < NR; r += S) cp_async8(tile + r * F0_L + l, in + (long long)r * s0 + l, l < nlines);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  long long q = blockIdx.x, base = 0;
  int nlines = 0;
  if (q < groups) {
    tile_of(q, base, nlines);
    load(base, nlines);
  }
  const double* tl = tile + l + (r0 + FS_G) * F0_L;  // row r0 of my line
  for (; q < groups; q += gridDim.x) {
    cp_async_wait_all();
    __syncthreads();
    // ---- 1. right-hand side (full order: the global line is cyclic) and the
    // segment's forward recurrence from zero
    double yv[MM > 0 ? MM : 1];
    double yp = 0.0, hs = 0.0;
    if constexpr (MM > 0) {
      double ww[MM + 10];
#pragma unroll
      for (int k = 0; k < 10; ++k) ww[k] = tl[(k - 5) * F0_L];
#pragma unroll
      for (int rr = 0; rr < MM; ++rr) {
        ww[rr + 10] = tl[(rr + 5) * F0_L];
        const double rhs = fs_rhs5(ww + rr, a.fc);
        yp = fma(-fm[r0 + rr], yp, rhs);
        hs = fma(hh[r0 + rr], rhs, hs);
        yv[rr] = yp;
      }
    } else {
      for (int rr = 0; rr < cnt; ++rr) {
        double ww[11];
#pragma unroll
        for (int k = 0; k < 11; ++k) ww[k] = tl[(rr + k - 5) * F0_L];
        const double rhs = fs_rhs5(ww, a.fc);
        yp = fma(-fm[r0 + rr], yp, rhs);
        hs = fma(hh[r0 + rr], rhs, hs);
        ysm[(r0 + rr) * F0_L + l] = yp;
      }
    }
    Yend[tid] = yp;
    Hs[tid] = hs;
    __syncthreads();
    // the staged input is consumed: the next tile's rows can land now
    long long nbase = 0;
    int nnl = 0;
    if (q + gridDim.x < groups) {
      tile_of(q + gridDim.x, nbase, nnl);
      load(nbase, nnl);
    }
    // ---- 2. forward carry within the rank, fix-up, local back substitution
    double c = 0.0;
    for (int t = 0; t < s; ++t) c = fma(Ps[min(t * m + m, nl) - 1], c, Yend[t * F0_L + l]);
    double xn = 0.0, ylast = 0.0;
    if constexpr (MM > 0) {
#pragma unroll
      for (int rr = MM - 1; rr >= 0; --rr) {
        const double y = fma(Ps[r0 + rr], c, yv[rr]);
        if (rr == MM - 1) ylast = y;
        xn = fma(-gg[r0 + rr], xn, y * ri[r0 + rr]);
        yv[rr] = xn;
      }
    } else {
      for (int rr = cnt - 1; rr >= 0; --rr) {
        const double y = fma(Ps[r0 + rr], c, ysm[(r0 + rr) * F0_L + l]);
        if (rr == cnt - 1) ylast = y;
        xn = fma(-gg[r0 + rr], xn, y * ri[r0 + rr]);
        ysm[(r0 + rr) * F0_L + l] = xn;
      }
    }
    Xst[tid] = xn;
    __syncthreads();
    // ---- 3. backward carry within the rank, store x' and the line's exports
    double c2 = 0.0;
    for (int t = S - 1; t > s; --t)
      if (t * m < nl) c2 = fma(Qs[t * m], c2, Xst[t * F0_L + l]);
    if (l < nlines) {
      double* po = a.out + base + l + (long long)r0 * s0;
      double x0 = 0.0;
      if constexpr (MM > 0) {
#pragma unroll
        for (int rr = 0; rr < MM; ++rr) {
          const double x = fma(Qs[r0 + rr], c2, yv[rr]);
          if (rr == 0) x0 = x;
          __stcs(po, x);
          po += s0;
        }
      } else {
        for (int rr = 0; rr < cnt; ++rr) {
          const double x = fma(Qs[r0 + rr], c2, ysm[(r0 + rr) * F0_L + l]);
          if (rr == 0) x0 = x;
          __stcs(po, x);
          po += s0;
        }
      }
      const long long line = base + l;
      if (cnt > 0 && r0 + cnt == nl) a.mine[line] = ylast;
      if (s == 0) {
        a.mine[lines + line] = x0;
        double hsum = 0.0;
        for (int t = 0; t < S; ++t) hsum += Hs[t * F0_L + l];
        a.mine[2 * lines + line] = hsum;
      }
    }
    base = nbase;
    nlines = nnl;
    // Yend / Xst / Hs / ysm of this tile are rewritten only after the next
    // iteration's first __syncthreads (every thread is past its reads then)
  }
}

inline size_t f0_smem_bytes(int nl, bool generic) {
  const size_t NR = (size_t)nl + 2 * FS_G;
  return (((size_t)6 * nl + 3) & ~(size_t)3) * 8 + NR * F0_L * 8 + 3 * F0_L * F0_SMAX * 8 +
         (generic ? (size_t)nl * F0_L * 8 : 0);
}

// Per-line carries of this rank from the gathered [P][3][lines] exports:
// coef[0] = cf (y of row lo - 1), coef[1] = cb (x of row hi), coef[2] = f.
__global__ void k_f0_carry(const double* __restrict__ all, double* __restrict__ coef,
                           long long lines, F0Tables T, const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < lines;
       q += (long long)gridDim.x * blockDim.x) {
    double cf = 0.0, cfr = 0.0, hsum = 0.0;
    double cfq[8];  // cf(q) per rank (P <= 8)
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      if (p < T.P) {
        cfq[p] = cf;
        if (p == T.rank) cfr = cf;
        const double* g = all + (3LL * p) * lines + q;
        hsum += g[2 * lines];
        cf = fma(T.blk[3 * p], cf, g[0]);
      }
    }
    double cb = 0.0;
#pragma unroll
    for (int p = 7; p >= 1; --p) {
      if (p < T.P && p > T.rank) {
        const double* g = all + (3LL * p) * lines + q;
        cb = fma(T.blk[3 * p + 1], cb, fma(cfq[p], T.blk[3 * p + 2], g[lines]));
      }
    }
    coef[q] = cfr;
    coef[lines + q] = cb;
    coef[2 * lines + q] = hsum * T.rden;
  }
}

// x = x' + cf W_r + cb Qp_r - f z_r, in place: one thread per line and
// F0_FR rows (grid.y), the rows' loads issued together
constexpr int F0_FR = 8;
__global__ void __launch_bounds__(256) k_f0_fix(double* x, const double* __restrict__ coef, int nl,
                                                long long lines, F0Tables T, const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  const double* Wt = T.tab + 6 * nl;
  const double* Qp = Wt + nl;
  const double* zz = Qp + nl;
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= lines) return;
  const int r0 = blockIdx.y * F0_FR;
  const double cf = coef[q], cb = coef[lines + q], f = coef[2 * lines + q];
  double* px = x + q + (long long)r0 * lines;
  double v[F0_FR];
#pragma unroll
  for (int k = 0; k < F0_FR; ++k)
    if (r0 + k < nl) v[k] = __ldcs(px + (long long)k * lines);
#pragma unroll
  for (int k = 0; k < F0_FR; ++k)
    if (r0 + k < nl) {
      double t = fma(cf, __ldg(Wt + r0 + k), v[k]);
      t = fma(cb, __ldg(Qp + r0 + k), t);
      t = fma(-f, __ldg(zz + r0 + k), t);
      __stcs(px + (long long)k * lines, t);
    }
}

}  // namespace wd
