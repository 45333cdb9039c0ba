// Implicit-filter sweep along one axis (operators.py:305-352) for the fused
// 3-D path, in LAPACK dgtsv elimination order (no row interchanges occur
// for the filter matrix) -- bit-identical to the
// generic k_filter / the reference.
//
// One thread owns one grid line.  Axes 0/1: consecutive threads own
// consecutive k, so every row access of a warp is one coalesced 256-byte
// segment; axis 2 (contiguous lines): consecutive threads own consecutive
// j and each lane reads its own line sequentially (one 32-byte sector per
// four rows, served from L1).
//
// Checkpointed two-pass solve (no scratch field):
//   pass 1 streams the line forward (11-point right-hand side from a
//          register window, y_i = r_i - f_{i-1} y_{i-1}) and keeps only
//          y at the last row of every 16-row block in shared memory;
//   pass 2 walks the blocks backwards, recomputes the block's y from its
//          checkpoint (identical operations -> identical bits) and runs the
//          back substitution x_i = (y_i - du_i x_{i+1}) / d_i on it.
// HBM traffic: the input is read twice and the output written once
// (+ phi once for the fused convergence reduction on the last axis); all
// lines are in flight at once, so the latency of the recurrences is hidden.
//
// Periodic lines (EXTENSION): Sherman-Morrison with f = (h . r) / denom,
// h = B^-1 v accumulated in pass 1 (oracle/wd.py:cyclic_apply), so the
// correction x - f z is applied inside pass 2.
//
// Division: x = s / d is evaluated as a correctly rounded quotient from the
// precomputed reciprocal r = RN(1/d) (Markstein: q0 = s*r,
// e = fma(-q0, d, s), q = fma(e, r, q0)), equal to IEEE s / d; the parity
// tests check bit equality with the reference.
#pragma once

#include "wd_kernels.cuh"

namespace wd {

constexpr int FB = 16;  // rows per checkpoint block

struct SweepArgs {
  const double* in;
  double* out;
  int n;               // line length
  int axis;            // 0, 1, 2
  int n0, n1, n2;
  long long s0;        // n1 * n2
  int per;
  // factor (dgtsv order, no interchanges) + cyclic correction
  const double* fact;  // n
  const double* du;    // n
  const double* d;     // n
  const double* rinv;  // n, RN(1/d)
  const double* z;     // n (cyclic)
  const double* h;     // n (cyclic)
  double denom;
  FilterCoef fc;
  // fused convergence reduction (last axis)
  const double* A;     // nullptr -> no reduction
  Status* st;
  // slab decomposition (scan form, last sweep): rank-separable correction of
  // the partitioned axis-0 filter, added on the way out (wd_dist_filter0.cuh)
  const double* fixc = nullptr;    // [3][n1 n2] filtered per-line coefficients
  const double* fixrow = nullptr;  // [3][n0] per-plane factors W, Qp, z
};

__device__ __forceinline__ double div_rn(double s, double d, double r) {
  const double q0 = s * r;
  const double e = fma(-q0, d, s);
  return fma(e, r, q0);
}

// filter RHS for row r from the window (w[5] = row r): order of
// _filter_rhs_row (operators.py:298-302).
__device__ __forceinline__ double filt_rhs(const double* w, int h, const FilterCoef& fc) {
  if (h == 0) return w[5];
  const double* c = fc.hc + h * 6;
  double v = c[0] * w[5];
#pragma unroll
  for (int k = 1; k <= 5; ++k)
    if (k <= h) v = v + c[k] * (w[5 + k] + w[5 - k]);
  return v;
}
__device__ __forceinline__ double filt_rhs5(const double* w, const FilterCoef& fc) {
  const double* c = fc.hc + 30;
  return c[0] * w[5] + c[1] * (w[6] + w[4]) + c[2] * (w[7] + w[3]) + c[3] * (w[8] + w[2]) +
         c[4] * (w[9] + w[1]) + c[5] * (w[10] + w[0]);
}

// Rows [r0, r0+16) of the warp's 32 lines -> v[s] (lane = line).  Axes
// 0/1: direct coalesced loads.  Axis 2: 16 loads of two 128-byte line
// segments each, transposed through the warp's 32x17 shared tile.
template <bool CONTIG>
__device__ __forceinline__ void sw_rows(const double* __restrict__ in, long long lbase,
                                        long long gbase, long long rstride, long long lstride,
                                        int nl, int n, int per, int r0, double (*T)[17], int lane,
                                        double* v) {
  if (CONTIG) {
    int r = r0 + (lane & 15);
    bool ok = true;
    if (r < 0 || r >= n) {
      if (per) {
        while (r < 0) r += n;
        while (r >= n) r -= n;
      } else {
        ok = false;
      }
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int m = 2 * q + (lane >> 4);
      T[m][lane & 15] = (ok && m < nl) ? __ldcs(in + gbase + (long long)m * lstride + r) : 0.0;
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < 16; ++s) v[s] = T[lane][s];
    __syncwarp();
  } else {
    if (r0 >= 0 && r0 + 16 <= n) {  // in range: no wrap, no bounds
      const double* p = in + lbase + (long long)r0 * rstride;
#pragma unroll
      for (int s = 0; s < 16; ++s) v[s] = __ldcs(p + (long long)s * rstride);
    } else {
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        int r = r0 + s;
        bool ok = true;
        if (per) {
          while (r < 0) r += n;
          while (r >= n) r -= n;
        } else {
          ok = r >= 0 && r < n;
        }
        v[s] = ok ? __ldcs(in + lbase + (long long)r * rstride) : 0.0;
      }
    }
  }
}

// L2 prefetch of rows [r0, r0+16) of the lane's line (in range only):
// the sweep consumes each 16-row block right after loading it, so blocks
// are prefetched SW_PF blocks ahead to keep HBM latency off the recurrence.
constexpr int SW_PF = 2;
template <bool CONTIG>
__device__ __forceinline__ void sw_prefetch(const double* __restrict__ in, long long lbase,
                                            long long rstride, int n, int r0) {
  if (r0 < 0 || r0 + 16 > n) return;
  const double* p = in + lbase + (long long)r0 * rstride;
  if (CONTIG) {  // the lane's 16 rows are 128 contiguous bytes
    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p + 15));
  } else {
#pragma unroll
    for (int s = 0; s < 16; ++s) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p + s * rstride));
  }
}

template <bool CONTIG>
__global__ void __launch_bounds__(128) k_filter_sweep(SweepArgs a) {
  if (a.st->state != WD_STATE_RUNNING) return;
  extern __shared__ double sw_smem[];
  const int n = a.n;
  const int nb = (n + FB - 1) / FB;
  double* sfact = sw_smem;
  double* sdu = sfact + n;
  double* sd = sdu + n;
  double* srinv = sd + n;
  double* sz = srinv + n;
  double* sh = sz + n;
  double* ck = sh + n;  // [nb][blockDim.x]
  double(*tiles)[32][17] = reinterpret_cast<double(*)[32][17]>(ck + (size_t)nb * blockDim.x);
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    sfact[t] = a.fact[t];
    sdu[t] = a.du[t];
    sd[t] = a.d[t];
    srinv[t] = a.rinv[t];
    sz[t] = a.per ? a.z[t] : 0.0;
    sh[t] = a.per ? a.h[t] : 0.0;
  }
  __syncthreads();
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  double(*T)[17] = tiles[wib];
  // a warp owns 32 lines: consecutive k (axes 0/1) or consecutive j (axis 2)
  long long groups, per_row_blk, rstride, lstride;
  int fast_n;
  if (a.axis == 0) {
    fast_n = a.n2;
    per_row_blk = (a.n2 + 31) / 32;
    groups = (long long)a.n1 * per_row_blk;
    rstride = a.s0;
    lstride = 1;
  } else if (a.axis == 1) {
    fast_n = a.n2;
    per_row_blk = (a.n2 + 31) / 32;
    groups = (long long)a.n0 * per_row_blk;
    rstride = a.n2;
    lstride = 1;
  } else {
    fast_n = a.n1;
    per_row_blk = (a.n1 + 31) / 32;
    groups = (long long)a.n0 * per_row_blk;
    rstride = 1;
    lstride = a.n2;
  }
  const int gw = blockIdx.x * (blockDim.x >> 5) + wib;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  const int per = a.per;
  double md = 0.0, ma = 0.0;
  int bad = 0;
  for (long long g = gw; g < groups; g += nwarps) {
    const long long outer = g / per_row_blk;
    const int blk = (int)(g % per_row_blk);
    const int inner0 = blk * 32;
    const int nl = min(32, fast_n - inner0);
    const bool valid = lane < nl;
    long long gbase;  // element (row 0) of the group's first line
    if (a.axis == 0) gbase = outer * a.n2 + inner0;
    else if (a.axis == 1) gbase = outer * a.s0 + inner0;
    else gbase = outer * a.s0 + (long long)inner0 * a.n2;
    const long long lbase = gbase + (valid ? lane : 0) * lstride;
    // ---------------- pass 1: forward elimination, checkpoints
    // u[q] = row 16b - 5 + q; 10 rows carried between blocks, 16 loaded
    double u[FB + 10];
    {
      double v[16];
      sw_rows<CONTIG>(a.in, lbase, gbase, rstride, lstride, nl, n, per, -5, T, lane, v);
#pragma unroll
      for (int q = 0; q < 10; ++q) u[q] = v[q];
    }
    double y = 0.0, hs = 0.0;
    for (int b = 0; b < nb; ++b) {
      const int r0 = b * FB;
      {
        double v[16];
        if (valid) sw_prefetch<CONTIG>(a.in, lbase, rstride, n, r0 + 5 + SW_PF * FB);
        sw_rows<CONTIG>(a.in, lbase, gbase, rstride, lstride, nl, n, per, r0 + 5, T, lane, v);
#pragma unroll
        for (int s = 0; s < 16; ++s) u[10 + s] = v[s];
      }
      if ((per && r0 + FB <= n) || (!per && r0 >= 5 && r0 + FB + 5 <= n)) {
        // interior block: full-order rows, no conditionals
#pragma unroll
        for (int s = 0; s < FB; ++s) {
          const int r = r0 + s;
          const double rhs = filt_rhs5(u + s, a.fc);
          y = r == 0 ? rhs : rhs - sfact[r > 0 ? r - 1 : 0] * y;
          if (per) hs = hs + sh[r] * rhs;
        }
      } else {
#pragma unroll
        for (int s = 0; s < FB; ++s) {
          const int r = r0 + s;
          if (r >= n) break;
          const int hh = per ? 5 : ((r == 0 || r == n - 1) ? 0 : min(min(r, n - 1 - r), 5));
          const double rhs = filt_rhs(u + s, hh, a.fc);
          y = r == 0 ? rhs : rhs - sfact[r - 1] * y;
          if (per) hs = hs + sh[r] * rhs;
        }
      }
      if (b + 1 < nb) ck[b * blockDim.x + tid] = y;  // y at row 16b + 15
#pragma unroll
      for (int q = 0; q < 10; ++q) u[q] = u[16 + q];
    }
    const double f = per ? hs / a.denom : 0.0;
    // ---------------- pass 2: blocks backwards, recompute y, back-substitute
    // u[q] = row 16b - 5 + q; rows 16b+11.. carried from block b+1
    double xn = 0.0;
    {
      const int r0 = (nb - 1) * FB;
      double v[16];
      sw_rows<CONTIG>(a.in, lbase, gbase, rstride, lstride, nl, n, per, r0 + 11, T, lane, v);
#pragma unroll
      for (int q = 0; q < 10; ++q) u[16 + q] = v[q];
    }
    for (int b = nb - 1; b >= 0; --b) {
      const int r0 = b * FB;
      {
        double v[16];
        if (valid) sw_prefetch<CONTIG>(a.in, lbase, rstride, n, r0 - 5 - SW_PF * FB);
        if (valid && a.A) sw_prefetch<CONTIG>(a.A, lbase, rstride, n, r0 - SW_PF * FB);
        sw_rows<CONTIG>(a.in, lbase, gbase, rstride, lstride, nl, n, per, r0 - 5, T, lane, v);
#pragma unroll
        for (int s = 0; s < 16; ++s) u[s] = v[s];
      }
      double av[16];
      if (a.A) sw_rows<CONTIG>(a.A, lbase, gbase, rstride, lstride, nl, n, 0, r0, T, lane, av);
      double yp = b > 0 ? ck[(b - 1) * blockDim.x + tid] : 0.0;
      double yb[FB];
      if ((per && r0 + FB <= n) || (!per && r0 >= 5 && r0 + FB + 5 <= n)) {
#pragma unroll
        for (int s = 0; s < FB; ++s) {
          const int r = r0 + s;
          const double rhs = filt_rhs5(u + s, a.fc);
          yp = r == 0 ? rhs : rhs - sfact[r > 0 ? r - 1 : 0] * yp;
          yb[s] = yp;
        }
      } else {
#pragma unroll
        for (int s = 0; s < FB; ++s) {
          const int r = r0 + s;
          const int hh =
              per ? (r < n ? 5 : 0) : ((r == 0 || r >= n - 1) ? 0 : min(min(r, n - 1 - r), 5));
          const double rhs = filt_rhs(u + s, hh, a.fc);
          yp = r == 0 ? rhs : rhs - sfact[r > 0 && r <= n ? r - 1 : 0] * yp;
          yb[s] = yp;
        }
      }
      double xo[FB];
#pragma unroll
      for (int s = FB - 1; s >= 0; --s) {
        const int r = r0 + s;
        double xv = 0.0;
        if (r < n) {
          const double x =
              r == n - 1 ? yb[s] / sd[r] : div_rn(yb[s] - sdu[r] * xn, sd[r], srinv[r]);
          xn = x;
          xv = per ? x - f * sz[r] : x;
          if (a.A && valid) {
            if (!isfinite(xv)) bad = 1;
            ma = fmax(ma, fabs(xv));
            md = fmax(md, fabs(xv - av[s]));
          }
        }
        xo[s] = xv;
      }
      // store rows [r0, r0+16)
      if (CONTIG) {
#pragma unroll
        for (int s = 0; s < 16; ++s) T[lane][s] = xo[s];
        __syncwarp();
        const int r = r0 + (lane & 15);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int m = 2 * q + (lane >> 4);
          if (m < nl && r < n) __stcs(a.out + gbase + (long long)m * lstride + r, T[m][lane & 15]);
        }
        __syncwarp();
      } else if (valid) {
        double* p = a.out + lbase + (long long)r0 * rstride;
#pragma unroll
        for (int s = 0; s < 16; ++s)
          if (r0 + s < n) __stcs(p + (long long)s * rstride, xo[s]);
      }
#pragma unroll
      for (int q = 0; q < 10; ++q) u[16 + q] = u[q];
    }
  }
  if (a.A) {
    md = warp_max(md);
    ma = warp_max(ma);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      atomicMax(&a.st->max_delta_bits, (unsigned long long)__double_as_longlong(md));
      atomicMax(&a.st->max_abs_bits, (unsigned long long)__double_as_longlong(ma));
      if (bad) atomicOr(&a.st->nonfinite, 1);
    }
  }
}

}  // namespace wd
