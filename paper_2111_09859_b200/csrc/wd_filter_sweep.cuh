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
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    sfact[t] = a.fact[t];
    sdu[t] = a.du[t];
    sd[t] = a.d[t];
    srinv[t] = a.rinv[t];
    sz[t] = a.per ? a.z[t] : 0.0;
    sh[t] = a.per ? a.h[t] : 0.0;
  }
  __syncthreads();
  const int tid = threadIdx.x;
  // lines: axis 0 -> (j, k), axis 1 -> (i, k), axis 2 -> (i, j); the
  // fastest-varying index of the line id is k (axes 0/1) or j (axis 2)
  long long L, rstride;
  int fast_n;
  if (a.axis == 0) {
    L = (long long)a.n1 * a.n2;
    rstride = a.s0;
    fast_n = a.n2;
  } else if (a.axis == 1) {
    L = (long long)a.n0 * a.n2;
    rstride = a.n2;
    fast_n = a.n2;
  } else {
    L = (long long)a.n0 * a.n1;
    rstride = 1;
    fast_n = a.n1;
  }
  const bool interior_ok = a.per != 0;
  double md = 0.0, ma = 0.0;
  int bad = 0;
  for (long long line = blockIdx.x * (long long)blockDim.x + tid; line < L;
       line += (long long)gridDim.x * blockDim.x) {
    const long long outer = line / fast_n;
    const int inner = (int)(line % fast_n);
    long long base;
    if (a.axis == 0) base = outer * a.n2 + inner;
    else if (a.axis == 1) base = outer * a.s0 + inner;
    else base = outer * a.s0 + (long long)inner * a.n2;
    const double* __restrict__ src = a.in + base;
    auto ld = [&](int row) -> double {
      int r = row;
      if (a.per) {
        while (r < 0) r += n;
        while (r >= n) r -= n;
      } else if (r < 0 || r >= n) {
        return 0.0;
      }
      return src[(long long)r * rstride];
    };
    // ---------------- pass 1: forward elimination, checkpoints
    double w[11];
#pragma unroll
    for (int s = 0; s < 6; ++s) w[s] = 0.0;
#pragma unroll
    for (int s = 6; s < 11; ++s) w[s] = ld(s - 11);  // rows -5..-1
    double y = 0.0, hs = 0.0;
    for (int c = 0; c < nb; ++c) {
      const int r0 = c * FB;
      double v[FB];
#pragma unroll
      for (int s = 0; s < FB; ++s) v[s] = r0 + s < n ? src[(long long)(r0 + s) * rstride] : 0.0;
      const bool full = interior_ok || (r0 >= 10 && r0 + FB <= n);
#pragma unroll
      for (int s = 0; s < FB; ++s) {
        const int t = r0 + s;  // newest row in the window
        if (t >= n) continue;
#pragma unroll
        for (int q = 0; q < 10; ++q) w[q] = w[q + 1];
        w[10] = v[s];
        const int r = t - 5;
        if (r < 0) continue;
        double rhs;
        if (full) {
          rhs = filt_rhs5(w, a.fc);
        } else {
          const int hh = (r == 0 || r == n - 1) ? 0 : min(min(r, n - 1 - r), 5);
          rhs = filt_rhs(w, hh, a.fc);
        }
        y = r == 0 ? rhs : rhs - sfact[r - 1] * y;
        if (a.per) hs = hs + sh[r] * rhs;
        if ((r % FB) == FB - 1) ck[(r / FB) * blockDim.x + tid] = y;
      }
    }
#pragma unroll
    for (int s = 0; s < 5; ++s) {  // rows n..n+4 complete the last 5 RHS
      const int t = n + s;
#pragma unroll
      for (int q = 0; q < 10; ++q) w[q] = w[q + 1];
      w[10] = ld(t);
      const int r = t - 5;
      if (r < 0) continue;
      const int hh = a.per ? 5 : ((r == 0 || r == n - 1) ? 0 : min(min(r, n - 1 - r), 5));
      const double rhs = filt_rhs(w, hh, a.fc);
      y = r == 0 ? rhs : rhs - sfact[r - 1] * y;
      if (a.per) hs = hs + sh[r] * rhs;
      if ((r % FB) == FB - 1) ck[(r / FB) * blockDim.x + tid] = y;
    }
    const double f = a.per ? hs / a.denom : 0.0;
    // ---------------- pass 2: blocks backwards, recompute y, back-substitute
    double xn = 0.0;
    for (int b = nb - 1; b >= 0; --b) {
      const int r0 = b * FB;
      double u[FB + 10];
      if (r0 >= 5 && r0 + FB + 5 <= n) {  // interior block: plain loads
        const double* p = src + (long long)(r0 - 5) * rstride;
#pragma unroll
        for (int q = 0; q < FB + 10; ++q) u[q] = p[(long long)q * rstride];
      } else {
#pragma unroll
        for (int q = 0; q < FB + 10; ++q) u[q] = ld(r0 - 5 + q);
      }
      double av[FB];
      if (a.A) {
#pragma unroll
        for (int s = 0; s < FB; ++s)
          av[s] = r0 + s < n ? __ldcs(a.A + base + (long long)(r0 + s) * rstride) : 0.0;
      }
      const bool full = interior_ok || (r0 >= 5 && r0 + FB + 5 <= n);
      double yp = b > 0 ? ck[(b - 1) * blockDim.x + tid] : 0.0;
      double yb[FB];
#pragma unroll
      for (int s = 0; s < FB; ++s) {
        const int r = r0 + s;
        double rhs;
        if (full) {
          rhs = filt_rhs5(u + s, a.fc);
        } else {
          const int hh = (r == 0 || r >= n - 1) ? 0 : min(min(r, n - 1 - r), 5);
          rhs = filt_rhs(u + s, hh, a.fc);
        }
        yp = r == 0 ? rhs : rhs - sfact[r > 0 ? r - 1 : 0] * yp;
        yb[s] = yp;
      }
#pragma unroll
      for (int s = FB - 1; s >= 0; --s) {
        const int r = r0 + s;
        if (r >= n) continue;
        const double x = r == n - 1 ? yb[s] / sd[r] : div_rn(yb[s] - sdu[r] * xn, sd[r], srinv[r]);
        xn = x;
        const double xv = a.per ? x - f * sz[r] : x;
        const long long idx = base + (long long)r * rstride;
        __stcs(a.out + idx, xv);
        if (a.A) {
          if (!isfinite(xv)) bad = 1;
          ma = fmax(ma, fabs(xv));
          md = fmax(md, fabs(xv - av[s]));
        }
      }
    }
  }
  if (a.A) {
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

}  // namespace wd
