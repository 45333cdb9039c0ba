// Fused implicit-filter sweep along one axis (operators.py:305-352) for the
// specialised 3-D path, in LAPACK dgtsv elimination order (no row
// interchanges occur for the filter matrix).
//
// Layout / data movement: one warp owns 32 grid lines (lane = line) and
// walks them row by row in chunks of 32 rows.  Axes 0/1: the 32 lines are 32
// consecutive k, so every row access is one coalesced 256-byte segment.
// Axis 2 (contiguous lines): each chunk is staged through a padded 32x33
// shared-memory transpose.  The forward-elimination values are parked in a
// lane-contiguous scratch slab private to the warp (sized so all resident
// warps' slabs stay L2-resident) and read back in reverse for the back
// substitution.  Every chunk is loaded into registers one chunk ahead, so
// the only serial dependency is the recurrence itself.  The factor
// (dgtsv order) lives in shared memory.  HBM traffic: one read + one write
// per node (+ one read of phi for the fused convergence reduction on the
// last axis).
//
// Division: x_i = (y_i - du_i x_{i+1}) / d_i is evaluated as a correctly
// rounded quotient from the precomputed reciprocal r_i = RN(1/d_i)
// (Markstein: q0 = s*r, e = fma(-q0, d, s), q = fma(e, r, q0)), equal to
// IEEE s / d; the parity tests check bit equality with the reference.
#pragma once

#include "wd_kernels.cuh"

namespace wd {


struct SweepArgs {
  const double* in;
  double* out;
  double* scratch;     // >= total_warps * n * 32 doubles
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
  double vn, denom;
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

// filter RHS for row r from the window (slot 5 = row r): order of
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

// rows per chunk: 32 for the transposed (contiguous-line) axis, 16 otherwise
template <bool CONTIG>
struct SwCh { static constexpr int v = 16; };

template <bool CONTIG>
__device__ __forceinline__ void sw_load_chunk(const SweepArgs& a, double (*T)[17], int lane, int c,
                                              int nl, bool valid, long long base,
                                              long long gbase, long long rstride, double* v) {
  constexpr int CH = SwCh<CONTIG>::v;
  const int n = a.n;
  const int r0 = c * CH;
  if (CONTIG) {
    // element q of this lane: line 2q + (lane >> 4), row r0 + (lane & 15)
    const int r = r0 + (lane & 15);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int m = 2 * q + (lane >> 4);
      v[q] = (m < nl && r < n) ? __ldcs(a.in + gbase + (long long)m * a.n2 + r) : 0.0;
    }
  } else {
#pragma unroll
    for (int s = 0; s < CH; ++s) {
      const int r = r0 + s;
      v[s] = (valid && r < n) ? __ldcs(a.in + base + (long long)r * rstride) : 0.0;
    }
  }
}

template <bool CONTIG>
__global__ void __launch_bounds__(128, 3) k_filter_sweep(SweepArgs a) {
  if (a.st->state != WD_STATE_RUNNING) return;
  extern __shared__ double sw_smem[];
  double(*tile)[32][17] = reinterpret_cast<double(*)[32][17]>(sw_smem);
  const int n = a.n;
  double* sf0 = sw_smem + 4 * 32 * 17;  // fact | du | d | rinv | z, n each
  double* sf1 = sf0 + n;
  double* sf2 = sf1 + n;
  double* sf3 = sf2 + n;
  double* sf4 = sf3 + n;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    sf0[t] = a.fact[t];
    sf1[t] = a.du[t];
    sf2[t] = a.d[t];
    sf3[t] = a.rinv[t];
    sf4[t] = a.per ? a.z[t] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gw = blockIdx.x * (blockDim.x >> 5) + wib;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  double(*T)[17] = tile[wib];
  double* scr = a.scratch + (long long)gw * n * 32;
  long long groups, lines_per_row_blk;
  long long rstride;
  if (a.axis == 2) {
    lines_per_row_blk = (a.n1 + 31) / 32;
    groups = (long long)a.n0 * lines_per_row_blk;
    rstride = 1;
  } else {
    lines_per_row_blk = (a.n2 + 31) / 32;
    groups = (long long)(a.axis == 0 ? a.n1 : a.n0) * lines_per_row_blk;
    rstride = a.axis == 0 ? a.s0 : a.n2;
  }
  constexpr int CH = SwCh<CONTIG>::v;
  const int nch = (n + CH - 1) / CH;
  double md = 0.0, ma = 0.0;
  int bad = 0;
  for (long long g = gw; g < groups; g += nwarps) {
    const long long outer = g / lines_per_row_blk;
    const int blk = (int)(g % lines_per_row_blk);
    long long base, gbase = 0;
    bool valid;
    if (a.axis == 2) {
      const int j = blk * 32 + lane;
      valid = j < a.n1;
      base = outer * a.s0 + (long long)j * a.n2;
      gbase = outer * a.s0 + (long long)(blk * 32) * a.n2;
    } else {
      const int k = blk * 32 + lane;
      valid = k < a.n2;
      base = (a.axis == 0 ? outer * a.n2 : outer * a.s0) + k;
    }
    const int nl = a.axis == 2 ? min(32, a.n1 - blk * 32) : min(32, a.n2 - blk * 32);
    auto ld = [&](int row) -> double {  // scalar load, row may wrap
      if (!valid) return 0.0;
      int r = row;
      if (a.per) {
        r = r % n;
        if (r < 0) r += n;
      } else if (r < 0 || r >= n) {
        return 0.0;
      }
      return a.in[base + (long long)r * rstride];
    };
    // ---------------- forward elimination
    double w[11];
#pragma unroll
    for (int s = 0; s < 6; ++s) w[s] = 0.0;
#pragma unroll
    for (int s = 6; s < 11; ++s) w[s] = ld(s - 11);  // rows -5..-1
    double y = 0.0;
    double nxt[CH];
    sw_load_chunk<CONTIG>(a, T, lane, 0, nl, valid, base, gbase, rstride, nxt);
    for (int c = 0; c < nch; ++c) {
      const int r0 = c * CH;
      double v[CH];
      if (CONTIG) {
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 16; ++q) T[2 * q + (lane >> 4)][lane & 15] = nxt[q];
        __syncwarp();
#pragma unroll
        for (int s = 0; s < 16; ++s) v[s] = T[lane][s];
      } else {
#pragma unroll
        for (int s = 0; s < CH; ++s) v[s] = nxt[s];
      }
      if (c + 1 < nch) sw_load_chunk<CONTIG>(a, T, lane, c + 1, nl, valid, base, gbase, rstride, nxt);
      const bool interior = a.per || (r0 >= 10 && r0 + CH + 5 <= n - 5);
      double yo[CH];
#pragma unroll
      for (int s = 0; s < CH; ++s) {
        const int t = r0 + s;  // newest row
        if (t >= n) continue;
#pragma unroll
        for (int q = 0; q < 10; ++q) w[q] = w[q + 1];
        w[10] = v[s];
        const int r = t - 5;
        double rhs;
        if (interior) {
          rhs = filt_rhs5(w, a.fc);
        } else {
          const int h = (r <= 0 || r >= n - 1) ? 0 : min(min(r, n - 1 - r), 5);
          rhs = filt_rhs(w, h, a.fc);
        }
        if (r >= 0) y = r == 0 ? rhs : rhs - sf0[r - 1] * y;
        yo[s] = y;
      }
#pragma unroll
      for (int s = 0; s < CH; ++s) {
        const int r = r0 + s - 5;
        if (r >= 0 && r0 + s < n) scr[(long long)r * 32 + lane] = yo[s];
      }
    }
    // rows n..n+4 (periodic wrap or zero) finish the last 5 right-hand sides
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const int t = n + s;
#pragma unroll
      for (int q = 0; q < 10; ++q) w[q] = w[q + 1];
      w[10] = ld(t);
      const int r = t - 5;
      if (r >= 0 && r < n) {
        const int h = a.per ? 5 : ((r == 0 || r == n - 1) ? 0 : min(min(r, n - 1 - r), 5));
        const double rhs = filt_rhs(w, h, a.fc);
        y = r == 0 ? rhs : rhs - sf0[r - 1] * y;
        scr[(long long)r * 32 + lane] = y;
      }
    }
    __syncwarp();
    // ---------------- back substitution (+ cyclic correction)
    const bool cyc = a.per;
    double x1 = 0.0, xlast = 0.0;
    double yn[CH];
#pragma unroll
    for (int s = 0; s < CH; ++s) {
      const int r = (nch - 1) * CH + s;
      yn[s] = r < n ? scr[(long long)r * 32 + lane] : 0.0;
    }
    for (int c = nch - 1; c >= 0; --c) {
      const int r0 = c * CH;
      double yv[CH];
#pragma unroll
      for (int s = 0; s < CH; ++s) yv[s] = yn[s];
      if (c > 0) {
#pragma unroll
        for (int s = 0; s < CH; ++s) yn[s] = scr[(long long)(r0 - CH + s) * 32 + lane];
      }
      double o[CH];
#pragma unroll
      for (int s = CH - 1; s >= 0; --s) {
        const int r = r0 + s;
        double x = 0.0;
        if (r < n) {
          if (r == n - 1) {
            x = yv[s] / sf2[r];
            xlast = x;
          } else {
            x = div_rn(yv[s] - sf1[r] * x1, sf2[r], sf3[r]);
          }
          x1 = x;
        }
        o[s] = x;
      }
      if (cyc) {
#pragma unroll
        for (int s = 0; s < CH; ++s)
          if (r0 + s < n) scr[(long long)(r0 + s) * 32 + lane] = o[s];
        continue;
      }
      // final values: write out (+ convergence reduction)
      if (CONTIG) {
        __syncwarp();
#pragma unroll
        for (int s = 0; s < 16; ++s) T[lane][s] = o[s];
        __syncwarp();
        const int r = r0 + (lane & 15);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int m = 2 * q + (lane >> 4);
          if (m < nl && r < n) {
            const long long idx = gbase + (long long)m * a.n2 + r;
            const double xv = T[m][lane & 15];
            __stcs(a.out + idx, xv);
            if (a.A) {
              if (!isfinite(xv)) bad = 1;
              ma = fmax(ma, fabs(xv));
              md = fmax(md, fabs(xv - __ldcs(a.A + idx)));
            }
          }
        }
      } else if (valid) {
#pragma unroll
        for (int s = 0; s < CH; ++s) {
          const int r = r0 + s;
          if (r < n) {
            const long long idx = base + (long long)r * rstride;
            __stcs(a.out + idx, o[s]);
            if (a.A) {
              const double xv = o[s];
              if (!isfinite(xv)) bad = 1;
              ma = fmax(ma, fabs(xv));
              md = fmax(md, fabs(xv - __ldcs(a.A + idx)));
            }
          }
        }
      }
    }
    if (cyc) {
      // x = y - f z,  f = (y_0 + vn y_{n-1}) / denom  (oracle/wd.py:cyclic_apply)
      const double f = (x1 + a.vn * xlast) / a.denom;
      __syncwarp();
      for (int c = 0; c < nch; ++c) {
        const int r0 = c * CH;
        double o[CH];
#pragma unroll
        for (int s = 0; s < CH; ++s) {
          const int r = r0 + s;
          o[s] = r < n ? scr[(long long)r * 32 + lane] : 0.0;
        }
#pragma unroll
        for (int s = 0; s < CH; ++s) {
          const int r = r0 + s;
          o[s] = r < n ? o[s] - f * sf4[r] : 0.0;
        }
        if (CONTIG) {
          __syncwarp();
#pragma unroll
          for (int s = 0; s < 16; ++s) T[lane][s] = o[s];
          __syncwarp();
          const int r = r0 + (lane & 15);
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int m = 2 * q + (lane >> 4);
            if (m < nl && r < n) {
              const long long idx = gbase + (long long)m * a.n2 + r;
              const double xv = T[m][lane & 15];
              __stcs(a.out + idx, xv);
              if (a.A) {
                if (!isfinite(xv)) bad = 1;
                ma = fmax(ma, fabs(xv));
                md = fmax(md, fabs(xv - __ldcs(a.A + idx)));
              }
            }
          }
        } else if (valid) {
#pragma unroll
          for (int s = 0; s < CH; ++s) {
            const int r = r0 + s;
            if (r < n) {
              const long long idx = base + (long long)r * rstride;
              __stcs(a.out + idx, o[s]);
              if (a.A) {
                const double xv = o[s];
                if (!isfinite(xv)) bad = 1;
                ma = fmax(ma, fabs(xv));
                md = fmax(md, fabs(xv - __ldcs(a.A + idx)));
              }
            }
          }
        }
      }
    }
    __syncwarp();
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
