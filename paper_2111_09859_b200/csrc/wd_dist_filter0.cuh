// Partitioned axis-0 filter for the slab-decomposed fast path
// (paper_2111_09859_b200/dist.py, SolveConfig.arith = "fast").
//
// The axis-0 lines are split over the P ranks (rank r owns global rows
// [lo, lo + nl)).  The implicit filter (operators.py:305-352, cyclic by
// Sherman-Morrison, oracle/wd.py:cyclic_apply) is the LU solve
//     y_i = rhs_i - fm_i y_{i-1},   x_i = y_i / d_i - g_i x_{i+1},
//     x <- x - (h . rhs / denom) z,
// whose recurrences are affine in their carries, so a rank's block of rows
// acts on an incoming carry c as  c_out = Y_blk + P_blk c  (forward) and
// x_lo = X_blk + Q_blk c2 (backward), with P_blk = prod(-fm), Q_blk =
// prod(-g) over the block -- field independent, precomputed on the host.
// Instead of transposing the whole slab twice (all_to_all, ~2 x 117 MB per
// GPU per step at P = 8) the ranks exchange one or two doubles per line:
//   phase 1: local forward from 0 -> (Y_blk, h.rhs partial)   [all_gather]
//   phase 2: carry-in from the gathered blocks of ranks < r, forward
//            (y -> out), local backward from 0 (x' -> out) -> X_blk [all_gather]
//   phase 3: carry from the blocks of ranks > r, x = x' + Qpref c2 - f z.
// One thread per line (consecutive k -> coalesced rows).  Same linear
// system as the single-GPU scan filter; round-off-level differences.
#pragma once

#include "wd_kernels.cuh"

namespace wd {

struct D0Tables {
  const double* row;   // per local row r (nl entries each): fm, 1/d, g, h, z, Qpref
  const double* blk;   // per rank q: P_blk, Q_blk
  int P, rank, nl;
  double denom;        // cyclic Sherman-Morrison denominator
};

__device__ __forceinline__ double d0_rhs(const double* w, long long s, const FilterCoef& fc) {
  // full-order (10th) row, same expression as the single-GPU fast sweep
  const double* c = fc.hc + 30;
  double v = c[5] * (w[5 * s] + w[-5 * s]);
  v = fma(c[4], w[4 * s] + w[-4 * s], v);
  v = fma(c[3], w[3 * s] + w[-3 * s], v);
  v = fma(c[2], w[2 * s] + w[-2 * s], v);
  v = fma(c[1], w[s] + w[-s], v);
  return fma(c[0], w[0], v);
}

// in: ghosted slab (nl + 2G, n1, n2); out: interior slab (nl, n1, n2)
// xa: [P][2][lines] gathered (Y_blk, hs); xb: [P][lines] gathered X_blk;
// mine: this rank's outgoing slot (phase 1: 2 x lines, phase 2: lines)
template <int PHASE>
__global__ void k_dist_filter0(const double* __restrict__ in, double* out, int n1, int n2, int G,
                               D0Tables T, FilterCoef fc, const double* __restrict__ xa,
                               const double* __restrict__ xb, double* mine, const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  const long long lines = (long long)n1 * n2;
  const long long s = lines;  // row stride
  const int nl = T.nl;
  const double* fm = T.row;
  const double* ri = T.row + nl;
  const double* gg = T.row + 2 * nl;
  const double* hh = T.row + 3 * nl;
  const double* zz = T.row + 4 * nl;
  const double* qp = T.row + 5 * nl;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < lines;
       q += (long long)gridDim.x * blockDim.x) {
    const double* w = in + (long long)G * s + q;  // row 0 of the line
    double* o = out + q;
    if (PHASE == 1) {
      double y = 0.0, hs = 0.0;
      for (int r = 0; r < nl; ++r) {
        const double b = d0_rhs(w + r * s, s, fc);
        y = fma(-fm[r], y, b);
        hs = fma(hh[r], b, hs);
      }
      mine[q] = y;
      mine[lines + q] = hs;
    } else if (PHASE == 2) {
      double c = 0.0;  // y of global row lo - 1
      for (int p = 0; p < T.rank; ++p) c = fma(T.blk[2 * p], c, xa[(2LL * p) * lines + q]);
      double y = c;
      for (int r = 0; r < nl; ++r) {
        const double b = d0_rhs(w + r * s, s, fc);
        y = fma(-fm[r], y, b);
        o[r * s] = y;
      }
      double x = 0.0;  // local backward from x(lo + nl) = 0
      for (int r = nl - 1; r >= 0; --r) {
        x = fma(-gg[r], x, o[r * s] * ri[r]);
        o[r * s] = x;
      }
      mine[q] = x;  // X_blk: x' of row lo
    } else {
      double c2 = 0.0;  // x of global row lo + nl
      for (int p = T.P - 1; p > T.rank; --p) c2 = fma(T.blk[2 * p + 1], c2, xb[p * lines + q]);
      double f = 0.0;
      if (T.denom != 0.0) {
        double hsum = 0.0;
        for (int p = 0; p < T.P; ++p) hsum += xa[(2LL * p + 1) * lines + q];
        f = hsum / T.denom;
      }
      for (int r = 0; r < nl; ++r) {
        double x = fma(qp[r], c2, o[r * s]);
        if (T.denom != 0.0) x = fma(-f, zz[r], x);
        o[r * s] = x;
      }
    }
  }
}

}  // namespace wd
