// Validation kernels (reference metrics.py): the brute-force
// wall-distance oracle, the 1/J-weighted L2 error norm and |grad phi|.
#pragma once

#include "wd_kernels.cuh"

namespace wd {

// metrics.py:20-34 sampled_wall_distance: out_i = sqrt(min_m sum_d
// (p_id - w_md)^2), the sum in numpy's order ((dx^2 + dy^2) + dz^2) and the
// min order-free, so the result is bit-identical.  O(n m) fp64: each thread
// owns MP_PTS query points; the wall samples stream through shared memory in
// tiles read by every thread (broadcast), so the loop is pure DFMA-free
// fp64 arithmetic on registers.
constexpr int MP_T = 256;     // threads per CTA
constexpr int MP_PTS = 2;     // query points per thread
constexpr int MP_TILE = 1024; // wall samples per shared tile

template <int D>
__global__ void __launch_bounds__(MP_T) k_sampled_distance(const double* __restrict__ pts,
                                                           long long n,
                                                           const double* __restrict__ wall,
                                                           long long m, double* __restrict__ out) {
  __shared__ double sw[MP_TILE * D];
  const long long i0 = ((long long)blockIdx.x * MP_T + threadIdx.x) * MP_PTS;
  double p[MP_PTS][D], best[MP_PTS];
#pragma unroll
  for (int a = 0; a < MP_PTS; ++a) {
    best[a] = INFINITY;
#pragma unroll
    for (int c = 0; c < D; ++c) p[a][c] = i0 + a < n ? pts[(i0 + a) * D + c] : 0.0;
  }
  for (long long m0 = 0; m0 < m; m0 += MP_TILE) {
    const int cnt = (int)min((long long)MP_TILE, m - m0);
    __syncthreads();
    for (int t = threadIdx.x; t < cnt * D; t += MP_T) sw[t] = wall[m0 * D + t];
    __syncthreads();
#pragma unroll 4
    for (int q = 0; q < cnt; ++q) {
#pragma unroll
      for (int a = 0; a < MP_PTS; ++a) {
        const double dx = p[a][0] - sw[q * D];
        double d2 = dx * dx;
#pragma unroll
        for (int c = 1; c < D; ++c) {
          const double dc = p[a][c] - sw[q * D + c];
          d2 = d2 + dc * dc;
        }
        best[a] = fmin(best[a], d2);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < MP_PTS; ++a)
    if (i0 + a < n) out[i0 + a] = sqrt(best[a]);
}

// metrics.py:54-66 l2_norm: sqrt(sum_i w_i (phi_i - ex_i)^2), w_i = 1 / J_i
// (J from jac, or the constant jc).  Deterministic: fixed-order per-thread
// sums, a fixed shared-memory tree per block, then one block sums the block
// partials in index order (numpy's pairwise sum is not reproduced bitwise;
// tests compare at 1e-13 relative).
constexpr int L2_T = 256;
constexpr int L2_B = 1184;

__global__ void __launch_bounds__(L2_T) k_l2_partial(const double* __restrict__ phi,
                                                     const double* __restrict__ ex,
                                                     const double* __restrict__ jac, double jc,
                                                     long long N, double* __restrict__ part) {
  __shared__ double sm[L2_T];
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * L2_T + threadIdx.x; i < N;
       i += (long long)gridDim.x * L2_T) {
    const double w = 1.0 / (jac ? jac[i] : jc);
    const double d = phi[i] - ex[i];
    acc += w * (d * d);
  }
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int s = L2_T / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sm[threadIdx.x] += sm[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

__global__ void k_l2_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double sm[L2_T];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nb; i += L2_T) acc += part[i];
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int s = L2_T / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sm[threadIdx.x] += sm[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sqrt(sm[0]);
}

// metrics.py:121-124 gradient_magnitude: sqrt(sum(u * u for u in U)),
// Python's sum order (0 + U0^2 skipped: identical value up to the zero sign)
__global__ void k_gradmag(MVec3 U, long long N, int nd, double* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x) {
    double s = U.p[0][i] * U.p[0][i];
    for (int a = 1; a < nd; ++a) s = s + U.p[a][i] * U.p[a][i];
    out[i] = sqrt(s);
  }
}

// levelset.py:169-202 rate(p) = source - F |grad p|, |grad p| as above
__global__ void k_ls_rate(MVec3 U, long long N, int nd, double F, double source,
                          double* __restrict__ k) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x) {
    double s = U.p[0][i] * U.p[0][i];
    for (int a = 1; a < nd; ++a) s = s + U.p[a][i] * U.p[a][i];
    k[i] = source - F * sqrt(s);
  }
}

__global__ void k_fill(double* __restrict__ out, double v, long long N) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = v;
}

}  // namespace wd

namespace wd {

// Marching-squares segment extraction (reference levelset.py:214-318 keeps
// this on the host; here every cell is one thread).  Cell (i, j) of an
// (n0, n1) field: corner bits 1 = (i, j), 2 = (i+1, j), 4 = (i+1, j+1),
// 8 = (i, j+1) set where f - level > 0 (exact zeros count as +1e-30, the
// reference's tie rule); each crossed cell edge carries the linearly
// interpolated point (1 - t) x_a + t x_b, t = h_a / (h_a - h_b); the two
// saddle codes connect around the corner pair whose sign differs from the
// sign of the corner sum.  Output per cell: count (0..2) and per segment two
// edge identities (2 * node + 0 for the edge towards i+1, + 1 towards j+1,
// node = i * n1 + j) with their (x, y) points -- chained on the host.
struct IsoEdge {
  long long id;
  double x, y;
};

__device__ __forceinline__ IsoEdge iso_edge(const double* f, const double* cx, const double* cy,
                                            double level, int n1, int i, int j, int towards_j) {
  const long long a = (long long)i * n1 + j;
  const long long b = towards_j ? a + 1 : a + n1;
  double ha = f[a] - level, hb = f[b] - level;
  if (ha == 0.0) ha = 1e-30;
  if (hb == 0.0) hb = 1e-30;
  const double t = ha / (ha - hb);
  IsoEdge e;
  e.id = 2 * a + towards_j;
  e.x = (1.0 - t) * cx[a] + t * cx[b];
  e.y = (1.0 - t) * cy[a] + t * cy[b];
  return e;
}

static __global__ void k_iso_segments(const double* __restrict__ f, const double* __restrict__ cx,
                                      const double* __restrict__ cy, int n0, int n1, double level,
                                      int* __restrict__ count, long long* __restrict__ ids,
                                      double* __restrict__ pts) {
  const long long cells = (long long)(n0 - 1) * (n1 - 1);
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < cells;
       c += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(c / (n1 - 1)), j = (int)(c % (n1 - 1));
    double h[4];
    const long long a = (long long)i * n1 + j;
    h[0] = f[a] - level;
    h[1] = f[a + n1] - level;
    h[2] = f[a + n1 + 1] - level;
    h[3] = f[a + 1] - level;
    int code = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (h[q] == 0.0) h[q] = 1e-30;
      if (h[q] > 0.0) code |= 1 << q;
    }
    // the four cell edges: 0 bottom (j), 1 right (i+1), 2 top (j+1), 3 left (i)
    // crossed edge pairs per code, two bits per edge, up to two segments
    int ns = 0, e[4] = {0, 0, 0, 0};
    auto seg = [&](int p, int q) {
      e[2 * ns] = p;
      e[2 * ns + 1] = q;
      ++ns;
    };
    const bool mid_up = ((h[0] + h[1]) + h[2]) + h[3] > 0.0;
    switch (code) {
      case 1: case 14: seg(3, 0); break;
      case 2: case 13: seg(0, 1); break;
      case 3: case 12: seg(3, 1); break;
      case 4: case 11: seg(1, 2); break;
      case 6: case 9: seg(0, 2); break;
      case 7: case 8: seg(3, 2); break;
      case 5:
        if (mid_up) { seg(3, 2); seg(0, 1); } else { seg(3, 0); seg(1, 2); }
        break;
      case 10:
        if (mid_up) { seg(3, 0); seg(1, 2); } else { seg(0, 1); seg(2, 3); }
        break;
      default: break;
    }
    count[c] = ns;
    for (int s = 0; s < 2 * ns; ++s) {
      IsoEdge g;
      switch (e[s]) {
        case 0: g = iso_edge(f, cx, cy, level, n1, i, j, 0); break;       // (i,j)-(i+1,j)
        case 1: g = iso_edge(f, cx, cy, level, n1, i + 1, j, 1); break;   // (i+1,j)-(i+1,j+1)
        case 2: g = iso_edge(f, cx, cy, level, n1, i, j + 1, 0); break;   // (i,j+1)-(i+1,j+1)
        default: g = iso_edge(f, cx, cy, level, n1, i, j, 1); break;      // (i,j)-(i,j+1)
      }
      ids[4 * c + s] = g.id;
      pts[8 * c + 2 * s] = g.x;
      pts[8 * c + 2 * s + 1] = g.y;
    }
  }
}

}  // namespace wd
