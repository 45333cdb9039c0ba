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
