// Fast-arithmetic implicit filter sweep for FEW LONG lines (2-D grids whose
// lines exceed the 512 rows of k_filter_scan: BASELINE config 3, the
// 1025 x 513 bump).
//
// Same system (operators.py:305-352; cyclic lines by Sherman-Morrison,
// oracle/wd.py:cyclic_apply) and the same segmented affine scan as
// wd_filter_scan.cuh, cut for the other end of the shape range: a 2-D grid
// has ~10^3 lines of ~10^3 rows, so the exact sweep is 10^3 dependency chains
// of 2 x 10^3 dependent fp64 steps (~100 us per sweep, half of config 3's
// step) on a GPU that is otherwise empty.  Here a CTA takes 4 adjacent lines
// (32-byte runs on the strided axis), splits each into 64 segments of
// m = ceil(n / 64) <= 32 rows (256 threads), and the longest chain left is
// the 63-step carry over the segment ends.  Tables as scan_pack builds them
// for 64 segments; n <= 2048.
#pragma once

#include "wd_filter_scan.cuh"

namespace wd {

constexpr int FL_L = 4;             // lines per CTA
constexpr int FL_S = 64;            // segments per line
constexpr int FL_T = FL_L * FL_S;   // threads
constexpr int FL_NMAX = FL_S * FS_M;

struct LongScanArgs {
  const double* in;
  double* out;
  long long L;                 // lines
  long long rstride, lstride;  // row / line strides (one of them is 1)
  int per;
  ScanDev T;
  FilterCoef fc;
  const Status* st;
};

inline size_t filter_long_smem(int n) {
  return ((size_t)((7 * n + 36 + 1) & ~1) + (size_t)(n + 2 * FS_G) * FL_L + 3 * FL_T) *
         sizeof(double);
}

// UM: compile-time bound on the rows per segment (register windows), m <= UM
template <int UM>
static __global__ void __launch_bounds__(FL_T, UM <= 20 ? 2 : 1) k_filter_long(LongScanArgs a) {
  if (a.st && a.st->state != WD_STATE_RUNNING) return;
  extern __shared__ __align__(16) double fl_smem[];
  const int n = a.T.n, m = a.T.m, per = a.per;
  const double2* T1 = reinterpret_cast<const double2*>(fl_smem);  // (fm, h)
  const double2* T2 = T1 + n;                                     // (P, g)
  const double2* T4 = T2 + n;                                     // (Q, z)
  const double* T3 = fl_smem + 6 * n;                             // 1/d
  double* shc = fl_smem + 7 * n;
  double* tile = fl_smem + ((7 * n + 36 + 1) & ~1);  // [row + 5][line]
  const int NR = n + 2 * FS_G;
  double* Yend = tile + NR * FL_L;
  double* Xst = Yend + FL_T;
  double* Hs = Xst + FL_T;
  const int tid = threadIdx.x, l = tid % FL_L, s = tid / FL_L;
  for (int t = tid; t < 7 * n; t += FL_T) fl_smem[t] = a.T.tab[t];
  if (tid < 36) shc[tid] = a.fc.hc[tid];
  const int r0 = s * m;
  const int cnt = max(0, min(m, n - r0));
  const int nseg = (n + m - 1) / m;
  const long long groups = (a.L + FL_L - 1) / FL_L;
  const double rden = 1.0 / a.T.denom;
  double* tl = tile + l + (r0 + FS_G) * FL_L;  // row r0 of my line

  for (long long q = blockIdx.x; q < groups; q += gridDim.x) {
    const long long line0 = q * FL_L;
    const int nl = (int)min((long long)FL_L, a.L - line0);
    __syncthreads();  // tables staged / previous tile stored
    // rows -5 .. n+4 of the tile's lines (ghosts wrapped when periodic, else 0)
    for (int idx = tid; idx < NR * FL_L; idx += FL_T) {
      const int ll = idx % FL_L;
      int r = idx / FL_L - FS_G;
      bool ok = ll < nl;
      if (r < 0 || r >= n) {
        ok = ok && per;
        r = r < 0 ? r + n : r - n;
      }
      tile[idx] = ok ? __ldg(a.in + (line0 + ll) * a.lstride + (long long)r * a.rstride) : 0.0;
    }
    __syncthreads();
    // ---- 1. right-hand side + local forward recurrence (from zero)
    double yv[UM];
    double hs = 0.0, yp = 0.0;
    {
      double ww[UM + 10];
#pragma unroll
      for (int k = 0; k < 10; ++k) ww[k] = tl[(k - 5) * FL_L];
#pragma unroll
      for (int rr = 0; rr < UM; ++rr) {
        if (rr < cnt) {
          ww[rr + 10] = tl[(rr + 5) * FL_L];
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
    Yend[tid] = yp;
    Hs[tid] = hs;
    __syncthreads();  // every right-hand side taken: the tile is free
    // ---- 2. forward carry, fix-up, local back substitution
    double c = 0.0;
    for (int t = 0; t < s; ++t) c = fma(T2[t * m + m - 1].x, c, Yend[t * FL_L + l]);
    double xn = 0.0;
#pragma unroll
    for (int rr = UM - 1; rr >= 0; --rr) {
      if (rr < cnt) {
        const int r = r0 + rr;
        const double2 t2 = T2[r];
        const double y = fma(t2.x, c, yv[rr]);
        xn = fma(-t2.y, xn, y * T3[r]);
        yv[rr] = xn;
      }
    }
    Xst[tid] = xn;
    __syncthreads();
    // ---- 3. backward carry, fix-up, cyclic correction -> tile
    double c2 = 0.0;
    for (int t = nseg - 1; t > s; --t) c2 = fma(T4[t * m].x, c2, Xst[t * FL_L + l]);
    double f = 0.0;
    if (per) {
      double hsum = 0.0;
      for (int t = 0; t < nseg; ++t) hsum += Hs[t * FL_L + l];
      f = hsum * rden;
    }
#pragma unroll
    for (int rr = 0; rr < UM; ++rr) {
      if (rr < cnt) {
        const double2 t4 = T4[r0 + rr];
        double x = fma(t4.x, c2, yv[rr]);
        if (per) x = fma(-f, t4.y, x);
        tl[rr * FL_L] = x;
      }
    }
    __syncthreads();
    // ---- 4. store
    for (int idx = tid; idx < n * FL_L; idx += FL_T) {
      const int ll = idx % FL_L, r = idx / FL_L;
      if (ll < nl)
        a.out[(line0 + ll) * a.lstride + (long long)r * a.rstride] = tile[idx + FS_G * FL_L];
    }
  }
}

// one sweep: the instantiation for the segment length, shared-memory limit raised
inline void launch_filter_long(const LongScanArgs& a, cudaStream_t s) {
  const size_t sm = filter_long_smem(a.T.n);
  const unsigned grid = (unsigned)((a.L + FL_L - 1) / FL_L);
  auto go = [&](void (*k)(LongScanArgs)) {
    cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<grid, FL_T, sm, s>>>(a);
  };
  if (a.T.m <= 12) go(k_filter_long<12>);
  else if (a.T.m <= 20) go(k_filter_long<20>);
  else go(k_filter_long<FS_M>);
}

}  // namespace wd
