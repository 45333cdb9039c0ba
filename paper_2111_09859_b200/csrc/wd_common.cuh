// Common device-side definitions for the B200 wall-distance solver.
//
// Arithmetic contract ("exact mode"): every kernel in this library is
// compiled with -fmad=false and writes each expression in the operation
// order of the reference's numpy code (left-to-right Python sums, constant
// folding such as (0.5*a)*(...), true IEEE divisions and square roots), so
// results are bit-identical to the reference / oracle up to the sign of
// zero.  See DESIGN.md sec. 4 for the per-expression mapping.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "../../include/walldist_b200.h"

namespace wd {

constexpr int kMaxDim = 3;

// Runtime-indexed read of a small kernel-parameter array as a select chain:
// indexing a by-value struct member with a runtime index would copy the
// whole struct to local memory (stack) in every thread.
template <class T, int K>
__device__ __forceinline__ T pick(const T (&a)[K], int i) {
  T r = a[0];
#pragma unroll
  for (int k = 1; k < K; ++k)
    if (i == k) r = a[k];
  return r;
}

// Division by a grid-invariant 32-bit divisor as multiply-high + add +
// shift (round-up method: l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1,
// q = (mulhi(m, x) + x) >> l with a 33-bit sum): exact for every 32-bit x,
// ~3 instructions instead of the ~20 of a runtime unsigned division.
struct FDiv {
  unsigned m, l;
};
inline FDiv fdiv_make(unsigned long long d) {
  unsigned l = 0;
  while ((1ull << l) < d) ++l;
  const unsigned long long m = ((1ull << 32) * ((1ull << l) - d)) / d + 1;
  return FDiv{(unsigned)m, l};
}
__device__ __forceinline__ unsigned fdiv(unsigned x, FDiv f) {
  return (unsigned)(((unsigned long long)__umulhi(x, f.m) + x) >> f.l);
}

// Structured-grid geometry: C-order (n0, n1[, n2]); unused axes have n = 1.
struct Geom {
  int nd;
  int n[kMaxDim];
  long long s[kMaxDim];   // element strides
  long long N;            // total nodes
  int per[kMaxDim];       // periodic axes
  int face[2 * kMaxDim];  // WD_FACE_* per face (imin, imax, jmin, ...)
  const uint8_t* mask;    // solid mask (N) or nullptr
  FDiv fs[kMaxDim], fn[kMaxDim];  // fast division by s[a], n[a] (N < 2^32)
};

// Metric terms: either uniform diagonal constants or (d, d, N) fields.
struct Metric {
  const double* m;        // nullptr when uniform
  double c[kMaxDim];      // uniform: d xi_l / d x_l
  long long N;            // nodes per term (kdiv > 1: per compact term)
  int nd;
  int kdiv;               // > 1: terms stored once per line of the last axis (index idx / kdiv)
  __device__ __forceinline__ double get(int l, int mm, long long idx) const {
    if (m == nullptr) return l == mm ? pick(c, l) : 0.0;
    return m[(long long)(l * nd + mm) * N + idx];
  }
};

// Scheme constants, folded exactly as the reference's Python expressions
// (operators.py:29-34, 111-113; EXTENSION E6 = oracle/wd.py:E6_ABC).
constexpr double E2_CA = 0.5 * 1.0;
constexpr double E4_CA = 0.5 * (4.0 / 3.0);
constexpr double E4_CB = 0.25 * (-1.0 / 3.0);
constexpr double E6_CA = 0.5 * 1.5;
constexpr double E6_CB = 0.25 * -0.6;
constexpr double E6_CC = 0.1 / 6.0;
constexpr double C4_CA = 0.5 * 1.5;
constexpr double C6_CA = 0.5 * (14.0 / 9.0);
constexpr double C6_CB = 0.25 * (1.0 / 9.0);

__device__ __forceinline__ double np_min(double a, double b) {
  // numpy.minimum: NaN-propagating
  if (a != a) return a;
  if (b != b) return b;
  return a < b ? a : b;
}
__device__ __forceinline__ double np_max(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a > b ? a : b;
}

// Line accessor with periodic wrap and coordinate period offset.
struct Line {
  const double* __restrict__ p;  // pointer to element 0 of the line
  long long st;
  int n;
  int per;
  double off;
  __device__ __forceinline__ double operator()(int j) const {
    if (!per) return p[(long long)j * st];
    if (j < 0) {
      double v = p[(long long)(j + n) * st];
      return off == 0.0 ? v : v + (-1.0 * off);
    }
    if (j >= n) {
      double v = p[(long long)(j - n) * st];
      return off == 0.0 ? v : v + off;
    }
    return p[(long long)j * st];
  }
};

// ---- explicit first derivative at row i of a line (operators.py:109-128)
template <class L>
__device__ __forceinline__ double e4_closure(const L& w, int i, int n) {
  if (i == 0)
    return (-25.0 * w(0) + 48.0 * w(1) - 36.0 * w(2) + 16.0 * w(3) - 3.0 * w(4)) / 12.0;
  if (i == 1)
    return (-3.0 * w(0) - 10.0 * w(1) + 18.0 * w(2) - 6.0 * w(3) + w(4)) / 12.0;
  if (i == n - 1)
    return (25.0 * w(n - 1) - 48.0 * w(n - 2) + 36.0 * w(n - 3) - 16.0 * w(n - 4) +
            3.0 * w(n - 5)) / 12.0;
  // i == n - 2
  return (3.0 * w(n - 1) + 10.0 * w(n - 2) - 18.0 * w(n - 3) + 6.0 * w(n - 4) - w(n - 5)) /
         12.0;
}

template <class L>
__device__ __forceinline__ double deriv_explicit_at(const L& w, int i, int n, int scheme,
                                                    int per) {
  if (scheme == WD_E2) {
    if (!per) {
      if (i == 0) return -1.5 * w(0) + 2.0 * w(1) - 0.5 * w(2);
      if (i == n - 1) return 1.5 * w(n - 1) - 2.0 * w(n - 2) + 0.5 * w(n - 3);
    }
    return E2_CA * (w(i + 1) - w(i - 1));
  }
  if (scheme == WD_E4) {
    if (!per && (i < 2 || i > n - 3)) return e4_closure(w, i, n);
    return E4_CA * (w(i + 1) - w(i - 1)) + E4_CB * (w(i + 2) - w(i - 2));
  }
  // WD_E6 (EXTENSION): E4 closures on rows 0,1,n-2,n-1; E4 central on 2,n-3
  if (!per) {
    if (i < 2 || i > n - 3) return e4_closure(w, i, n);
    if (i == 2 || i == n - 3)
      return E4_CA * (w(i + 1) - w(i - 1)) + E4_CB * (w(i + 2) - w(i - 2));
  }
  return E6_CA * (w(i + 1) - w(i - 1)) + E6_CB * (w(i + 2) - w(i - 2)) +
         E6_CC * (w(i + 3) - w(i - 3));
}

// ---- compact right-hand side at row i (operators.py:109-145)
template <class L>
__device__ __forceinline__ double compact_rhs_at(const L& w, int i, int n, int scheme,
                                                 int per) {
  if (!per) {
    if (i == 0) return (-17.0 * w(0) + 9.0 * w(1) + 9.0 * w(2) - w(3)) / 6.0;
    if (i == n - 1) return (17.0 * w(n - 1) - 9.0 * w(n - 2) - 9.0 * w(n - 3) + w(n - 4)) / 6.0;
  }
  if (scheme == WD_C4) return C4_CA * (w(i + 1) - w(i - 1));
  if (!per && (i == 1 || i == n - 2)) return 0.75 * (w(i + 1) - w(i - 1));
  return C6_CA * (w(i + 1) - w(i - 1)) + C6_CB * (w(i + 2) - w(i - 2));
}

// ---- 4th derivative (operators.py:236-250)
template <class L>
__device__ __forceinline__ double d4_at(const L& w, int i, int n, int per) {
  if (!per) {
    if (i < 2) i = 2;
    if (i > n - 3) i = n - 3;
  }
  return w(i - 2) - 4.0 * w(i - 1) + 6.0 * w(i) - 4.0 * w(i + 1) + w(i + 2);
}

// ---- boundary conditions (solver.py:87-110) as a source redirect:
// after the reference's far-field copies, node x holds the pre-BC value of
// src(x) (separable per axis); walls and the solid mask are then zeroed.
// Index arithmetic: 32-bit unsigned division whenever every index fits
// (N <= 2^32 - 1: every grid the generic path can hold), 64-bit otherwise;
// a 64-bit division costs several times the 32-bit one.
__device__ __forceinline__ int axis_coord(const Geom& g, long long idx, int a) {
  const long long s = pick(g.s, a);
  const int n = pick(g.n, a);
  if (g.N <= 0xffffffffLL) {
    const unsigned q = fdiv((unsigned)idx, pick(g.fs, a));
    return (int)(q - fdiv(q, pick(g.fn, a)) * (unsigned)n);
  }
  return (int)((idx / s) % n);
}

// One axis of a Geom as plain scalars (per-node kernels along an axis).
struct AxisGeom {
  long long N;   // total nodes
  long long sa;  // stride of the axis
  int n;         // length of the axis
  FDiv fs, fn;   // fast division by sa, n (N < 2^32)
  __device__ __forceinline__ int coord(long long idx) const {
    if (N <= 0xffffffffLL) {
      const unsigned q = fdiv((unsigned)idx, fs);
      return (int)(q - fdiv(q, fn) * (unsigned)n);
    }
    return (int)((idx / sa) % n);
  }
};
__host__ __device__ __forceinline__ AxisGeom axis_geom(const Geom& g, int axis) {
  return AxisGeom{g.N, g.s[axis], g.n[axis], g.fs[axis], g.fn[axis]};
}

__device__ __forceinline__ void node_coords(const Geom& g, long long idx, int c[kMaxDim]) {
#pragma unroll
  for (int a = 0; a < kMaxDim; ++a) c[a] = axis_coord(g, idx, a);
}

__device__ __forceinline__ bool is_pinned(const Geom& g, long long idx, const int c[kMaxDim]) {
#pragma unroll
  for (int a = 0; a < kMaxDim; ++a) {
    if (a >= g.nd) break;
    if (c[a] == 0 && g.face[2 * a] == WD_FACE_WALL) return true;
    if (c[a] == g.n[a] - 1 && g.face[2 * a + 1] == WD_FACE_WALL) return true;
  }
  return g.mask != nullptr && g.mask[idx] != 0;
}

__device__ __forceinline__ long long bc_source(const Geom& g, long long idx,
                                               const int c[kMaxDim]) {
  long long src = idx;
#pragma unroll
  for (int a = 0; a < kMaxDim; ++a) {
    if (a >= g.nd) break;
    if (c[a] == 0 && g.face[2 * a] == WD_FACE_FARFIELD) src += g.s[a];
    if (c[a] == g.n[a] - 1 && g.face[2 * a + 1] == WD_FACE_FARFIELD) src -= g.s[a];
  }
  return src;
}

// Host -> device copy that has LANDED when it returns.  A plain cudaMemcpy
// from pageable memory returns once the bytes are staged; the DMA runs on the
// legacy stream and is not ordered against the solver's non-blocking streams,
// so a kernel (or a communicator callback) launched right after could still
// read the old contents.
inline cudaError_t upload_sync(void* dst, const void* src, size_t bytes) {
  const cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
  return e != cudaSuccess ? e : cudaStreamSynchronize(cudaStreamLegacy);
}
inline cudaError_t memset_sync(void* dst, int v, size_t bytes) {
  const cudaError_t e = cudaMemset(dst, v, bytes);
  return e != cudaSuccess ? e : cudaStreamSynchronize(cudaStreamLegacy);
}

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may be scheduled while its predecessor
// in the stream still runs; it must not touch anything the predecessor
// writes (the status word included) before pdl_wait(), which returns once
// every prerequisite grid has completed and flushed.  pdl_trigger() at the
// top of a kernel lets ITS successor be scheduled as soon as all of this
// grid's CTAs have started.  Both are no-ops in a normally launched grid.
// Wired into the launch-bound 2-D step (wd_stage_explicit.cuh, WD_PDL=1);
// inside a CUDA-graph replay it measured slower than plain edges (wd_capi.cu:
// launch_pdl), so the default launches are plain.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// Device status word shared by the step kernels (freeze-on-stop).
struct Status {
  int state;          // WD_STATE_*
  int iters;          // completed pseudo-steps
  int max_iters;
  int diverged_iter;  // iteration at which divergence was detected
  unsigned long long max_delta_bits;  // running max |phi_new - phi| (>= 0 -> bit order)
  unsigned long long max_abs_bits;    // running max |phi_new|
  int nonfinite;
  int pad;
};

}  // namespace wd
