// Generic line / pointwise kernels of the wall-distance hot path.
//
// These are the "reference-structured" kernels: one launch per operator
// pass, any dimensionality, curvilinear metrics, every scheme and
// formulation.  They define the arithmetic (bit-identical to the reference)
// and are the fallback-free path for everything the fused kernels
// (wd_fused3d.cu) do not specialise.  Reference lines are cited per kernel.
#pragma once

#include "wd_common.cuh"

namespace wd {

// Device-resident tridiagonal factor (dgtsv elimination order, see
// oracle/wd.py:gtsv_factor and LAPACK dgtsv.f).  Packed arrays of n each.
struct TriDev {
  int n;
  int cyclic;
  const double* fact;
  const double* d;
  const double* du;
  const double* du2;
  const double* swap;  // 0.0 / 1.0
  const double* z;     // cyclic correction vector
  const double* rinv;  // RN(1/d) per row (fused sweeps)
  const double* h;     // cyclic: B^-1 v, f = (h . rhs) / denom
  double vn, denom;
};

// Epilogue of a derivative pass: out = D | c*D | acc + c*D, c = per-node
// field or scalar.  Used to fuse the metric contractions of
// formulations.py:87-98 / 135-143 and the LAD sensor (164-176).
struct Epi {
  int mode;              // 0: D, 1: c*D, 2: acc + c*D
  const double* acc;     // may alias out
  const double* cfield;  // per-node coefficient or nullptr
  double cscal;
  // the same coefficient stored once per line of the last axis (metric terms
  // of an extruded grid; index idx / cdiv), for the kernels that know of it
  // (wd_deriv_scan.cuh); cdiv <= 1: none
  const double* ccomp = nullptr;
  int cdiv = 0;
  __device__ __forceinline__ double apply(double D, long long idx) const {
    if (mode == 0) return D;
    double c = cfield ? cfield[idx] : cscal;
    double t = c * D;
    if (mode == 1) return t;
    return acc[idx] + t;
  }
};

__device__ __forceinline__ long long line_base(const Geom& g, int axis, long long q) {
  long long base = 0;
  if (g.N <= 0xffffffffLL) {
    unsigned u = (unsigned)q;
#pragma unroll
    for (int a = kMaxDim - 1; a >= 0; --a) {
      if (a == axis) continue;
      const unsigned n = (unsigned)g.n[a];
      const unsigned qn = u / n;
      base += (long long)(u - qn * n) * g.s[a];
      u = qn;
    }
    return base;
  }
#pragma unroll
  for (int a = kMaxDim - 1; a >= 0; --a) {
    if (a == axis) continue;
    long long c = q % g.n[a];
    q /= g.n[a];
    base += c * g.s[a];
  }
  return base;
}

__device__ __forceinline__ void tri_solve_line(double* __restrict__ x, long long st,
                                               const TriDev& T) {
  const int n = T.n;
  if (n == 1) {
    x[0] = x[0] / T.d[0];
    return;
  }
  double hs = 0.0;  // cyclic: h . rhs in row order (oracle/wd.py:cyclic_apply)
  if (T.cyclic)
    for (int i = 0; i < n; ++i) hs = hs + T.h[i] * x[(long long)i * st];
  for (int i = 0; i < n - 1; ++i) {
    const double f = T.fact[i];
    double* xi = x + (long long)i * st;
    double* xj = xi + st;
    if (T.swap[i] != 0.0) {
      double t = *xi;
      double b1 = *xj;
      *xi = b1;
      *xj = t - f * b1;
    } else {
      *xj = *xj - f * *xi;
    }
  }
  x[(long long)(n - 1) * st] = x[(long long)(n - 1) * st] / T.d[n - 1];
  x[(long long)(n - 2) * st] =
      (x[(long long)(n - 2) * st] - T.du[n - 2] * x[(long long)(n - 1) * st]) / T.d[n - 2];
  for (int i = n - 3; i >= 0; --i) {
    double* xi = x + (long long)i * st;
    *xi = ((*xi - T.du[i] * xi[st]) - T.du2[i] * xi[2 * st]) / T.d[i];
  }
  if (T.cyclic) {
    const double f = hs / T.denom;
    for (int i = 0; i < n; ++i) {
      double* xi = x + (long long)i * st;
      *xi = *xi - f * T.z[i];
    }
  }
}

// ---------------------------------------------------------------- kernels

// Explicit first derivative along `axis` (operators.py:109-128) + epilogue.
static __global__ void k_deriv_explicit(const double* __restrict__ in, double* out, AxisGeom ag,
                                 int scheme, int per, double off, Epi epi, const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  const long long sa = ag.sa;
  const int n = ag.n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < ag.N;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = ag.coord(idx);
    Line w{in + (idx - (long long)i * sa), sa, n, per, off};
    out[idx] = epi.apply(deriv_explicit_at(w, i, n, scheme, per), idx);
  }
}

// Compact first derivative: RHS + dgtsv-order solve per line
// (operators.py:130-148, 53-78).  One thread per grid line; `scratch`
// holds the raw solution (may equal out when epi.mode == 0).
static __global__ void k_deriv_compact(const double* __restrict__ in, double* scratch, double* out,
                                Geom g, int axis, int scheme, int per, double off, TriDev T,
                                Epi epi, const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  const long long sa = pick(g.s, axis);
  const int n = pick(g.n, axis);
  const long long L = g.N / n;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < L;
       q += (long long)gridDim.x * blockDim.x) {
    const long long base = line_base(g, axis, q);
    Line w{in + base, sa, n, per, off};
    double* x = scratch + base;
    for (int i = 0; i < n; ++i) x[(long long)i * sa] = compact_rhs_at(w, i, n, scheme, per);
    tri_solve_line(x, sa, T);
    if (epi.mode != 0 || out != scratch)
      for (int i = 0; i < n; ++i) {
        const long long idx = base + (long long)i * sa;
        out[idx] = epi.apply(scratch[idx], idx);
      }
  }
}

// 4th derivative (operators.py:236-250) + epilogue.
static __global__ void k_d4(const double* __restrict__ in, double* out, AxisGeom ag, int per,
                     Epi epi, const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  const long long sa = ag.sa;
  const int n = ag.n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < ag.N;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = ag.coord(idx);
    Line w{in + (idx - (long long)i * sa), sa, n, per, 0.0};
    out[idx] = epi.apply(d4_at(w, i, n, per), idx);
  }
}

// Implicit filter along `axis` (operators.py:305-352).  hc[h*6+k] holds
// the folded row coefficients: k = 0 -> a_0, k >= 1 -> 0.5*a_k of the
// half-order-h filter (operators.py:269-302).  pin: explicit pinned array
// (wd_filter) or, when use_geom_pin, walls + solid mask of g
// (BoundarySpec.pinned_mask solver.py:59-70).
struct FilterCoef {
  double hc[6 * 6];
};

static __global__ void k_filter(const double* __restrict__ in, double* out, Geom g, int axis, int per,
                         FilterCoef fc, TriDev T, const uint8_t* pin, int use_geom_pin,
                         const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  const long long sa = pick(g.s, axis);
  const int n = pick(g.n, axis);
  const long long L = g.N / n;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < L;
       q += (long long)gridDim.x * blockDim.x) {
    const long long base = line_base(g, axis, q);
    Line w{in + base, sa, n, per, 0.0};
    double* x = out + base;
    if (n < 3 && !per) {
      for (int i = 0; i < n; ++i) x[(long long)i * sa] = w(i);
      continue;
    }
    for (int i = 0; i < n; ++i) {
      double r;
      int h;
      if (per) {
        h = 5;
      } else if (i == 0 || i == n - 1) {
        h = 0;
      } else {
        h = min(min(i, n - 1 - i), 5);
      }
      if (h == 0) {
        r = w(i);
      } else {
        const double* c = fc.hc + h * 6;
        r = c[0] * w(i);
        for (int k = 1; k <= h; ++k) r = r + c[k] * (w(i + k) + w(i - k));
      }
      x[(long long)i * sa] = r;
    }
    tri_solve_line(x, sa, T);
    for (int i = 0; i < n; ++i) {
      const long long idx = base + (long long)i * sa;
      bool p;
      if (use_geom_pin) {
        int c[kMaxDim];
        node_coords(g, idx, c);
        p = is_pinned(g, idx, c);
      } else {
        p = pin != nullptr && pin[idx] != 0;
      }
      if (p) out[idx] = in[idx];
    }
  }
}

__device__ __forceinline__ double sign1(double x) { return x >= 0.0 ? 1.0 : -1.0; }

// UW one-sided differences + front-selected derivative
// (operators.py:151-193).
static __global__ void k_uw_bf(const double* __restrict__ in, double* Bo, double* Fo, double* dphi,
                        AxisGeom ag, int per, const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  const long long sa = ag.sa;
  const int n = ag.n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < ag.N;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = ag.coord(idx);
    Line w{in + (idx - (long long)i * sa), sa, n, per, 0.0};
    double B, F;
    if (per) {
      B = w(i) - w(i - 1);
      F = w(i + 1) - w(i);
    } else {
      B = i > 0 ? w(i) - w(i - 1) : w(1) - w(0);
      F = i < n - 1 ? w(i + 1) - w(i) : w(n - 1) - w(n - 2);
    }
    const double s_fb = sign1(F + B);
    const double nim1 = 0.25 * (1.0 + s_fb) * (1.0 + sign1(B));
    const double nip1 = 0.25 * (1.0 - s_fb) * (1.0 - sign1(F));
    Bo[idx] = B;
    Fo[idx] = F;
    dphi[idx] = nim1 * B + nip1 * F;
  }
}

struct Vec3 {
  const double* p[kMaxDim];
};
struct MVec3 {
  double* p[kMaxDim];
};

// U_m = sum_l M[l,m] dphi_l ; Uhat_l = sum_m M[l,m] U_m
// (formulations.py:87-98, Python sum order).
// nzm: bit l*nd+m set when M[l,m] is not identically zero (k_metric_nonzero);
// a skipped term is +-0, which leaves a running sum unchanged (up to the
// sign of an all-zero sum), so the result equals the full sum.
// Optional pointwise products of the same node, computed here from the
// registers instead of re-reading U / U_hat / dphi in later kernels
// (expressions identical to k_tendency / k_normal, so bit-identical):
//   adv = sum_l Uhat_l dphi_l        (formulations.py:114-121, central)
//   gmo = |grad phi| = sqrt(sum U^2)  (formulations.py:207)
//   nrm = U / (|grad phi| + eps0)     (formulations.py:212-214)
//   uabs = sum_l |Uhat_l|             (solver.py:170, k_timestep's order)
// U_hat itself is then only written when Uh.p[0] != nullptr.
struct AsmExtra {
  double* adv;
  double* gm;
  MVec3 nrm;
  double eps0;
  double* uabs;
};

// M[l, m] at node idx with a compile-time dimension (constant field offsets)
template <int ND>
__device__ __forceinline__ double mget(const Metric& M, int l, int m, long long idx) {
  if (M.m == nullptr) return l == m ? pick(M.c, l) : 0.0;
  if (M.kdiv > 1)  // compact terms (N < 2^32 whenever they are built)
    return M.m[(long long)(l * ND + m) * M.N + (unsigned)idx / (unsigned)M.kdiv];
  return M.m[(long long)(l * ND + m) * M.N + idx];
}

template <int ND>
static __global__ void k_assemble(Vec3 dphi, Metric M, MVec3 U, MVec3 Uh, long long N, int nd_,
                                  unsigned nzm, AsmExtra x, const Status* st) {
  constexpr int nd = ND;
  if (st && st->state != WD_STATE_RUNNING) return;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
    double d[kMaxDim], u[kMaxDim];
#pragma unroll
    for (int l = 0; l < kMaxDim; ++l) d[l] = l < nd ? dphi.p[l][idx] : 0.0;
#pragma unroll
    for (int m = 0; m < kMaxDim; ++m) {
      if (m >= nd) break;
      double s = 0.0;
      bool any = false;
#pragma unroll
      for (int l = 0; l < kMaxDim; ++l)
        if (l < nd && ((nzm >> (l * nd + m)) & 1u)) {
          const double t = mget<ND>(M, l, m, idx) * d[l];
          s = any ? s + t : t;
          any = true;
        }
      u[m] = s;
      U.p[m][idx] = s;
    }
    double adv = 0.0, ua = 0.0;
    if (Uh.p[0] != nullptr || x.adv || x.uabs)
#pragma unroll
      for (int l = 0; l < kMaxDim; ++l) {
        if (l >= nd) break;
        double s = 0.0;
        bool any = false;
#pragma unroll
        for (int m = 0; m < kMaxDim; ++m)
          if (m < nd && ((nzm >> (l * nd + m)) & 1u)) {
            const double t = mget<ND>(M, l, m, idx) * u[m];
            s = any ? s + t : t;
            any = true;
          }
        if (Uh.p[0] != nullptr) Uh.p[l][idx] = s;
        if (x.adv) {
          const double t = s * d[l];
          adv = l == 0 ? t : adv + t;
        }
        ua = l == 0 ? fabs(s) : ua + fabs(s);
      }
    if (x.adv) x.adv[idx] = adv;
    if (x.uabs) x.uabs[idx] = ua;
    if (x.gm) {
      double s = 0.0;
#pragma unroll
      for (int m = 0; m < kMaxDim; ++m) {
        if (m >= nd) break;
        s = m == 0 ? u[0] * u[0] : s + u[m] * u[m];
      }
      const double gm = sqrt(s);
      x.gm[idx] = gm;
      if (x.nrm.p[0])
#pragma unroll
        for (int m = 0; m < kMaxDim; ++m)
          if (m < nd) x.nrm.p[m][idx] = u[m] / (gm + x.eps0);
    }
  }
}

// k_assemble for two consecutive nodes per thread (N even): 16-byte loads and
// stores, twice the bytes in flight per thread -- one node per thread with
// ~150 (U only) to 400 (curvature extras) instructions left the kernel bound
// by load latency at half occupancy (2.5-3.6 TB/s) -- and the set of
// non-zero metric terms as a template parameter (NZ != 0: the bit tests and
// the first-term selects of the sums fold away; NZ == 0: run-time nzm).
// Every expression is k_assemble's, per node, so the results are identical.
// UONLY: only U is wanted (Poisson, the UW Laplacian's E2 gradient): the
// instantiation carries none of the optional outputs' registers (40 instead
// of ~100: three times the resident warps).
template <int ND, unsigned NZ, bool UONLY = false>
static __global__ void __launch_bounds__(256) k_assemble2(Vec3 dphi, Metric M, MVec3 U, MVec3 Uh,
                                                          long long N, unsigned nzm, AsmExtra x,
                                                          const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  const unsigned nz = NZ ? NZ : nzm;
  const long long half = N >> 1;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < half;
       q += (long long)gridDim.x * blockDim.x) {
    const long long idx = 2 * q;
    double d[ND][2], mm[ND * ND][2];
#pragma unroll
    for (int l = 0; l < ND; ++l) {
      const double2 v = *reinterpret_cast<const double2*>(dphi.p[l] + idx);
      d[l][0] = v.x;
      d[l][1] = v.y;
    }
    // compact terms: idx and idx + 1 lie on one line of the last axis (kdiv even)
    const long long mi = M.kdiv > 1 ? (long long)((unsigned)idx / (unsigned)M.kdiv) : idx;
#pragma unroll
    for (int t = 0; t < ND * ND; ++t) {
      mm[t][0] = mm[t][1] = 0.0;
      if ((nz >> t) & 1u) {
        if (M.m == nullptr) {
          mm[t][0] = mm[t][1] = (t / ND == t % ND) ? pick(M.c, t / ND) : 0.0;
        } else if (M.kdiv > 1) {
          mm[t][0] = mm[t][1] = M.m[(long long)t * M.N + mi];
        } else {
          const double2 v = *reinterpret_cast<const double2*>(M.m + (long long)t * M.N + idx);
          mm[t][0] = v.x;
          mm[t][1] = v.y;
        }
      }
    }
    double u[ND][2], uh[ND][2], adv[2] = {0.0, 0.0}, ua[2] = {0.0, 0.0}, gm[2] = {0.0, 0.0};
    double nr[ND][2];
    const bool second = !UONLY && (Uh.p[0] != nullptr || x.adv || x.uabs);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
#pragma unroll
      for (int m = 0; m < ND; ++m) {
        double sacc = 0.0;
        bool any = false;
#pragma unroll
        for (int l = 0; l < ND; ++l)
          if ((nz >> (l * ND + m)) & 1u) {
            const double t = mm[l * ND + m][e] * d[l][e];
            sacc = any ? sacc + t : t;
            any = true;
          }
        u[m][e] = sacc;
      }
      if (second) {
#pragma unroll
        for (int l = 0; l < ND; ++l) {
          double sacc = 0.0;
          bool any = false;
#pragma unroll
          for (int m = 0; m < ND; ++m)
            if ((nz >> (l * ND + m)) & 1u) {
              const double t = mm[l * ND + m][e] * u[m][e];
              sacc = any ? sacc + t : t;
              any = true;
            }
          uh[l][e] = sacc;
          if (x.adv) {
            const double t = sacc * d[l][e];
            adv[e] = l == 0 ? t : adv[e] + t;
          }
          ua[e] = l == 0 ? fabs(sacc) : ua[e] + fabs(sacc);
        }
      }
      if (!UONLY && x.gm) {
        double sq = 0.0;
#pragma unroll
        for (int m = 0; m < ND; ++m) sq = m == 0 ? u[0][e] * u[0][e] : sq + u[m][e] * u[m][e];
        gm[e] = sqrt(sq);
        if (x.nrm.p[0])
#pragma unroll
          for (int m = 0; m < ND; ++m) nr[m][e] = u[m][e] / (gm[e] + x.eps0);
      }
    }
    auto put = [&](double* f, const double v[2]) {
      *reinterpret_cast<double2*>(f + idx) = make_double2(v[0], v[1]);
    };
#pragma unroll
    for (int m = 0; m < ND; ++m) put(U.p[m], u[m]);
    if (UONLY) continue;
    if (second && Uh.p[0] != nullptr)
#pragma unroll
      for (int l = 0; l < ND; ++l) put(Uh.p[l], uh[l]);
    if (x.adv) put(x.adv, adv);
    if (x.uabs) put(x.uabs, ua);
    if (x.gm) {
      put(x.gm, gm);
      if (x.nrm.p[0])
#pragma unroll
        for (int m = 0; m < ND; ++m) put(x.nrm.p[m], nr[m]);
    }
  }
}

// Curvature normal n_m = U_m / (|U| + eps0) (formulations.py:212-214).
static __global__ void k_normal(Vec3 U, MVec3 nrm, long long N, int nd, double eps0,
                         const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
    double u[kMaxDim];
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < kMaxDim; ++m) {
      if (m >= nd) break;
      u[m] = U.p[m][idx];
      s = m == 0 ? u[0] * u[0] : s + u[m] * u[m];
    }
    const double gm = sqrt(s);
#pragma unroll
    for (int m = 0; m < kMaxDim; ++m)
      if (m < nd) nrm.p[m][idx] = u[m] / (gm + eps0);
  }
}

// LAD diffusivity min(eps phi, C |sensor|) (formulations.py:175-176).
static __global__ void k_gamma_lad(const double* __restrict__ p, const double* __restrict__ sensor,
                            double* gam, long long N, double eps, double c, const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x)
    gam[idx] = np_min(eps * p[idx], c * fabs(sensor[idx]));
}

struct ResidualArgs {
  int kind, scheme, nd;
  double eps;
  const double* p;
  const double* lap;
  const double* gam;    // LAD gamma or nullptr
  const double* kappa;  // curvature
  const double* adv;    // precomputed advection (k_assemble) or nullptr
  const double* gm;     // precomputed |grad phi| (k_assemble) or nullptr
  Vec3 U, Uh, dphi, B, F;
};

// Tendency (formulations.py:153-252) at one node.  UW advection:
// flux_from_bf (operators.py:216-219); central: Uhat . dphi.
__device__ __forceinline__ double residual_at(const ResidualArgs& a, long long idx) {
  if (a.kind == WD_POISSON) {
    const double r = -1.0 - a.lap[idx];
    return -r;
  }
  double adv = 0.0;
#pragma unroll
  for (int l = 0; l < kMaxDim; ++l) {
    if (l >= a.nd || a.adv) break;
    const double uh = a.Uh.p[l][idx];
    double t;
    if (a.scheme == WD_UW) {
      const double au = fabs(uh);
      t = 0.5 * ((uh + au) * a.B.p[l][idx] + (uh - au) * a.F.p[l][idx]);
    } else {
      t = uh * a.dphi.p[l][idx];
    }
    adv = l == 0 ? t : adv + t;
  }
  if (a.adv) adv = a.adv[idx];
  if (a.kind == WD_EIKONAL) return 1.0 - adv;
  if (a.kind == WD_HJ || a.kind == WD_HJ_LAD) {
    const double gam = a.kind == WD_HJ ? a.eps * a.p[idx] : a.gam[idx];
    return 1.0 + gam * a.lap[idx] - adv;
  }
  // WD_HJ_CURVATURE
  double gm;
  if (a.gm) {
    gm = a.gm[idx];
  } else {
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < kMaxDim; ++m) {
      if (m >= a.nd) break;
      const double u = a.U.p[m][idx];
      s = m == 0 ? u * u : s + u * u;
    }
    gm = sqrt(s);
  }
  const double om = 1.0 - gm;
  const double nu = 0.001 * (om * om);
  const double gam = a.eps * a.p[idx] + nu;
  const double corr = a.lap[idx] - np_max(0.0, gm * a.kappa[idx]);
  return 1.0 + gam * corr - adv;
}

static __global__ void k_tendency(ResidualArgs a, double* k, long long N, const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x)
    k[idx] = residual_at(a, idx);
}

struct DtArgs {
  int kind, nd;
  double eps, cfl;
  const double* p;
  const double* gam;     // LAD gamma
  Vec3 Uh;
  const double* uabs;    // precomputed sum |U_hat| (k_assemble) or nullptr
  const double* sumS;    // field or nullptr (then sumS_c)
  double sumS_c;
  const double* cflms;   // cfl * min_spacing field or nullptr
  double cflms_c;
};

// local_timestep (solver.py:160-180).
static __global__ void k_timestep(DtArgs a, double* dt, long long N, const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
    const double sS = a.sumS ? a.sumS[idx] : a.sumS_c;
    if (a.kind == WD_POISSON) {
      dt[idx] = a.cfl / (2.0 * sS);
      continue;
    }
    double den;
    if (a.uabs) {
      den = a.uabs[idx];
    } else {
      den = fabs(a.Uh.p[0][idx]);
#pragma unroll
      for (int l = 1; l < kMaxDim; ++l)
        if (l < a.nd) den = den + fabs(a.Uh.p[l][idx]);
    }
    if (a.kind == WD_HJ || a.kind == WD_HJ_CURVATURE)
      den = den + 2.0 * (a.eps * a.p[idx]) * sS;
    else if (a.kind == WD_HJ_LAD)
      den = den + 2.0 * a.gam[idx] * sS;
    const double d = a.cfl / (den + 1e-30);
    dt[idx] = np_min(d, a.cflms ? a.cflms[idx] : a.cflms_c);
  }
}

// RK4 stage update with the boundary conditions fused as a source
// redirect (solver.py:198-206 + 87-110).
//   stage 1..3: out = BC(phi + c(dt) k), c = 0.5*dt | 0.5*dt | dt
//   stage 2, 3 also: acc = acc + 2 k   (acc holds k1 after stage 1)
//   stage 4:  out = BC(phi + (dt/6)(acc + k))
// Node coordinates by successive division by the axis lengths (2 fast
// divisions in 3-D instead of a division and a modulo per axis).
template <int ND>
__device__ __forceinline__ void node_coords_nd(const Geom& g, long long idx, int c[kMaxDim]) {
  c[0] = c[1] = c[2] = 0;
  if (g.N <= 0xffffffffLL) {
    unsigned q = (unsigned)idx;
#pragma unroll
    for (int a = ND - 1; a > 0; --a) {
      const unsigned qn = fdiv(q, g.fn[a]);
      c[a] = (int)(q - qn * (unsigned)g.n[a]);
      q = qn;
    }
    c[0] = (int)q;
    return;
  }
  long long q = idx;
#pragma unroll
  for (int a = ND - 1; a > 0; --a) {
    c[a] = (int)(q % g.n[a]);
    q /= g.n[a];
  }
  c[0] = (int)q;
}

template <int ND>
static __global__ void k_rk_stage(int stage, const double* __restrict__ phi,
                                  const double* __restrict__ dt, const double* __restrict__ k,
                                  double* acc, double* out, Geom g, const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < g.N;
       idx += (long long)gridDim.x * blockDim.x) {
    int c[kMaxDim];
    node_coords_nd<ND>(g, idx, c);
    long long s = idx;
    bool pinned = false;
#pragma unroll
    for (int a = 0; a < ND; ++a) {  // bc_source / is_pinned, ND axes
      if (c[a] == 0) {
        if (g.face[2 * a] == WD_FACE_FARFIELD) s += g.s[a];
        if (g.face[2 * a] == WD_FACE_WALL) pinned = true;
      }
      if (c[a] == g.n[a] - 1) {
        if (g.face[2 * a + 1] == WD_FACE_FARFIELD) s -= g.s[a];
        if (g.face[2 * a + 1] == WD_FACE_WALL) pinned = true;
      }
    }
    if (g.mask != nullptr && g.mask[idx] != 0) pinned = true;
    double v;
    if (stage == 4) {
      v = phi[s] + (dt[s] / 6.0) * (acc[s] + k[s]);
    } else {
      const double cdt = stage == 3 ? dt[s] : 0.5 * dt[s];
      v = phi[s] + cdt * k[s];
    }
    out[idx] = pinned ? 0.0 : v;
    // stages 2/3 read acc nowhere else, so the accumulation rides along
    // (k[idx] is k[s] or its neighbour: one DRAM pass over k)
    if (stage == 2 || stage == 3) acc[idx] = acc[idx] + 2.0 * k[idx];
  }
}

// Sum of divergence terms evaluated concurrently (small grids): out =
// sum_t M[l_t, m_t] D_t in launch_divergence's order -- c D for the first
// term, acc + c D for the others, exactly the Epi chain of the serial path.
struct DivTerms {
  const double* D[9];
  int l[9], m[9];
  int count;
};
template <int ND>
static __global__ void k_div_combine(DivTerms t, Metric M, double* out, long long N,
                                     const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      if (q >= t.count) break;
      const double v = mget<ND>(M, t.l[q], t.m[q], idx) * t.D[q][idx];
      s = q == 0 ? v : s + v;
    }
    out[idx] = s;
  }
}

// k_tendency + k_rk_stage in one pass (the solve loop's generic path): the
// residual is pointwise in the assembled fields, so the stage update
// evaluates it at its source node (and at the node itself for the running
// sum acc) instead of reading a stored k.  Same expressions, bit-identical.
template <int ND>
static __global__ void k_tend_rk(int stage, ResidualArgs a, const double* __restrict__ phi,
                                 const double* __restrict__ dt, double* acc, double* out, Geom g,
                                 const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < g.N;
       idx += (long long)gridDim.x * blockDim.x) {
    int c[kMaxDim];
    node_coords_nd<ND>(g, idx, c);
    long long s = idx;
    bool pinned = false;
#pragma unroll
    for (int ax = 0; ax < ND; ++ax) {
      if (c[ax] == 0) {
        if (g.face[2 * ax] == WD_FACE_FARFIELD) s += g.s[ax];
        if (g.face[2 * ax] == WD_FACE_WALL) pinned = true;
      }
      if (c[ax] == g.n[ax] - 1) {
        if (g.face[2 * ax + 1] == WD_FACE_FARFIELD) s -= g.s[ax];
        if (g.face[2 * ax + 1] == WD_FACE_WALL) pinned = true;
      }
    }
    if (g.mask != nullptr && g.mask[idx] != 0) pinned = true;
    const bool moved = s != idx;
    const double k_me = (stage != 4 || !moved) ? residual_at(a, idx) : 0.0;
    const double k_s = moved ? residual_at(a, s) : k_me;
    double v;
    if (stage == 4) {
      v = phi[s] + (dt[s] / 6.0) * (acc[s] + k_s);
    } else {
      const double cdt = stage == 3 ? dt[s] : 0.5 * dt[s];
      v = phi[s] + cdt * k_s;
    }
    out[idx] = pinned ? 0.0 : v;
    if (stage == 1) acc[idx] = k_me;
    if (stage == 2 || stage == 3) acc[idx] = acc[idx] + 2.0 * k_me;
  }
}

// Out-of-place boundary conditions (solver.py:87-110).
static __global__ void k_bc(const double* __restrict__ in, double* out, Geom g, const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < g.N;
       idx += (long long)gridDim.x * blockDim.x) {
    int c[kMaxDim];
    node_coords(g, idx, c);
    out[idx] = is_pinned(g, idx, c) ? 0.0 : in[bc_source(g, idx, c)];
  }
}

__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// max |new - old| over active nodes, max |new|, non-finite flag
// (solver.py:214-217, 253-256).  max is order-free -> deterministic.
static __global__ void k_change(const double* __restrict__ nw, const double* __restrict__ old,
                         const uint8_t* mask, Status* st, long long N) {
  if (st->state != WD_STATE_RUNNING) return;
  double md = 0.0, ma = 0.0;
  int bad = 0;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
    const double v = nw[idx];
    if (!isfinite(v)) bad = 1;
    ma = fmax(ma, fabs(v));
    if (mask == nullptr || mask[idx] == 0) md = fmax(md, fabs(v - old[idx]));
  }
  md = warp_max(md);
  ma = warp_max(ma);
  bad = __any_sync(0xffffffffu, bad);
  __shared__ double smd[32], sma[32];
  __shared__ int sbad[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    smd[wid] = md;
    sma[wid] = ma;
    sbad[wid] = bad;
  }
  __syncthreads();
  if (wid == 0) {
    const int nw_ = blockDim.x >> 5;
    md = lane < nw_ ? smd[lane] : 0.0;
    ma = lane < nw_ ? sma[lane] : 0.0;
    bad = lane < nw_ ? sbad[lane] : 0;
    md = warp_max(md);
    ma = warp_max(ma);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      atomicMax(&st->max_delta_bits, (unsigned long long)__double_as_longlong(md));
      atomicMax(&st->max_abs_bits, (unsigned long long)__double_as_longlong(ma));
      if (bad) atomicOr(&st->nonfinite, 1);
    }
  }
}

// k_bc + k_change in one pass: out = BC(in), and the running maxima of
// |out - old| (unmasked nodes), |out| and the non-finite flag.
static __global__ void k_bc_change(const double* __restrict__ in, double* out,
                                   const double* __restrict__ old, Geom g, Status* st) {
  pdl_trigger();
  pdl_wait();
  if (st->state != WD_STATE_RUNNING) return;
  double md = 0.0, ma = 0.0;
  int bad = 0;
  // four nodes a grid stride apart per iteration, their loads issued before
  // any store (one node per iteration: 1.12 ms for 3 words at 1024 x 512 x 256)
  constexpr int U = 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < g.N;
       idx += U * stride) {
    double v[U], o[U];
    bool cmp[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = idx + u * stride;
      v[u] = o[u] = 0.0;
      cmp[u] = false;
      if (i < g.N) {
        int c[kMaxDim];
        node_coords(g, i, c);
        v[u] = is_pinned(g, i, c) ? 0.0 : in[bc_source(g, i, c)];
        cmp[u] = g.mask == nullptr || g.mask[i] == 0;
        if (cmp[u]) o[u] = old[i];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = idx + u * stride;
      if (i < g.N) {
        out[i] = v[u];
        if (!isfinite(v[u])) bad = 1;
        ma = fmax(ma, fabs(v[u]));
        if (cmp[u]) md = fmax(md, fabs(v[u] - o[u]));
      }
    }
  }
  md = warp_max(md);
  ma = warp_max(ma);
  bad = __any_sync(0xffffffffu, bad);
  __shared__ double smd[32], sma[32];
  __shared__ int sbad[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    smd[wid] = md;
    sma[wid] = ma;
    sbad[wid] = bad;
  }
  __syncthreads();
  if (wid == 0) {
    const int nw_ = blockDim.x >> 5;
    md = lane < nw_ ? smd[lane] : 0.0;
    ma = lane < nw_ ? sma[lane] : 0.0;
    bad = lane < nw_ ? sbad[lane] : 0;
    md = warp_max(md);
    ma = warp_max(ma);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      atomicMax(&st->max_delta_bits, (unsigned long long)__double_as_longlong(md));
      atomicMax(&st->max_abs_bits, (unsigned long long)__double_as_longlong(ma));
      if (bad) atomicOr(&st->nonfinite, 1);
    }
  }
}

// Stop test + history (solver.py:253-272).
static __global__ void k_finalize(Status* st, double* hist, double lref, double tol, double limit) {
  pdl_trigger();
  pdl_wait();
  if (st->state == WD_STATE_RUNNING) {
    const double ma = __longlong_as_double((long long)st->max_abs_bits);
    if (st->nonfinite || ma > limit) {
      st->state = WD_STATE_DIVERGED;
      st->diverged_iter = st->iters + 1;
    } else {
      const double change = __longlong_as_double((long long)st->max_delta_bits) / lref;
      hist[st->iters] = change;
      st->iters += 1;
      if (change <= tol)
        st->state = WD_STATE_CONVERGED;
      else if (st->iters >= st->max_iters)
        st->state = WD_STATE_MAXITERS;
    }
  }
  st->max_delta_bits = 0ull;
  st->max_abs_bits = 0ull;
  st->nonfinite = 0;
}

// Poisson post-map (formulations.py:255-270): clip, radicand, sqrt.
static __global__ void k_poisson_clip(const double* __restrict__ pp, double* out, long long N) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
    const double v = pp[idx];
    out[idx] = (v < 0.0 && v > -1e-12) ? 0.0 : v;
  }
}

static __global__ void k_poisson_map(const double* __restrict__ pp, Vec3 U, double* out, long long N,
                              int nd, int* negative) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
    double gs = 0.0;
#pragma unroll
    for (int m = 0; m < kMaxDim; ++m) {
      if (m >= nd) break;
      const double u = U.p[m][idx];
      gs = m == 0 ? u * u : gs + u * u;
    }
    double rad = gs + 2.0 * pp[idx];
    if (rad < -1e-12) atomicOr(negative, 1);
    rad = np_max(rad, 0.0);
    out[idx] = -sqrt(gs) + sqrt(rad);
  }
}

// Per-node metric sums (grid.py:60-73): sumS = sum_l S_l, cfl*min spacing,
// sqrt(S_l) for the LAD sensor.
static __global__ void k_metric_sums(Metric M, double* sumS, double* cflms, double* sqrtS, double cfl,
                              long long N, int nd) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
    double tot = 0.0, ms = 0.0;
    for (int l = 0; l < nd; ++l) {
      double S = M.get(l, 0, idx) * M.get(l, 0, idx);
      for (int m = 1; m < nd; ++m) S = S + M.get(l, m, idx) * M.get(l, m, idx);
      tot = l == 0 ? S : tot + S;
      const double sq = sqrt(S);
      const double sp = 1.0 / sq;
      ms = l == 0 ? sp : np_min(ms, sp);
      sqrtS[(long long)l * N + idx] = sq;
    }
    sumS[idx] = tot;
    cflms[idx] = cfl * ms;
  }
}

// Which metric terms M[l, m] are not identically +-0 over the grid
// (blockIdx.y = l * nd + m; NaN counts as nonzero).  Terms that are zero at
// every node contribute exactly +-0 to the divergence sums of
// formulations.py:135-143, so the generic path skips their line solves
// (O-grids with a straight axis: 4 of 9 terms in 3-D).
static __global__ void k_metric_nonzero(const double* __restrict__ m, long long N, int* flags) {
  const double* f = m + (long long)blockIdx.y * N;
  bool nz = false;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x)
    nz |= !(f[idx] == 0.0);
  if (__syncthreads_or(nz) && threadIdx.x == 0) atomicOr(flags + blockIdx.y, 1);
}

// Metric terms that do not vary along the last axis (an O-grid extruded along
// z: BASELINE config 5) need one value per (i, j).  Computed metrics agree
// along such an axis only to round-off (z_k = k dz differenced: a few ulp;
// cross terms that are analytically zero come out as 1e-13 noise), so the
// test is |M - M_first| <= 1e-12 x the node's largest term; flag = 1 if any
// node fails it.  The gather keeps each line's first node.  Only the
// fast-arithmetic kernels read the compact copy (L2-resident: 4 MB per term
// instead of 1 GB at 1024 x 512 x 256); exact arithmetic never does.
constexpr double kKMetricTol = 1e-12;
static __global__ void k_metric_kvar(const double* __restrict__ m, long long N, int n2, int nt,
                                     int* flag) {
  bool var = false;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long first = idx - idx % n2;
    double sc = 0.0;
    for (int t = 0; t < nt; ++t) sc = fmax(sc, fabs(m[t * N + first]));
    for (int t = 0; t < nt; ++t)
      var |= !(fabs(m[t * N + idx] - m[t * N + first]) <= kKMetricTol * sc);
  }
  if (__syncthreads_or(var) && threadIdx.x == 0) atomicOr(flag, 1);
}
static __global__ void k_metric_kgather(const double* __restrict__ m, double* out, long long N,
                                        int n2, int nt) {
  const long long Nk = N / n2;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < Nk * nt;
       q += (long long)gridDim.x * blockDim.x) {
    const long long t = q / Nk, j = q - t * Nk;
    out[q] = m[t * N + j * n2];
  }
}

// 2-D / 3-D metric inversion (grid.py:196-216).  fwd[m*d+l] = dx_m/dxi_l.
static __global__ void k_metric_invert(const double* __restrict__ fwd, double* met, double* jac,
                                long long N, int nd, int* singular) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
#define A(m, l) fwd[(long long)((m) * nd + (l)) * N + idx]
#define O(l, m) met[(long long)((l) * nd + (m)) * N + idx]
    if (nd == 2) {
      const double det = A(0, 0) * A(1, 1) - A(0, 1) * A(1, 0);
      if (fabs(det) < 1e-14 || det != det) atomicOr(singular, 1);
      const double inv = 1.0 / det;
      O(0, 0) = A(1, 1) * inv;
      O(0, 1) = -A(0, 1) * inv;
      O(1, 0) = -A(1, 0) * inv;
      O(1, 1) = A(0, 0) * inv;
      jac[idx] = inv;
    } else {
      const double c00 = A(1, 1) * A(2, 2) - A(1, 2) * A(2, 1);
      const double c01 = A(1, 2) * A(2, 0) - A(1, 0) * A(2, 2);
      const double c02 = A(1, 0) * A(2, 1) - A(1, 1) * A(2, 0);
      const double det = A(0, 0) * c00 + A(0, 1) * c01 + A(0, 2) * c02;
      if (fabs(det) < 1e-14 || det != det) atomicOr(singular, 1);
      const double inv = 1.0 / det;
      O(0, 0) = c00 * inv;
      O(1, 0) = c01 * inv;
      O(2, 0) = c02 * inv;
      O(0, 1) = (A(0, 2) * A(2, 1) - A(0, 1) * A(2, 2)) * inv;
      O(1, 1) = (A(0, 0) * A(2, 2) - A(0, 2) * A(2, 0)) * inv;
      O(2, 1) = (A(0, 1) * A(2, 0) - A(0, 0) * A(2, 1)) * inv;
      O(0, 2) = (A(0, 1) * A(1, 2) - A(0, 2) * A(1, 1)) * inv;
      O(1, 2) = (A(0, 2) * A(1, 0) - A(0, 0) * A(1, 2)) * inv;
      O(2, 2) = (A(0, 0) * A(1, 1) - A(0, 1) * A(1, 0)) * inv;
      jac[idx] = inv;
    }
#undef A
#undef O
  }
}

static __global__ void k_linf(const double* __restrict__ a, const double* __restrict__ b,
                       const uint8_t* mask, unsigned long long* out, long long N) {
  double md = 0.0;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x)
    if (mask == nullptr || mask[idx] == 0) md = fmax(md, fabs(a[idx] - b[idx]));
  md = warp_max(md);
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(md));
}

}  // namespace wd
