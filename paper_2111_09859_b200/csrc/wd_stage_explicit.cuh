// Two-kernel RK stage for explicit central schemes on 2-D grids (BASELINE
// configs 1 and 3: 20 k - 526 k nodes, uniform or curvilinear, Eikonal / HJ).
//
// The generic path runs a stage as 8-9 launches in the reference's structure
// (one derivative per axis, metric contraction, one derivative per
// divergence term, residual, RK update); on grids this small every launch
// costs more than its work (C1: 36 launches per step for 20 k nodes).  Here
//   k_ex_grad    per node: the gradient along every axis, the contravariant
//                velocities U_m (stored: the divergence differentiates them),
//                the advection product and -- stage 1 -- the local time step;
//   k_ex_update  per node: lap = sum_m sum_l M[l,m] D_l(U_m) from the stored
//                U_m, the residual, and the RK update with the boundary
//                conditions as the source redirect of k_rk_stage.
// Every expression is the one the multi-kernel path evaluates
// (k_deriv_explicit, k_assemble, the Epi accumulation of launch_divergence,
// k_tendency, k_timestep, k_rk_stage), in the same order on the same
// operands, so the results are bit-identical (tests/test_gpu_parity.py runs
// both paths against the reference goldens).  (A single kernel per stage that
// re-evaluates U_m at the stencil neighbours was measured 2-3x slower: ~400
// loads per node instead of ~50.)
#pragma once

#include "wd_kernels.cuh"

namespace wd {

struct ExArgs {
  const double* A;    // phi at the start of the step
  const double* p;    // stage input (A for stage 1)
  double* out;        // stage output
  double* dt;
  double* acc;
  double* U[2];       // contravariant velocities of the stage input
  double* adv;        // advection product of the stage input
  Geom g;
  Metric M;
  unsigned nzm;       // bit l * nd + m: metric term not identically zero
  int scheme, kind;
  double eps, cfl;
  const double* sumS;   // per node or nullptr (then sumS_c)
  double sumS_c;
  const double* cflms;  // cfl * min spacing per node or nullptr
  double cflms_c;
  const Status* st;
};

template <int ND, bool DT>
static __global__ void __launch_bounds__(256) k_ex_grad(ExArgs a) {
  pdl_trigger();
  pdl_wait();
  if (a.st && a.st->state != WD_STATE_RUNNING) return;
  const Geom& g = a.g;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < g.N;
       idx += (long long)gridDim.x * blockDim.x) {
    int c[kMaxDim];
    node_coords_nd<ND>(g, idx, c);
    double d[ND], u[ND];
#pragma unroll
    for (int l = 0; l < ND; ++l) {  // k_deriv_explicit
      const long long sl = g.s[l];
      Line w{a.p + (idx - (long long)c[l] * sl), sl, g.n[l], g.per[l], 0.0};
      d[l] = deriv_explicit_at(w, c[l], g.n[l], a.scheme, g.per[l]);
    }
#pragma unroll
    for (int m = 0; m < ND; ++m) {  // k_assemble: U_m
      double s = 0.0;
      bool any = false;
#pragma unroll
      for (int l = 0; l < ND; ++l)
        if ((a.nzm >> (l * ND + m)) & 1u) {
          const double t = mget<ND>(a.M, l, m, idx) * d[l];
          s = any ? s + t : t;
          any = true;
        }
      u[m] = s;
      a.U[m][idx] = s;
    }
    double adv = 0.0, ua = 0.0;
#pragma unroll
    for (int l = 0; l < ND; ++l) {  // k_assemble: U_hat_l, advection, sum |U_hat|
      double s = 0.0;
      bool any = false;
#pragma unroll
      for (int m = 0; m < ND; ++m)
        if ((a.nzm >> (l * ND + m)) & 1u) {
          const double t = mget<ND>(a.M, l, m, idx) * u[m];
          s = any ? s + t : t;
          any = true;
        }
      const double t = s * d[l];
      adv = l == 0 ? t : adv + t;
      ua = l == 0 ? fabs(s) : ua + fabs(s);
    }
    a.adv[idx] = adv;
    if (DT) {  // k_timestep
      double den = ua;
      if (a.kind == WD_HJ)
        den = den + 2.0 * (a.eps * a.p[idx]) * (a.sumS ? a.sumS[idx] : a.sumS_c);
      const double q = a.cfl / (den + 1e-30);
      a.dt[idx] = np_min(q, a.cflms ? a.cflms[idx] : a.cflms_c);
    }
  }
}

// tendency at node e (coordinates ce) from the stored U / adv fields
template <int ND>
__device__ __forceinline__ double ex_tend(const ExArgs& a, long long e, const int ce[kMaxDim]) {
  const double adv = a.adv[e];
  if (a.kind == WD_EIKONAL) return 1.0 - adv;
  double lap = 0.0;
  bool first = true;
#pragma unroll
  for (int m = 0; m < ND; ++m)
#pragma unroll
    for (int l = 0; l < ND; ++l) {  // launch_divergence: m outer, l inner
      if (a.M.m == nullptr ? l != m : !((a.nzm >> (l * ND + m)) & 1u)) continue;
      const long long sl = a.g.s[l];
      Line w{a.U[m] + (e - (long long)ce[l] * sl), sl, a.g.n[l], a.g.per[l], 0.0};
      const double D = deriv_explicit_at(w, ce[l], a.g.n[l], a.scheme, a.g.per[l]);
      const double t = mget<ND>(a.M, l, m, e) * D;
      lap = first ? t : lap + t;
      first = false;
    }
  return 1.0 + (a.eps * a.p[e]) * lap - adv;
}

template <int ND, int STAGE>
static __global__ void __launch_bounds__(256) k_ex_update(ExArgs a) {
  pdl_trigger();
  pdl_wait();
  if (a.st && a.st->state != WD_STATE_RUNNING) return;
  const Geom& g = a.g;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < g.N;
       idx += (long long)gridDim.x * blockDim.x) {
    int c[kMaxDim], cs[kMaxDim];
    node_coords_nd<ND>(g, idx, c);
    long long s = idx;
    bool pinned = false;
#pragma unroll
    for (int ax = 0; ax < kMaxDim; ++ax) cs[ax] = c[ax];
#pragma unroll
    for (int ax = 0; ax < ND; ++ax) {  // bc_source / is_pinned of k_rk_stage
      if (c[ax] == 0) {
        if (g.face[2 * ax] == WD_FACE_FARFIELD) { s += g.s[ax]; cs[ax] += 1; }
        if (g.face[2 * ax] == WD_FACE_WALL) pinned = true;
      }
      if (c[ax] == g.n[ax] - 1) {
        if (g.face[2 * ax + 1] == WD_FACE_FARFIELD) { s -= g.s[ax]; cs[ax] -= 1; }
        if (g.face[2 * ax + 1] == WD_FACE_WALL) pinned = true;
      }
    }
    if (g.mask != nullptr && g.mask[idx] != 0) pinned = true;
    const bool moved = s != idx;
    const bool need_me = STAGE != 4 || !moved;
    const double k_me = need_me ? ex_tend<ND>(a, idx, c) : 0.0;
    const double k_s = moved ? ex_tend<ND>(a, s, cs) : k_me;
    const double dts = a.dt[s];
    double v;
    if (STAGE == 4) {
      v = a.A[s] + (dts / 6.0) * (a.acc[s] + k_s);
    } else {
      const double cdt = STAGE == 3 ? dts : 0.5 * dts;
      v = a.A[s] + cdt * k_s;
    }
    a.out[idx] = pinned ? 0.0 : v;
    if (STAGE == 1) a.acc[idx] = k_me;
    if (STAGE == 2 || STAGE == 3) a.acc[idx] = a.acc[idx] + 2.0 * k_me;
  }
}

}  // namespace wd
