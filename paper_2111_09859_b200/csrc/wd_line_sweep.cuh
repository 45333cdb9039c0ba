// Generic line solves (compact first derivative, operators.py:130-148, and
// implicit filter, operators.py:305-352) for the generic path, in two
// kernels:
//
//   k_line_rhs    every node in parallel: the right-hand side row
//                 (compact_rhs_at / the filter row of half-order h) into a
//                 scratch field;
//   k_line_solve  a warp owns 32 lines (lane = line) and runs LAPACK dgtsv
//                 in its exact elimination order, row interchanges included
//                 (tri_solve_line, wd_kernels.cuh), restated as a carried
//                 row state: before step i the carry is the current row i
//                 of the eliminated system; step i with b = rhs[i+1] gives
//                   no swap: y_i = carry,  carry' = b - f_i * carry
//                   swap:    y_i = b,      carry' = carry - f_i * b
//                 and y_{n-1} = the final carry (y overwrites the scratch
//                 in place); back substitution
//                   x_i = ((y_i - du_i x_{i+1}) - du2_i x_{i+2}) / d_i
//                 (the quotient as the correctly rounded reciprocal
//                 product), periodic lines adding the Sherman-Morrison
//                 correction x - (h.rhs / denom) z (oracle/wd.py:
//                 cyclic_apply, h.rhs accumulated in row order).
//
// The recurrences are latency chains; everything that is not on the chain
// (stencils, boundary closures, pin tests, index arithmetic) runs in the
// fully parallel first kernel, so the solve issues ~10 instructions per row
// and the factor lives in shared memory.  Results are written through the
// derivative epilogue (JOB 0) or with the pinned-node restore (JOB 1).
#pragma once

#include "wd_kernels.cuh"

namespace wd {

constexpr int LS_WARPS = 4;  // warps per CTA of k_line_solve
constexpr int LS_U = 8;      // rows per unrolled group

__device__ __forceinline__ double ls_div(double s, double d, double r) {
  const double q0 = s * r;
  const double e = fma(-q0, d, s);
  return fma(e, r, q0);
}

template <int JOB>
static __global__ void k_line_rhs(const double* __restrict__ in, double* __restrict__ rhs,
                                  AxisGeom ag, int per, double off, int scheme, FilterCoef fc,
                                  const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  const long long sa = ag.sa;
  const int n = ag.n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < ag.N;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = ag.coord(idx);
    Line w{in + (idx - (long long)i * sa), sa, n, per, off};
    double r;
    if (JOB == 0) {
      r = compact_rhs_at(w, i, n, scheme, per);
    } else {
      const int h = per ? 5 : ((i == 0 || i == n - 1) ? 0 : min(min(i, n - 1 - i), 5));
      if (h == 0) {
        r = w(i);
      } else {
        const double* c = fc.hc + h * 6;
        r = c[0] * w(i);
        for (int k = 1; k <= h; ++k) r = r + c[k] * (w(i + k) + w(i - k));
      }
    }
    rhs[idx] = r;
  }
}

template <int JOB>
static __global__ void __launch_bounds__(LS_WARPS * 32)
    k_line_solve(const double* __restrict__ in, double* y, double* out, Geom g, int axis,
                 int n, long long sa, TriDev T, Epi epi, const uint8_t* pin, int use_geom_pin,
                 const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  // factor rows: fact, swap, du, du2, d, rinv, z, h; then one flag per
  // forward group (any row interchange in the group)
  extern __shared__ double ls_f[];
  const long long L = g.N / n;
  double* sfact = ls_f;
  double* sswap = sfact + n;
  double* sdu = sswap + n;
  double* sdu2 = sdu + n;
  double* sd = sdu2 + n;
  double* srinv = sd + n;
  double* sz = srinv + n;
  double* sh = sz + n;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    sfact[t] = t < n - 1 ? T.fact[t] : 0.0;
    sswap[t] = t < n - 1 ? T.swap[t] : 0.0;
    sdu[t] = t < n - 1 ? T.du[t] : 0.0;
    sdu2[t] = t < n - 2 ? T.du2[t] : 0.0;
    sd[t] = T.d[t];
    srinv[t] = T.rinv[t];
    sz[t] = T.cyclic ? T.z[t] : 0.0;
    sh[t] = T.cyclic ? T.h[t] : 0.0;
  }
  int* gswap = reinterpret_cast<int*>(sh + n);
  for (int k = threadIdx.x; k * LS_U < n; k += blockDim.x) {
    int any = 0;
    for (int s2 = 0; s2 < LS_U; ++s2) {
      const int t = k * LS_U + s2;
      if (t < n - 1 && T.swap[t] != 0.0) any = 1;
    }
    gswap[k] = any;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long nwarps = (long long)gridDim.x * LS_WARPS;
  for (long long grp = (long long)blockIdx.x * LS_WARPS + wib; grp * 32 < L; grp += nwarps) {
    const long long q = grp * 32 + lane;
    if (q >= L) continue;  // no warp-collective operations below
    const long long base = line_base(g, axis, q);
    double* yl = y + base;
    // pinned nodes of this line (JOB 1): whole line on a wall face of
    // another axis, the ends on this axis' wall faces, the solid mask
    bool line_pin = false, pin_lo = false, pin_hi = false;
    if (JOB == 1 && use_geom_pin) {
      int c[kMaxDim];
      node_coords(g, base, c);
#pragma unroll
      for (int b = 0; b < kMaxDim; ++b) {
        if (b >= g.nd || b == axis) continue;
        if (c[b] == 0 && g.face[2 * b] == WD_FACE_WALL) line_pin = true;
        if (c[b] == g.n[b] - 1 && g.face[2 * b + 1] == WD_FACE_WALL) line_pin = true;
      }
      pin_lo = pick(g.face, 2 * axis) == WD_FACE_WALL;
      pin_hi = pick(g.face, 2 * axis + 1) == WD_FACE_WALL;
    }
    // ---------------- forward elimination (y in place of the rhs)
    // Software-pipelined: the loads of group k+1 are issued before the
    // recurrence of group k runs (warps issue in order, so a load consumed
    // right away would stall the chain for a full memory latency).
    double carry = yl[0];
    double hs = 0.0;
    if (T.cyclic) hs = hs + sh[0] * carry;
    const int nf = (n - 1) / LS_U;  // full forward groups (steps 0 .. nf*U-1)
    auto fload = [&](int k, double (&b)[LS_U]) {
#pragma unroll
      for (int s = 0; s < LS_U; ++s) b[s] = yl[(long long)(k * LS_U + s + 1) * sa];
    };
    auto fproc = [&](int k, const double (&b)[LS_U]) {
      if (!gswap[k]) {  // no interchange in this group (CTA-uniform branch)
#pragma unroll
        for (int s = 0; s < LS_U; ++s) {
          const int i = k * LS_U + s;
          const double yv = carry;
          carry = b[s] - sfact[i] * carry;
          if (T.cyclic) hs = hs + sh[i + 1] * b[s];
          yl[(long long)i * sa] = yv;
        }
        return;
      }
#pragma unroll
      for (int s = 0; s < LS_U; ++s) {
        const int i = k * LS_U + s;
        const double f = sfact[i];
        double yv;
        if (sswap[i] != 0.0) {
          yv = b[s];
          carry = carry - f * b[s];
        } else {
          yv = carry;
          carry = b[s] - f * carry;
        }
        if (T.cyclic) hs = hs + sh[i + 1] * b[s];
        yl[(long long)i * sa] = yv;
      }
    };
    {
      double bA[LS_U], bB[LS_U];
      if (nf > 0) fload(0, bA);
      for (int k = 0; k < nf; k += 2) {
        if (k + 1 < nf) fload(k + 1, bB);
        fproc(k, bA);
        if (k + 1 >= nf) break;
        if (k + 2 < nf) fload(k + 2, bA);
        fproc(k + 1, bB);
      }
    }
    for (int i = nf * LS_U; i < n - 1; ++i) {
      const double bv = yl[(long long)(i + 1) * sa];
      const double f = sfact[i];
      double yv;
      if (sswap[i] != 0.0) {
        yv = bv;
        carry = carry - f * bv;
      } else {
        yv = carry;
        carry = bv - f * carry;
      }
      if (T.cyclic) hs = hs + sh[i + 1] * bv;
      yl[(long long)i * sa] = yv;
    }
    yl[(long long)(n - 1) * sa] = carry;
    const double fcor = T.cyclic ? hs / T.denom : 0.0;
    // ---------------- back substitution + output (pipelined the same way;
    // the epilogue's per-node operands are fetched with the group's y)
    const bool need_acc = JOB == 0 && epi.mode == 2;
    const bool need_c = JOB == 0 && epi.mode != 0 && epi.cfield != nullptr;
    auto emit = [&](int r, double x, double accv, double cv) {
      const double xv = T.cyclic ? x - fcor * sz[r] : x;
      const long long idx = base + (long long)r * sa;
      if (JOB == 0) {
        double o = xv;
        if (epi.mode != 0) {
          const double t = (epi.cfield ? cv : epi.cscal) * xv;
          o = epi.mode == 1 ? t : accv + t;
        }
        out[idx] = o;
      } else {
        bool p;
        if (use_geom_pin)
          p = line_pin || (r == 0 && pin_lo) || (r == n - 1 && pin_hi) ||
              (g.mask != nullptr && g.mask[idx] != 0);
        else
          p = pin != nullptr && pin[idx] != 0;
        // branch, not a select: an unconditional load of in[idx] would
        // stall the in-order warp for a memory latency on every row
        if (p) out[idx] = in[idx];
        else out[idx] = xv;
      }
    };
    auto eload = [&](int r, double& accv, double& cv) {
      const long long idx = base + (long long)r * sa;
      accv = need_acc ? epi.acc[idx] : 0.0;
      cv = need_c ? epi.cfield[idx] : 0.0;
    };
    double x1, x2;
    {
      double a0, c0;
      eload(n - 1, a0, c0);
      x1 = ls_div(carry, sd[n - 1], srinv[n - 1]);
      emit(n - 1, x1, a0, c0);
      x2 = x1;
      eload(n - 2, a0, c0);
      x1 = ls_div(yl[(long long)(n - 2) * sa] - sdu[n - 2] * x2, sd[n - 2], srinv[n - 2]);
      emit(n - 2, x1, a0, c0);
    }
    // rows n-3 .. 0 in groups of U going down: group k covers rows
    // n-3-kU .. n-3-kU-U+1
    const int nbk = (n - 2) / LS_U;
    auto bload = [&](int k, double (&yv)[LS_U], double (&av)[LS_U], double (&cv)[LS_U]) {
#pragma unroll
      for (int s = 0; s < LS_U; ++s) {
        const int rr = n - 3 - k * LS_U - s;
        yv[s] = yl[(long long)rr * sa];
        eload(rr, av[s], cv[s]);
      }
    };
    auto bproc = [&](int k, const double (&yv)[LS_U], const double (&av)[LS_U],
                     const double (&cv)[LS_U]) {
#pragma unroll
      for (int s = 0; s < LS_U; ++s) {
        const int rr = n - 3 - k * LS_U - s;
        const double x = ls_div((yv[s] - sdu[rr] * x1) - sdu2[rr] * x2, sd[rr], srinv[rr]);
        x2 = x1;
        x1 = x;
        emit(rr, x, av[s], cv[s]);
      }
    };
    {
      double yA[LS_U], aA[LS_U], cA[LS_U], yB[LS_U], aB[LS_U], cB[LS_U];
      if (nbk > 0) bload(0, yA, aA, cA);
      for (int k = 0; k < nbk; k += 2) {
        if (k + 1 < nbk) bload(k + 1, yB, aB, cB);
        bproc(k, yA, aA, cA);
        if (k + 1 >= nbk) break;
        if (k + 2 < nbk) bload(k + 2, yA, aA, cA);
        bproc(k + 1, yB, aB, cB);
      }
    }
    for (int r = n - 3 - nbk * LS_U; r >= 0; --r) {
      double av, cv;
      eload(r, av, cv);
      const double x =
          ls_div((yl[(long long)r * sa] - sdu[r] * x1) - sdu2[r] * x2, sd[r], srinv[r]);
      x2 = x1;
      x1 = x;
      emit(r, x, av, cv);
    }
  }
}

__host__ __forceinline__ size_t line_solve_smem(int n) {
  return (size_t)8 * n * sizeof(double) + (size_t)((n + LS_U - 1) / LS_U) * sizeof(int);
}
constexpr size_t kLineSolveMaxSmem = 200 * 1024;

}  // namespace wd
