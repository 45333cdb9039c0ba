// Fused 3-D RK4 stage kernel for uniform Cartesian grids with explicit
// central schemes (E2/E4/E6): one launch per RK stage computes the
// directional derivatives, U, U_hat, the Laplacian div(grad phi) as
// first derivatives of U (formulations.py:135-150), the HJ / Eikonal
// residual (formulations.py:153-197), the local time step (stage 1,
// solver.py:160-180) and the RK combine (solver.py:198-205) -- in the
// reference's exact operation order, so the result is bit-identical to the
// generic kernels.
//
// Data movement (B200): a CTA owns a TK x TJ column tile of the (j, k)
// plane and streams along i (axis 0).  Axis-0 stencils run out of register
// windows (p at i-R..i+4+R, U_0 at i-4..i+4, d_0 at i..i+4), so every p
// value is read from HBM once per stage; the in-plane stencils read a
// double-buffered shared-memory plane with a 7-point halo (the halo comes
// from L2).  Pointwise fields (phi0, dt, acc) are read/written once.
// Per update per stage: S1 4 words, S2/S3 6, S4 5.
#pragma once

#include "wd_kernels.cuh"

namespace wd {

constexpr int F3_TK = 32;
constexpr int F3_TJ = 16;
constexpr int F3_HP = 7;   // p halo (U halo 4 + stencil radius <= 3)
constexpr int F3_HU = 4;   // U halo (E4 closures reach 4 rows)
constexpr int F3_PW = F3_TK + 2 * F3_HP;  // 46
constexpr int F3_PH = F3_TJ + 2 * F3_HP;  // 30
constexpr int F3_UKW = F3_TK + 2 * F3_HU; // 40
constexpr int F3_UJH = F3_TJ + 2 * F3_HU; // 24
constexpr int F3_SMEM_DOUBLES = 2 * (F3_PH * F3_PW + F3_TJ * F3_UKW + F3_UJH * F3_TK);

struct F3Args {
  int n0, n1, n2;
  long long s0;          // n1 * n2
  int per0, per1, per2;
  int wall[6];
  double c0, c1, c2;     // d xi_l / d x_l
  double eps, cfl, sumS, cflms;
  const double* p;       // stage input field
  const double* A;       // field at step start
  double* dt;
  double* acc;
  double* out;
  int chunk;             // planes per CTA
  int i_lo, i_hi;        // planes to update (ghosted slabs: interior only)
  int tiles_k, tiles_j;
  const Status* st;
  // slab decomposition with peer memory (wd_dist.cuh): the planes
  // [i_lo, push_l_end) of `out` also go to the left neighbour's high ghost
  // planes (index + push_shift) and the planes [push_r_beg, i_hi) to the right
  // neighbour's low ghost planes (index - push_shift), as stores over NVLink
  double* peer_l = nullptr;
  double* peer_r = nullptr;
  long long push_shift = 0;
  int push_l_end = 0, push_r_beg = 0;
  // fast mode: central coefficients c[r] (r = 1..3) and the composite
  // (D o D) 13-point coefficients e[m] (m = 0..6), squared metrics
  double cr[4];
  double e[7];
  double cc0, cc1, cc2;
  // fast3 folded coefficients: D_l = sum_m fC[l][m] (p_m - p_-m) = sqrt(cc_l) d_l,
  // lap = fE0 p_0 + sum_l sum_m fE[l][m] (p_m + p_-m), adv = sum_l D_l^2
  double fC[3][4];
  double fE[3][7];
  double fE0;
  double fsq[3];
};

template <int R>
struct SchemeOf;
template <>
struct SchemeOf<1> { static constexpr int id = WD_E2; };
template <>
struct SchemeOf<2> { static constexpr int id = WD_E4; };
template <>
struct SchemeOf<3> { static constexpr int id = WD_E6; };

// central relation on values at offsets -R..R
template <int R>
__device__ __forceinline__ double central(double m3, double m2, double m1, double p1, double p2,
                                          double p3) {
  if (R == 1) return E2_CA * (p1 - m1);
  if (R == 2) return E4_CA * (p1 - m1) + E4_CB * (p2 - m2);
  return E6_CA * (p1 - m1) + E6_CB * (p2 - m2) + E6_CC * (p3 - m3);
}

// closures written on explicit values (same expression text as
// e4_closure / the E2 closures in wd_common.cuh)
__device__ __forceinline__ double e4_row0(double w0, double w1, double w2, double w3, double w4) {
  return (-25.0 * w0 + 48.0 * w1 - 36.0 * w2 + 16.0 * w3 - 3.0 * w4) / 12.0;
}
__device__ __forceinline__ double e4_row1(double w0, double w1, double w2, double w3, double w4) {
  return (-3.0 * w0 - 10.0 * w1 + 18.0 * w2 - 6.0 * w3 + w4) / 12.0;
}
// last row: wl = w(n-1), wl1 = w(n-2), ...
__device__ __forceinline__ double e4_rowl(double wl, double wl1, double wl2, double wl3,
                                          double wl4) {
  return (25.0 * wl - 48.0 * wl1 + 36.0 * wl2 - 16.0 * wl3 + 3.0 * wl4) / 12.0;
}
__device__ __forceinline__ double e4_rowl1(double wl, double wl1, double wl2, double wl3,
                                           double wl4) {
  return (3.0 * wl + 10.0 * wl1 - 18.0 * wl2 + 6.0 * wl3 - wl4) / 12.0;
}
__device__ __forceinline__ double e4_central(double m2, double m1, double p1, double p2) {
  return E4_CA * (p1 - m1) + E4_CB * (p2 - m2);
}

// Derivative along axis 0 at row i from the U window u[0..8] (positions
// i-4..i+4) -- every row type with compile-time slots.
template <int R>
__device__ __forceinline__ double d0_from_window(const double* u, int i, int n, int per) {
  if (per) return central<R>(u[1], u[2], u[3], u[5], u[6], u[7]);
  if (R == 1) {
    if (i == 0) return -1.5 * u[4] + 2.0 * u[5] - 0.5 * u[6];
    if (i == n - 1) return 1.5 * u[4] - 2.0 * u[3] + 0.5 * u[2];
    return central<1>(0, 0, u[3], u[5], 0, 0);
  }
  if (i == 0) return e4_row0(u[4], u[5], u[6], u[7], u[8]);
  if (i == 1) return e4_row1(u[3], u[4], u[5], u[6], u[7]);
  if (i == n - 1) return e4_rowl(u[4], u[3], u[2], u[1], u[0]);
  if (i == n - 2) return e4_rowl1(u[5], u[4], u[3], u[2], u[1]);
  if (R == 3 && (i == 2 || i == n - 3)) return e4_central(u[2], u[3], u[5], u[6]);
  return central<R>(u[1], u[2], u[3], u[5], u[6], u[7]);
}

// d_0 at the entering row q = i+5 from the p window w[0..4+2R]
// (positions i+1-R .. i+5+R, q at slot 4+R).  Only far-end closures occur.
template <int R>
__device__ __forceinline__ double d0_entering(const double* w, int q, int n, int per) {
  constexpr int Q = 4 + R;
  if (!per) {
    if (R == 1) {
      if (q == n - 1) return 1.5 * w[Q] - 2.0 * w[Q - 1] + 0.5 * w[Q - 2];
    } else {
      if (q == n - 1) return e4_rowl(w[Q], w[Q - 1], w[Q - 2], w[Q - 3], w[Q - 4]);
      if (q == n - 2) return e4_rowl1(w[Q + 1], w[Q], w[Q - 1], w[Q - 2], w[Q - 3]);
      if (R == 3 && q == n - 3) return e4_central(w[Q - 2], w[Q - 1], w[Q + 1], w[Q + 2]);
    }
  }
  return central<R>(R >= 3 ? w[Q - 3] : 0.0, R >= 2 ? w[Q - 2] : 0.0, w[Q - 1], w[Q + 1],
                    R >= 2 ? w[Q + 2] : 0.0, R >= 3 ? w[Q + 3] : 0.0);
}

struct SLine {  // shared-memory line addressed by global index
  const double* p;
  int base;
  int st;
  __device__ __forceinline__ double operator()(int j) const { return p[(j - base) * st]; }
};

__device__ __forceinline__ int wrapm(int x, int n) {
  x %= n;
  return x < 0 ? x + n : x;
}

// Values one thread loads for plane i (software-pipelined one plane ahead).
struct F3Plane {
  double own;    // own P slot when the thread is outside the domain (periodic wrap)
  double jh;     // j-halo row value (ty < 2*HP)
  double kh;     // k-halo column value (tx < 2*HP)
  double A, dt, acc;
  double pnext;  // axis-0 window entry p(i + 5 + R)
};

// Per-thread in-plane offsets, fixed for the whole i-stream (-1 = unused).
struct F3Offs {
  int own, jh, kh, node;
};

__device__ __forceinline__ F3Offs f3_offsets(const F3Args& a, int j0, int k0, int tx, int ty,
                                             bool act) {
  const int n1 = a.n1, n2 = a.n2;
  const int k = k0 + tx, j = j0 + ty;
  F3Offs o;
  o.node = act ? j * n2 + k : -1;
  o.own = -1;
  if (!act && (k < n2 || a.per2) && (j < n1 || a.per1)) {
    const int jw = j < n1 ? j : wrapm(j, n1), kw = k < n2 ? k : wrapm(k, n2);
    o.own = jw * n2 + kw;
  }
  o.jh = -1;
  if (ty < 2 * F3_HP && k < n2) {
    const int jg = j0 - F3_HP + (ty < F3_HP ? ty : ty + F3_TJ);
    if (a.per1) o.jh = wrapm(jg, n1) * n2 + k;
    else if (jg >= 0 && jg < n1) o.jh = jg * n2 + k;
  }
  o.kh = -1;
  if (tx < 2 * F3_HP && j < n1) {
    const int kg = k0 - F3_HP + (tx < F3_HP ? tx : tx + F3_TK);
    if (a.per2) o.kh = j * n2 + wrapm(kg, n2);
    else if (kg >= 0 && kg < n2) o.kh = j * n2 + kg;
  }
  return o;
}

template <int STAGE>
__device__ __forceinline__ void f3_load_plane(const F3Args& a, const double* __restrict__ pp,
                                              long long plane, const double* __restrict__ pn,
                                              const F3Offs& o, F3Plane& v) {
  v.own = o.own >= 0 ? pp[o.own] : 0.0;
  v.jh = o.jh >= 0 ? pp[o.jh] : 0.0;
  v.kh = o.kh >= 0 ? pp[o.kh] : 0.0;
  v.A = v.dt = v.acc = v.pnext = 0.0;
  if (o.node >= 0) {
    v.A = __ldcs(a.A + plane + o.node);
    if (STAGE > 1) v.dt = __ldcs(a.dt + plane + o.node);
    if (STAGE > 1) v.acc = __ldcs(a.acc + plane + o.node);
    if (pn) v.pnext = pn[o.node];
  }
}

template <int R, bool EIK, int STAGE>
__global__ void __launch_bounds__(F3_TK* F3_TJ, 1) k_f3_stage(F3Args a, const int* tiles) {
  if (a.st->state != WD_STATE_RUNNING) return;
  constexpr int SCH = SchemeOf<R>::id;
  constexpr int NPW = 5 + 2 * R;
  extern __shared__ double smem[];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int ntile = tiles ? tiles[0] : a.tiles_k * a.tiles_j;
  const int tile = tiles ? tiles[1 + blockIdx.x % ntile] : blockIdx.x % ntile;
  const int chunk_id = blockIdx.x / ntile;
  const int k0 = (tile % a.tiles_k) * F3_TK;
  const int j0 = (tile / a.tiles_k) * F3_TJ;
  const int i0 = a.i_lo + chunk_id * a.chunk;
  const int i1 = min(i0 + a.chunk, a.i_hi);
  if (i0 >= i1) return;
  const int k = k0 + tx, j = j0 + ty;
  const bool act = k < a.n2 && j < a.n1;
  const int n0 = a.n0, n1 = a.n1, n2 = a.n2;
  const long long s0 = a.s0;
  const long long col = (long long)j * n2 + k;  // offset of (0, j, k)

  // ---- prologue: register windows along axis 0
  double pw[NPW], uw[9], dw[5];
#pragma unroll
  for (int s = 0; s < NPW; ++s) {
    int pos = i0 - R + s;
    double v = 0.0;
    if (act) {
      if (a.per0) v = a.p[(long long)wrapm(pos, n0) * s0 + col];
      else if (pos >= 0 && pos < n0) v = a.p[(long long)pos * s0 + col];
    }
    pw[s] = v;
  }
  {
    Line gl{a.p + col, s0, n0, a.per0, 0.0};
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      const int q = i0 - 4 + s;
      double d = 0.0;
      if (act && (a.per0 || (q >= 0 && q < n0))) {
        const int qq = a.per0 ? wrapm(q, n0) : q;
        d = deriv_explicit_at(gl, qq, n0, SCH, a.per0);
      }
      uw[s] = a.c0 * d;
      if (s >= 4) dw[s - 4] = d;
    }
  }
  const F3Offs offs = f3_offsets(a, j0, k0, tx, ty, act);
  // plane index of the axis-0 window entry i + 5 + R (wrapped incrementally)
  int inext = a.per0 ? wrapm(i0 + 5 + R, n0) : i0 + 5 + R;
  auto next_ptr = [&](int ip) -> const double* {
    return (a.per0 || ip < n0) ? a.p + (long long)ip * s0 : nullptr;
  };
  F3Plane cur;
  f3_load_plane<STAGE>(a, a.p + (long long)i0 * s0, (long long)i0 * s0, next_ptr(inext), offs,
                       cur);
  // CTA-uniform: does the tile (with halo) stay clear of non-periodic ends?
  const bool kfast = a.per2 ? (k0 + F3_TK <= n2) : (k0 >= F3_HP && k0 + F3_TK + F3_HP <= n2);
  const bool jfast = a.per1 ? (j0 + F3_TJ <= n1) : (j0 >= F3_HP && j0 + F3_TJ + F3_HP <= n1);

  for (int i = i0; i < i1; ++i) {
    const int b = (i - i0) & 1;
    double* Pb = smem + b * (F3_PH * F3_PW);
    double* Ukb = smem + 2 * F3_PH * F3_PW + b * (F3_TJ * F3_UKW);
    double* Ujb = smem + 2 * F3_PH * F3_PW + 2 * F3_TJ * F3_UKW + b * (F3_UJH * F3_TK);
    const long long plane = (long long)i * s0;
    // ---- plane i into shared memory (own value from the window)
    Pb[(ty + F3_HP) * F3_PW + tx + F3_HP] = act ? pw[R] : cur.own;
    if (ty < 2 * F3_HP) Pb[(ty < F3_HP ? ty : ty + F3_TJ) * F3_PW + tx + F3_HP] = cur.jh;
    if (tx < 2 * F3_HP) Pb[(ty + F3_HP) * F3_PW + (tx < F3_HP ? tx : tx + F3_TK)] = cur.kh;
    const double Av = cur.A, dtin = cur.dt, accv = cur.acc, pnext = cur.pnext;
    // ---- prefetch plane i + 1 (latency hidden behind this plane's math)
    inext = inext + 1;
    if (a.per0 && inext == n0) inext = 0;
    if (i + 1 < i1)
      f3_load_plane<STAGE>(a, a.p + plane + s0, plane + s0, next_ptr(inext), offs, cur);
    __syncthreads();
    // ---- U_k on [TJ] x [TK + 2HU], U_j on [TJ + 2HU] x [TK]
    double d2 = 0.0, d1 = 0.0;
    if (kfast) {  // interior / periodic tile: central stencil, compile-time offsets
      const double* row = Pb + (ty + F3_HP) * F3_PW + 3;  // row[t] <-> kg = k0 - 4 + t
      Ukb[ty * F3_UKW + tx] = a.c2 * central<R>(row[tx - 3], row[tx - 2], row[tx - 1],
                                                row[tx + 1], row[tx + 2], row[tx + 3]);
      {  // the 16 x 8 extra halo positions on 4 full warps (no 8-of-32 lanes)
        const int L = ty * F3_TK + tx;
        if (L < F3_TJ * 2 * F3_HU) {
          const int rr = L / (2 * F3_HU), t = F3_TK + L % (2 * F3_HU);
          const double* row2 = Pb + (rr + F3_HP) * F3_PW + 3;
          Ukb[rr * F3_UKW + t] = a.c2 * central<R>(row2[t - 3], row2[t - 2], row2[t - 1],
                                                   row2[t + 1], row2[t + 2], row2[t + 3]);
        }
      }
      const int c = tx + 4;
      d2 = central<R>(row[c - 3], row[c - 2], row[c - 1], row[c + 1], row[c + 2], row[c + 3]);
    } else {
      for (int t = tx; t < F3_UKW; t += F3_TK) {
        const int kg = k0 - F3_HU + t;
        double v = 0.0;
        if (j < n1 && (a.per2 || (kg >= 0 && kg < n2))) {
          SLine ln{Pb + (ty + F3_HP) * F3_PW, k0 - F3_HP, 1};
          v = a.c2 * deriv_explicit_at(ln, kg, n2, SCH, a.per2);
        }
        Ukb[ty * F3_UKW + t] = v;
      }
      if (act) {
        SLine lk{Pb + (ty + F3_HP) * F3_PW, k0 - F3_HP, 1};
        d2 = deriv_explicit_at(lk, k, n2, SCH, a.per2);
      }
    }
    if (jfast) {
      const double* colp = Pb + tx + F3_HP + 3 * F3_PW;  // colp[t*PW] <-> jg = j0 - 4 + t
      Ujb[ty * F3_TK + tx] =
          a.c1 * central<R>(colp[(ty - 3) * F3_PW], colp[(ty - 2) * F3_PW],
                            colp[(ty - 1) * F3_PW], colp[(ty + 1) * F3_PW],
                            colp[(ty + 2) * F3_PW], colp[(ty + 3) * F3_PW]);
      if (ty < 2 * F3_HU) {
        const int t = ty + F3_TJ;
        Ujb[t * F3_TK + tx] =
            a.c1 * central<R>(colp[(t - 3) * F3_PW], colp[(t - 2) * F3_PW],
                              colp[(t - 1) * F3_PW], colp[(t + 1) * F3_PW],
                              colp[(t + 2) * F3_PW], colp[(t + 3) * F3_PW]);
      }
      const int c = ty + 4;
      d1 = central<R>(colp[(c - 3) * F3_PW], colp[(c - 2) * F3_PW], colp[(c - 1) * F3_PW],
                      colp[(c + 1) * F3_PW], colp[(c + 2) * F3_PW], colp[(c + 3) * F3_PW]);
    } else {
      for (int t = ty; t < F3_UJH; t += F3_TJ) {
        const int jg = j0 - F3_HU + t;
        double v = 0.0;
        if (k < n2 && (a.per1 || (jg >= 0 && jg < n1))) {
          SLine ln{Pb + tx + F3_HP, j0 - F3_HP, F3_PW};
          v = a.c1 * deriv_explicit_at(ln, jg, n1, SCH, a.per1);
        }
        Ujb[t * F3_TK + tx] = v;
      }
      if (act) {
        SLine lj{Pb + tx + F3_HP, j0 - F3_HP, F3_PW};
        d1 = deriv_explicit_at(lj, j, n1, SCH, a.per1);
      }
    }
    __syncthreads();
    if (act) {
      double D2, D1;
      if (kfast) {
        const double* u = Ukb + ty * F3_UKW + tx + F3_HU;
        D2 = central<R>(u[-3], u[-2], u[-1], u[1], u[2], u[3]);
      } else {
        SLine uk{Ukb + ty * F3_UKW, k0 - F3_HU, 1};
        D2 = deriv_explicit_at(uk, k, n2, SCH, a.per2);
      }
      if (jfast) {
        const double* u = Ujb + (ty + F3_HU) * F3_TK + tx;
        D1 = central<R>(u[-3 * F3_TK], u[-2 * F3_TK], u[-F3_TK], u[F3_TK], u[2 * F3_TK],
                        u[3 * F3_TK]);
      } else {
        SLine uj{Ujb + tx, j0 - F3_HU, F3_TK};
        D1 = deriv_explicit_at(uj, j, n1, SCH, a.per1);
      }
      const double D0 = (a.per0 || (i >= 4 && i <= n0 - 5))
                            ? central<R>(uw[1], uw[2], uw[3], uw[5], uw[6], uw[7])
                            : d0_from_window<R>(uw, i, n0, a.per0);
      const double d0 = dw[0];
      const double pv = pw[R];
      // U_m = c_m d_m ; U_hat_l = c_l U_l (diagonal metrics)
      const double U0 = a.c0 * d0, U1 = a.c1 * d1, U2 = a.c2 * d2;
      const double H0 = a.c0 * U0, H1 = a.c1 * U1, H2 = a.c2 * U2;
      const double adv = H0 * d0 + H1 * d1 + H2 * d2;
      double kv;
      if (EIK) {
        kv = 1.0 - adv;
      } else {
        const double lap = a.c0 * D0 + a.c1 * D1 + a.c2 * D2;
        kv = 1.0 + (a.eps * pv) * lap - adv;
      }
      const bool pinned = (i == 0 && a.wall[0]) || (i == n0 - 1 && a.wall[1]) ||
                          (j == 0 && a.wall[2]) || (j == n1 - 1 && a.wall[3]) ||
                          (k == 0 && a.wall[4]) || (k == n2 - 1 && a.wall[5]);
      const long long idx = plane + col;
      if (STAGE == 1) {
        double den = fabs(H0) + fabs(H1) + fabs(H2);
        if (!EIK) den = den + 2.0 * (a.eps * pv) * a.sumS;
        const double d = a.cfl / (den + 1e-30);
        const double dtv = np_min(d, a.cflms);
        __stcs(a.dt + idx, dtv);
        __stcs(a.acc + idx, kv);
        a.out[idx] = pinned ? 0.0 : Av + (0.5 * dtv) * kv;
      } else if (STAGE == 2 || STAGE == 3) {
        __stcs(a.acc + idx, accv + 2.0 * kv);
        const double cdt = STAGE == 3 ? dtin : 0.5 * dtin;
        a.out[idx] = pinned ? 0.0 : Av + cdt * kv;
      } else {
        a.out[idx] = pinned ? 0.0 : Av + (dtin / 6.0) * (accv + kv);
      }
    }
    // ---- advance the axis-0 windows
#pragma unroll
    for (int s = 0; s < NPW - 1; ++s) pw[s] = pw[s + 1];
    pw[NPW - 1] = pnext;
    const int q = i + 5;
    double dq = 0.0;
    if (act && (a.per0 || q < n0)) {
      constexpr int Q = 4 + R;
      dq = (a.per0 || q <= n0 - 5)
               ? central<R>(R >= 3 ? pw[Q - 3] : 0.0, R >= 2 ? pw[Q - 2] : 0.0, pw[Q - 1],
                            pw[Q + 1], R >= 2 ? pw[Q + 2] : 0.0, R >= 3 ? pw[Q + 3] : 0.0)
               : d0_entering<R>(pw, q, n0, a.per0);
    }
#pragma unroll
    for (int s = 0; s < 8; ++s) uw[s] = uw[s + 1];
    uw[8] = a.c0 * dq;
#pragma unroll
    for (int s = 0; s < 4; ++s) dw[s] = dw[s + 1];
    dw[4] = dq;
  }
}


// ======================================================================
// FAST arithmetic variant (opt-in, SolveConfig.arith = "fast"): same
// discretisation, but the Laplacian term c_l D_l(c_l D_l p) is evaluated
// as c_l^2 (D o D)_l p with the composite 13-point stencil and FMA
// contraction, so no U_l staging or halo recomputation is needed.  Equal to
// the exact path in real arithmetic; differs by round-off (tests bound the
// drift and the converged field against the oracle).  Tiles that touch a
// non-periodic boundary fall back to the exact kernel (wd_fused.cu).
template <int R>
__device__ __forceinline__ double f_d(const F3Args& a, double m3, double m2, double m1, double p1,
                                      double p2, double p3) {
  double d = a.cr[1] * (p1 - m1);
  if (R >= 2) d = fma(a.cr[2], p2 - m2, d);
  if (R >= 3) d = fma(a.cr[3], p3 - m3, d);
  return d;
}
template <int R>
__device__ __forceinline__ double f_dd(const F3Args& a, const double* w /* w[-2R..2R] centred */) {
  double s = a.e[0] * w[0];
#pragma unroll
  for (int m = 1; m <= 2 * R; ++m) s = fma(a.e[m], w[m] + w[-m], s);
  return s;
}

template <int R, bool EIK, int STAGE>
__global__ void __launch_bounds__(F3_TK* F3_TJ, 1) k_f3_fast(F3Args a, const int* tiles) {
  if (a.st->state != WD_STATE_RUNNING) return;
  constexpr int H = 2 * R;          // composite half-width
  constexpr int NW = 2 * H + 1;     // axis-0 window p(i-H .. i+H)
  extern __shared__ double smem[];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int ntile = tiles[0];
  const int tile = tiles[1 + blockIdx.x % ntile];
  const int chunk_id = blockIdx.x / ntile;
  const int k0 = (tile % a.tiles_k) * F3_TK;
  const int j0 = (tile / a.tiles_k) * F3_TJ;
  const int i0 = a.i_lo + chunk_id * a.chunk;
  const int i1 = min(i0 + a.chunk, a.i_hi);
  if (i0 >= i1) return;
  const int k = k0 + tx, j = j0 + ty;  // interior tiles: always inside
  const int n0 = a.n0;
  const long long s0 = a.s0;
  const long long col = (long long)j * a.n2 + k;
  const F3Offs offs = f3_offsets(a, j0, k0, tx, ty, true);
  double pw[NW];
#pragma unroll
  for (int s = 0; s < NW; ++s) {
    const int pos = i0 - H + s;
    double v = 0.0;
    if (a.per0) v = a.p[(long long)wrapm(pos, n0) * s0 + col];
    else if (pos >= 0 && pos < n0) v = a.p[(long long)pos * s0 + col];
    pw[s] = v;
  }
  int inext = a.per0 ? wrapm(i0 + H + 1, n0) : i0 + H + 1;
  const double* pp0 = a.p + (long long)i0 * s0;
  double nA = __ldcs(a.A + (long long)i0 * s0 + col);
  double ndt = STAGE > 1 ? __ldcs(a.dt + (long long)i0 * s0 + col) : 0.0;
  double nacc = STAGE > 1 ? __ldcs(a.acc + (long long)i0 * s0 + col) : 0.0;
  double njh = offs.jh >= 0 ? pp0[offs.jh] : 0.0;
  double nkh = offs.kh >= 0 ? pp0[offs.kh] : 0.0;
  double npn = (a.per0 || inext < n0) ? a.p[(long long)inext * s0 + col] : 0.0;
  for (int i = i0; i < i1; ++i) {
    double* Pb = smem + ((i - i0) & 1) * (F3_PH * F3_PW);
    const long long plane = (long long)i * s0;
    Pb[(ty + F3_HP) * F3_PW + tx + F3_HP] = pw[H];
    if (ty < 2 * F3_HP) Pb[(ty < F3_HP ? ty : ty + F3_TJ) * F3_PW + tx + F3_HP] = njh;
    if (tx < 2 * F3_HP) Pb[(ty + F3_HP) * F3_PW + (tx < F3_HP ? tx : tx + F3_TK)] = nkh;
    const double Av = nA, dtin = ndt, accv = nacc, pnext = npn;
    inext = inext + 1;
    if (a.per0 && inext == n0) inext = 0;
    if (i + 1 < i1) {
      const double* pp = a.p + plane + s0;
      nA = __ldcs(a.A + plane + s0 + col);
      if (STAGE > 1) ndt = __ldcs(a.dt + plane + s0 + col);
      if (STAGE > 1) nacc = __ldcs(a.acc + plane + s0 + col);
      njh = offs.jh >= 0 ? pp[offs.jh] : 0.0;
      nkh = offs.kh >= 0 ? pp[offs.kh] : 0.0;
      npn = (a.per0 || inext < n0) ? a.p[(long long)inext * s0 + col] : 0.0;
    }
    __syncthreads();
    const double* row = Pb + (ty + F3_HP) * F3_PW + tx + F3_HP;  // row[0] = own
    const double* cl = row;                                       // column: cl[r*PW]
    double wk[2 * H + 1], wj[2 * H + 1];
#pragma unroll
    for (int m = -H; m <= H; ++m) {
      wk[m + H] = row[m];
      wj[m + H] = cl[m * F3_PW];
    }
    const double d2 = f_d<R>(a, wk[H - 3 < 0 ? 0 : H - 3], wk[H - 2 < 0 ? 0 : H - 2], wk[H - 1],
                             wk[H + 1], wk[H + 2 > 2 * H ? 2 * H : H + 2],
                             wk[H + 3 > 2 * H ? 2 * H : H + 3]);
    const double d1 = f_d<R>(a, wj[H - 3 < 0 ? 0 : H - 3], wj[H - 2 < 0 ? 0 : H - 2], wj[H - 1],
                             wj[H + 1], wj[H + 2 > 2 * H ? 2 * H : H + 2],
                             wj[H + 3 > 2 * H ? 2 * H : H + 3]);
    const double dd2 = f_dd<R>(a, wk + H);
    const double dd1 = f_dd<R>(a, wj + H);
    double d0, dd0;
    if (a.per0 || (i >= H && i <= n0 - 1 - H)) {
      d0 = f_d<R>(a, pw[H - 3 < 0 ? 0 : H - 3], pw[H - 2 < 0 ? 0 : H - 2], pw[H - 1], pw[H + 1],
                  pw[H + 2 > 2 * H ? 2 * H : H + 2], pw[H + 3 > 2 * H ? 2 * H : H + 3]);
      dd0 = f_dd<R>(a, pw + H);
    } else {  // non-periodic axis-0 boundary planes: closures via U_0 (exact order)
      constexpr int SCH = SchemeOf<R>::id;
      Line gl{a.p + col, s0, n0, 0, 0.0};
      d0 = deriv_explicit_at(gl, i, n0, SCH, 0);
      double u[9];
#pragma unroll
      for (int s = 0; s < 9; ++s) {
        const int q = i - 4 + s;
        u[s] = (q >= 0 && q < n0) ? a.c0 * deriv_explicit_at(gl, q, n0, SCH, 0) : 0.0;
      }
      // D_0(U_0) at i then divide out c0: keep the c0 * D0(U0) product form
      const double D0 = d0_from_window<R>(u, i, n0, 0);
      dd0 = D0 / a.c0;  // lap term below multiplies by c0^2 -> c0 * D0
    }
    const double pv = pw[H];
    const double h0 = a.cc0 * d0, h1 = a.cc1 * d1, h2 = a.cc2 * d2;
    double adv = h0 * d0;
    adv = fma(h1, d1, adv);
    adv = fma(h2, d2, adv);
    double kv;
    if (EIK) {
      kv = 1.0 - adv;
    } else {
      double lap = a.cc0 * dd0;
      lap = fma(a.cc1, dd1, lap);
      lap = fma(a.cc2, dd2, lap);
      kv = fma(a.eps * pv, lap, 1.0) - adv;
    }
    const bool pinned = (i == 0 && a.wall[0]) || (i == n0 - 1 && a.wall[1]);
    const long long idx = plane + col;
    if (STAGE == 1) {
      double den = fabs(h0) + fabs(h1) + fabs(h2);
      if (!EIK) den = fma(2.0 * (a.eps * pv), a.sumS, den);
      const double dtv = fmin(a.cfl / (den + 1e-30), a.cflms);
      __stcs(a.dt + idx, dtv);
      __stcs(a.acc + idx, kv);
      a.out[idx] = pinned ? 0.0 : fma(0.5 * dtv, kv, Av);
    } else if (STAGE == 2 || STAGE == 3) {
      __stcs(a.acc + idx, fma(2.0, kv, accv));
      const double cdt = STAGE == 3 ? dtin : 0.5 * dtin;
      a.out[idx] = pinned ? 0.0 : fma(cdt, kv, Av);
    } else {
      a.out[idx] = pinned ? 0.0 : fma(dtin / 6.0, accv + kv, Av);
    }
#pragma unroll
    for (int s = 0; s < NW - 1; ++s) pw[s] = pw[s + 1];
    pw[NW - 1] = pnext;
  }
}

// ----------------------------------------------------------------------
// FAST variant, paired: 256 threads = 16 k-pairs x 16 j-rows; each thread
// owns the adjacent nodes (k, k+1) of its row, so the k stencils of both
// nodes come from 7 aligned 16-byte shared loads, the j stencils from 13,
// and every global access is a 16-byte vector.  Tile 32 (k) x 16 (j), plane
// tile with an 8-wide k halo (16-byte alignment) and a 7-row j halo.
constexpr int F2_PW = F3_TK + 16;        // 48 doubles per plane row
constexpr int F2_PH = F3_TJ + 2 * F3_HP; // 30 rows

__device__ __forceinline__ double2 ld2(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}
__device__ __forceinline__ double2 ldcs2(const double* p) {
  return __ldcs(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ void stcs2(double* p, double x, double y) {
  __stcs(reinterpret_cast<double2*>(p), make_double2(x, y));
}

constexpr int F2_PF = 3;  // L2 prefetch distance (planes)
__device__ __forceinline__ void l2_prefetch(const double* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];\n" ::"l"(p));
}

template <int R, bool EIK, int STAGE>
__global__ void __launch_bounds__(256, 1) k_f3_fast2(F3Args a, const int* tiles) {
  if (a.st->state != WD_STATE_RUNNING) return;
  constexpr int H = 2 * R;       // composite half-width (<= 6)
  constexpr int NW = 2 * H + 1;  // axis-0 window
  extern __shared__ double smem[];
  const int tx = threadIdx.x, ty = threadIdx.y;  // tx: 0..15 (pairs), ty: 0..15
  const int ntile = tiles[0];
  const int tile = tiles[1 + blockIdx.x % ntile];
  const int chunk_id = blockIdx.x / ntile;
  const int k0 = (tile % a.tiles_k) * F3_TK;
  const int j0 = (tile / a.tiles_k) * F3_TJ;
  const int i0 = a.i_lo + chunk_id * a.chunk;
  const int i1 = min(i0 + a.chunk, a.i_hi);
  if (i0 >= i1) return;
  const int n0 = a.n0, n1 = a.n1, n2 = a.n2;
  const long long s0 = a.s0;
  const int k = k0 + 2 * tx, j = j0 + ty;
  const int col = j * n2 + k;  // in-plane offset of the pair
  // halo offsets (in-plane), fixed over the stream
  int jh = -1, kh = -1;
  if (ty < 2 * F3_HP) {  // j-halo rows: row jj, pair tx
    const int jg = j0 - F3_HP + (ty < F3_HP ? ty : ty + F3_TJ);
    jh = (a.per1 ? wrapm(jg, n1) : jg) * n2 + k;
  }
  if (tx < 8) {  // k-halo: 4 pairs left (k0-8..k0-1), 4 pairs right (k0+32..)
    const int kg = tx < 4 ? k0 - 8 + 2 * tx : k0 + F3_TK + 2 * (tx - 4);
    kh = j * n2 + (a.per2 ? wrapm(kg, n2) : kg);
  }
  double2 pw[NW];
#pragma unroll
  for (int s = 0; s < NW; ++s) {
    const int pos = a.per0 ? wrapm(i0 - H + s, n0) : i0 - H + s;
    pw[s] = (pos >= 0 && pos < n0) ? ld2(a.p + (long long)pos * s0 + col) : make_double2(0.0, 0.0);
  }
  int inext = a.per0 ? wrapm(i0 + H + 1, n0) : i0 + H + 1;
  const long long pl0 = (long long)i0 * s0;
  double2 nA = ldcs2(a.A + pl0 + col);
  double2 ndt = STAGE > 1 ? ldcs2(a.dt + pl0 + col) : make_double2(0.0, 0.0);
  double2 nacc = STAGE > 1 ? ldcs2(a.acc + pl0 + col) : make_double2(0.0, 0.0);
  double2 njh = jh >= 0 ? ld2(a.p + pl0 + jh) : make_double2(0.0, 0.0);
  double2 nkh = kh >= 0 ? ld2(a.p + pl0 + kh) : make_double2(0.0, 0.0);
  double2 npn = (a.per0 || inext < n0) ? ld2(a.p + (long long)inext * s0 + col)
                                        : make_double2(0.0, 0.0);
  for (int i = i0; i < i1; ++i) {
    double* Pb = smem + ((i - i0) & 1) * (F2_PH * F2_PW);
    const long long plane = (long long)i * s0;
    // own pair at row ty+7, col 8+2tx; halos
    *reinterpret_cast<double2*>(Pb + (ty + F3_HP) * F2_PW + 8 + 2 * tx) = pw[H];
    if (jh >= 0 || ty < 2 * F3_HP)
      *reinterpret_cast<double2*>(Pb + (ty < F3_HP ? ty : ty + F3_TJ) * F2_PW + 8 + 2 * tx) = njh;
    if (tx < 8)
      *reinterpret_cast<double2*>(Pb + (ty + F3_HP) * F2_PW +
                                  (tx < 4 ? 2 * tx : F3_TK + 8 + 2 * (tx - 4))) = nkh;
    const double2 Av = nA, dtin = ndt, accv = nacc, pnext = npn;
    inext = inext + 1;
    if (a.per0 && inext == n0) inext = 0;
    if (i + 1 < i1) {
      const long long pl = plane + s0;
      nA = ldcs2(a.A + pl + col);
      if (STAGE > 1) ndt = ldcs2(a.dt + pl + col);
      if (STAGE > 1) nacc = ldcs2(a.acc + pl + col);
      if (jh >= 0) njh = ld2(a.p + pl + jh);
      if (kh >= 0) nkh = ld2(a.p + pl + kh);
      npn = (a.per0 || inext < n0) ? ld2(a.p + (long long)inext * s0 + col)
                                   : make_double2(0.0, 0.0);
    }
    // L2 prefetch F2_PF planes ahead: the register prefetch above is only
    // one plane deep, so without it the loads it issues see full HBM latency
    if (i + F2_PF < i1) {
      const long long pl = plane + F2_PF * s0;
      l2_prefetch(a.A + pl + col);
      if (STAGE > 1) l2_prefetch(a.dt + pl + col);
      if (STAGE > 1) l2_prefetch(a.acc + pl + col);
      int ip = inext + F2_PF - 1;
      if (a.per0) ip = ip >= n0 ? ip - n0 : ip;
      if (ip < n0) l2_prefetch(a.p + (long long)ip * s0 + col);
    }
    __syncthreads();
    // k row: values k-6 .. k+7 (cols 2tx+2 .. 2tx+15)
    const double* rowp = Pb + (ty + F3_HP) * F2_PW + 2 * tx + 2;
    double rk[14];
#pragma unroll
    for (int q = 0; q < 7; ++q) {
      const double2 v = ld2(rowp + 2 * q);
      rk[2 * q] = v.x;
      rk[2 * q + 1] = v.y;
    }
    // j stencils of both nodes, accumulated over symmetric row pairs
    const double* colp = Pb + (ty + F3_HP) * F2_PW + 8 + 2 * tx;  // row j
    double dj[2], ddj[2];
    {
      const double2 c = ld2(colp);
      ddj[0] = a.e[0] * c.x;
      ddj[1] = a.e[0] * c.y;
      dj[0] = dj[1] = 0.0;
#pragma unroll
      for (int m = 1; m <= H; ++m) {
        const double2 lo = ld2(colp - m * F2_PW);
        const double2 hi = ld2(colp + m * F2_PW);
        ddj[0] = fma(a.e[m], hi.x + lo.x, ddj[0]);
        ddj[1] = fma(a.e[m], hi.y + lo.y, ddj[1]);
        if (m <= R) {
          if (m == 1) {
            dj[0] = a.cr[1] * (hi.x - lo.x);
            dj[1] = a.cr[1] * (hi.y - lo.y);
          } else {
            dj[0] = fma(a.cr[m], hi.x - lo.x, dj[0]);
            dj[1] = fma(a.cr[m], hi.y - lo.y, dj[1]);
          }
        }
      }
    }
    double out2[2], acc2[2], dt2[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const double* wk = rk + 6 + e - H + H;  // centre of node e: rk[6 + e]
      const double* ck = wk;
      const double* pwc;  // axis-0 window of node e (struct of pairs)
      double w0[NW];
#pragma unroll
      for (int s = 0; s < NW; ++s) w0[s] = e == 0 ? pw[s].x : pw[s].y;
      pwc = w0 + H;
      (void)pwc;
      const double d2 = f_d<R>(a, ck[-3 < -H ? -H : -3], ck[-2], ck[-1], ck[1], ck[2],
                               ck[3 > H ? H : 3]);
      const double d1 = dj[e];
      const double dd2 = f_dd<R>(a, ck);
      const double dd1 = ddj[e];
      double d0, dd0;
      if (a.per0 || (i >= H && i <= n0 - 1 - H)) {
        d0 = f_d<R>(a, w0[H - 3 < 0 ? 0 : H - 3], w0[H - 2 < 0 ? 0 : H - 2], w0[H - 1],
                    w0[H + 1], w0[H + 2 > 2 * H ? 2 * H : H + 2],
                    w0[H + 3 > 2 * H ? 2 * H : H + 3]);
        dd0 = f_dd<R>(a, w0 + H);
      } else {
        constexpr int SCH = SchemeOf<R>::id;
        Line gl{a.p + col + e, s0, n0, 0, 0.0};
        d0 = deriv_explicit_at(gl, i, n0, SCH, 0);
        double u[9];
#pragma unroll
        for (int s = 0; s < 9; ++s) {
          const int q = i - 4 + s;
          u[s] = (q >= 0 && q < n0) ? a.c0 * deriv_explicit_at(gl, q, n0, SCH, 0) : 0.0;
        }
        dd0 = d0_from_window<R>(u, i, n0, 0) / a.c0;
      }
      const double pv = w0[H];
      const double h0 = a.cc0 * d0, h1 = a.cc1 * d1, h2 = a.cc2 * d2;
      double adv = h0 * d0;
      adv = fma(h1, d1, adv);
      adv = fma(h2, d2, adv);
      double kv;
      if (EIK) {
        kv = 1.0 - adv;
      } else {
        double lap = a.cc0 * dd0;
        lap = fma(a.cc1, dd1, lap);
        lap = fma(a.cc2, dd2, lap);
        kv = fma(a.eps * pv, lap, 1.0) - adv;
      }
      const bool pinned = (i == 0 && a.wall[0]) || (i == n0 - 1 && a.wall[1]);
      const double Ae = e == 0 ? Av.x : Av.y;
      const double dte = e == 0 ? dtin.x : dtin.y;
      const double acce = e == 0 ? accv.x : accv.y;
      if (STAGE == 1) {
        double den = fabs(h0) + fabs(h1) + fabs(h2);
        if (!EIK) den = fma(2.0 * (a.eps * pv), a.sumS, den);
        const double dtv = fmin(a.cfl / (den + 1e-30), a.cflms);
        dt2[e] = dtv;
        acc2[e] = kv;
        out2[e] = pinned ? 0.0 : fma(0.5 * dtv, kv, Ae);
      } else if (STAGE == 2 || STAGE == 3) {
        acc2[e] = fma(2.0, kv, acce);
        const double cdt = STAGE == 3 ? dte : 0.5 * dte;
        out2[e] = pinned ? 0.0 : fma(cdt, kv, Ae);
      } else {
        out2[e] = pinned ? 0.0 : fma(dte / 6.0, acce + kv, Ae);
      }
    }
    const long long idx = plane + col;
    if (STAGE == 1) {
      stcs2(a.dt + idx, dt2[0], dt2[1]);
      stcs2(a.acc + idx, acc2[0], acc2[1]);
    } else if (STAGE == 2 || STAGE == 3) {
      stcs2(a.acc + idx, acc2[0], acc2[1]);
    }
    *reinterpret_cast<double2*>(a.out + idx) = make_double2(out2[0], out2[1]);
#pragma unroll
    for (int s = 0; s < NW - 1; ++s) pw[s] = pw[s + 1];
    pw[NW - 1] = pnext;
  }
}

}  // namespace wd
