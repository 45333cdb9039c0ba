// Fast-arithmetic RK stage for interior tiles of the fused 3-D path
// (SolveConfig.arith = "fast"; same discretisation as k_f3_stage /
// formulations.py:135-197 + solver.py:160-205, round-off differences only).
//
// B200 data movement, one CTA = 32 (k) x 16 (j) column tile streaming along i:
//   * every global -> shared transfer is cp.async (16 B, L2 only) in a
//     3-slot ring, issued two planes ahead of the plane being computed, so
//     no registers are spent on prefetch and HBM latency is covered by the
//     ring depth rather than by occupancy;
//   * per plane a slot holds the p tile with a 2R-row j halo and an 8-wide
//     k halo (16-byte aligned), the pointwise fields A / dt / acc, and the
//     interior of plane i + 2R, the entry of the axis-0 register windows;
//   * axis 0 runs as the two-pass D_0 (D_0 p) in registers: a p window
//     p(i .. i+2R) and a u = sqrt(cc_0) D_0 p window u(i-R .. i+R) (7 pairs
//     each for E6), indexed modulo 2R+1 inside a loop unrolled by 2R+1, so
//     they are never shifted (no register moves per plane);
//   * each thread owns two adjacent k nodes: the k stencils of both come
//     from 7 16-byte shared loads, the j stencils from 2R + 1.
// Registers <= 128 with 256 threads -> two CTAs (16 warps) per SM.
// Interior tiles only (no non-periodic k / j boundary inside the stencil
// reach; tiles touching one run the exact kernel, wd_fused.cu) and planes
// at least 2R from a non-periodic axis-0 end (periodic axis 0, or the
// ghosted slabs of the decomposed solve); otherwise k_f3_fast2.
#pragma once

#include "wd_fused3d.cuh"

namespace wd {

constexpr int S3_TK = F3_TK;       // 32
constexpr int S3_TJ = F3_TJ;       // 16
constexpr int S3_PW = S3_TK + 16;  // 48 doubles per plane row (8-wide k halo)
#ifndef WD_S3_D
#define WD_S3_D 2
#endif
#ifndef WD_S3_REG
#define WD_S3_REG 0
#endif
#ifndef WD_S3_LS
#define WD_S3_LS 1
#endif
constexpr int S3_D = WD_S3_D;      // planes in flight ahead of the computed one
// pointwise fields (A, dt, acc, axis-0 window entry) straight to registers,
// one plane ahead, instead of through shared memory (saves shared-memory
// bandwidth; measured slower: 7.27 vs 6.42 ms per step, one plane of
// register prefetch does not cover the HBM latency -> off)
constexpr bool S3_REG = WD_S3_REG != 0;
// low-storage RK4 (fast mode): k1 and k3 are recovered from the stage
// fields, k1 = (p1 - A) * 2 / dt, k3 = (p3 - A) / dt, so acc = k1 + 2 k2 is
// written once (stage 2) and read once (stage 4): 17 state words per step
// instead of 21 (stage 1: p -> p1, dt; 2: p1, A, dt -> p2, acc;
// 3: p2, A, dt -> p3; 4: p3, A, dt, acc -> out).  Round-off level change:
// the recovered k enters the update multiplied by dt again (<= 1 ulp of A).
constexpr bool S3_LS = WD_S3_LS != 0;
constexpr int S3_SLOTS = S3_D + 1;

template <int R>
struct S3Layout {
  static constexpr int H = 2 * R;                   // composite half-width
  static constexpr int PH = S3_TJ + 2 * H;          // plane rows
  static constexpr int PLANE = PH * S3_PW;          // doubles per plane slot
  static constexpr int PT = S3_TJ * S3_TK;          // 512 doubles per pointwise tile
  static constexpr int SLOT = PLANE + (S3_REG ? 0 : 4 * PT);  // plane (+ A, dt, acc, window entry)
  static constexpr int CHUNKS = PH * (S3_PW / 2);   // 16-byte chunks of a plane slot
  static constexpr int CPT = (CHUNKS + 255) / 256;  // chunks per thread
  static constexpr size_t SMEM = (size_t)S3_SLOTS * SLOT * sizeof(double);
};

__device__ __forceinline__ void s3_cp16(double* dst, const double* src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = ok ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(sz));
}
__device__ __forceinline__ void s3_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void s3_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// fast correctly-rounded-to-a-few-ulp quotient a / b (MUFU seed + Newton)
__device__ __forceinline__ double s3_div(double a, double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  double e = fma(-b, r, 1.0);
  r = fma(r, e, r);
  e = fma(-b, r, 1.0);
  r = fma(r, e, r);
  const double q = a * r;
  return fma(fma(-b, q, a), r, q);
}

__device__ __forceinline__ double s3_rcp(double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  double e = fma(-b, r, 1.0);
  r = fma(r, e, r);
  e = fma(-b, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double2 s3_ldcs2(const double* p) {
  return __ldcs(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ double2 s3_ldcg2(const double* p) {
  return __ldcg(reinterpret_cast<const double2*>(p));
}

// JB: tiles touching a non-periodic j end (walls).  Rows 0..5 / n1-6..n1-1
// see the E4/E6 closures (wd_common.cuh:deriv_explicit_at) inside the reach
// of D_j o D_j; there the j part is the closure-aware composite: the first
// derivative G p and the two-pass Laplacian M p = D (D p) as 12-point rows
// precomputed on the host (c_jbG, c_jbM: same discretisation as the exact
// kernel's U_j = c_1 D_j p, D_j U_j), wall rows pinned; other rows and the
// k / i parts stay composite.  No exact-kernel CTA shares the SMs (C4: the
// 2 of 32 j tile rows at y = 0, 1).
__constant__ double c_jbG[12][12];  // rows 0-5: low wall, 6-11: high wall (cols from base)
__constant__ double c_jbM[12][12];

// PUSH: slab decomposition with peer memory -- the boundary planes are also
// stored into the neighbours' ghost planes (a separate instantiation, so the
// single-GPU kernels carry neither the code nor the registers)
template <int R, bool EIK, int STAGE, bool JB, bool PUSH = false>
__global__ void __launch_bounds__(256, 2) k_f3_fast3(F3Args a, const int* tiles) {
  using LY = S3Layout<R>;
  constexpr int H = LY::H;
  constexpr int NW = H + 1;  // axis-0 windows: p(i .. i+2R), u(i-R .. i+R)
  if (a.st->state != WD_STATE_RUNNING) return;
  extern __shared__ double smem[];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;  // pair, row
  const int ntile = tiles[0];
  const int tile = tiles[1 + blockIdx.x % ntile];
  const int chunk_id = blockIdx.x / ntile;
  const int k0 = (tile % a.tiles_k) * S3_TK;
  const int j0 = (tile / a.tiles_k) * S3_TJ;
  const int i0 = a.i_lo + chunk_id * a.chunk;
  const int i1 = min(i0 + a.chunk, a.i_hi);
  if (i0 >= i1) return;
  const int n0 = a.n0, n1 = a.n1, n2 = a.n2;
  const long long s0 = a.s0;
  const int col = (j0 + ty) * n2 + k0 + 2 * tx;  // in-plane offset of the pair

  // ---- per-thread copy assignments (fixed over the stream)
  int coff[LY::CPT];  // in-plane source offset, -1 = zero fill, -2 = none
  int cdst[LY::CPT];
#pragma unroll
  for (int q = 0; q < LY::CPT; ++q) {
    const int c = tid + 256 * q;
    coff[q] = -2;
    cdst[q] = 0;
    if (c < LY::CHUNKS) {
      const int row = c / (S3_PW / 2), cc = c - row * (S3_PW / 2);
      int jg = j0 - H + row, kg = k0 - 8 + 2 * cc;
      bool ok = true;
      if (a.per1) jg = wrapm(jg, n1);
      else ok = ok && jg >= 0 && jg < n1;
      if (a.per2) kg = wrapm(kg, n2);
      else ok = ok && kg >= 0 && kg + 1 < n2;
      coff[q] = ok ? jg * n2 + kg : -1;
      cdst[q] = row * S3_PW + 2 * cc;
    }
  }
  const int own = ty * S3_TK + 2 * tx;  // pointwise slot offset of the pair
  // 32-bit element offsets (the plan guarantees N < 2^31)
  const int is0 = (int)s0;
  const int wrap0 = n0 * is0;
  // loads of plane ip into slot `slot`; the axis-0 window entry is plane
  // ip + H + 1 (periodic axis 0)
  constexpr bool NEED_ACC = S3_LS ? STAGE == 4 : STAGE > 1;  // acc read by this stage
  auto issue = [&](int ip, int slot) {
    double* sl = smem + slot * LY::SLOT;
    if (ip < i1) {
      const int po = ip * is0;
#pragma unroll
      for (int q = 0; q < LY::CPT; ++q)
        if (coff[q] != -2) s3_cp16(sl + cdst[q], a.p + (coff[q] >= 0 ? po + coff[q] : 0), coff[q] >= 0);
      const int pl = po + col;
      if (!S3_REG) {
        double* pt = sl + LY::PLANE + own;
        if (STAGE > 1) {  // stage 1: A = p, read from the plane tile
          s3_cp16(pt, a.A + pl, true);
          s3_cp16(pt + LY::PT, a.dt + pl, true);
          if (NEED_ACC) s3_cp16(pt + 2 * LY::PT, a.acc + pl, true);
        }
        int pw_off = pl + H * is0;  // window entry p(ip + 2R)
        bool wok = true;
        if (pw_off >= wrap0) {
          if (a.per0) pw_off -= wrap0;
          else wok = false;  // beyond the last plane: never used, zero fill
        }
        s3_cp16(pt + 3 * LY::PT, a.p + (wok ? pw_off : 0), wok);
      }
    }
    s3_commit();
  };
  // S3_REG: pointwise values of plane ip -> registers (A, dt: stages 2-4;
  // acc: stage 4 (low storage) or 2-4; window entry p(ip + 2R): all stages)
  double2 nA = make_double2(0.0, 0.0), ndt = nA, nacc = nA, nw = nA;
  auto pref = [&](int ip) {
    if (S3_REG && ip < i1) {
      const int pl = ip * is0 + col;
      if (STAGE > 1) {
        nA = s3_ldcs2(a.A + pl);
        ndt = s3_ldcs2(a.dt + pl);
      }
      if (NEED_ACC) nacc = s3_ldcs2(a.acc + pl);
      int pw_off = pl + H * is0;
      bool wok = true;
      if (pw_off >= wrap0) {
        if (a.per0) pw_off -= wrap0;
        else wok = false;
      }
      nw = wok ? s3_ldcg2(a.p + pw_off) : make_double2(0.0, 0.0);
    }
  };

  // ---- prologue: axis 0 runs as two passes in registers (same
  // discretisation as the composite D o D): u = sqrt(cc_0) D_0 p on a
  // window u(i-R .. i+R), p on p(i .. i+2R); both indexed modulo NW = 2R+1
  // inside a loop unrolled by NW, so neither is ever shifted.
  double2 pw[NW], uw[NW];
  {
    double2 pp[2 * H];  // p(i0-H .. i0+H-1)
#pragma unroll
    for (int s = 0; s < 2 * H; ++s) {
      int pos = i0 - H + s;
      bool ok = true;
      if (a.per0) pos = wrapm(pos, n0);
      else ok = pos >= 0 && pos < n0;
      pp[s] = ok ? *reinterpret_cast<const double2*>(a.p + (long long)pos * s0 + col)
                 : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int s = 0; s < H; ++s) pw[s] = pp[H + s];  // p(i0 + s) at slot s
#pragma unroll
    for (int s = 0; s < H; ++s) {  // u(i0 - R + s) at slot s, from p(i0-H+s .. i0+s)
      const int c = R + s;            // pp index of the centre i0 - R + s
      double2 v;
      v.x = a.fC[0][1] * (pp[c + 1].x - pp[c - 1].x);
      v.y = a.fC[0][1] * (pp[c + 1].y - pp[c - 1].y);
#pragma unroll
      for (int m = 2; m <= R; ++m) {
        v.x = fma(a.fC[0][m], pp[c + m].x - pp[c - m].x, v.x);
        v.y = fma(a.fC[0][m], pp[c + m].y - pp[c - m].y, v.y);
      }
      uw[s] = v;
    }
  }
#pragma unroll
  for (int d = 0; d < S3_D; ++d) issue(i0 + d, d);
  pref(i0);

  // slot of plane ib + u = (sb + u) mod SLOTS; NW = 7 = 1 (mod SLOTS)
  static_assert(NW % S3_SLOTS == 1, "slot rotation assumes NW = 1 mod SLOTS");
  int sb = 0;
  for (int ib = i0; ib < i1; ib += NW) {
#pragma unroll
    for (int u = 0; u < NW; ++u) {
      const int i = ib + u;
      if (i < i1) {
        int scur = sb + u % S3_SLOTS;
        scur = scur >= S3_SLOTS ? scur - S3_SLOTS : scur;
        int snext = scur + S3_D;
        snext = snext >= S3_SLOTS ? snext - S3_SLOTS : snext;
        s3_wait<S3_D - 1>();
        __syncthreads();
        issue(i + S3_D, snext);
        const double* sl = smem + scur * LY::SLOT;
        const double* pt = sl + LY::PLANE;
        double2 cA = nA, cdt = ndt, cacc = nacc;
        // window entry p(i + 2R) replaces p(i - 1); u(i + R) replaces u(i - R - 1)
        if (S3_REG) {
          pw[(u + H) % NW] = nw;
          pref(i + 1);
        } else {
          pw[(u + H) % NW] = *reinterpret_cast<const double2*>(pt + 3 * LY::PT + own);
        }
        {
          auto P = [&](int m) -> const double2& { return pw[(u + m + 2 * NW) % NW]; };  // p(i+m)
          double2 v;
          v.x = a.fC[0][1] * (P(R + 1).x - P(R - 1).x);
          v.y = a.fC[0][1] * (P(R + 1).y - P(R - 1).y);
#pragma unroll
          for (int m = 2; m <= R; ++m) {
            v.x = fma(a.fC[0][m], P(R + m).x - P(R - m).x, v.x);
            v.y = fma(a.fC[0][m], P(R + m).y - P(R - m).y, v.y);
          }
          uw[(u + H) % NW] = v;  // u(i + R): slot (u + R + R) mod NW
        }
        // k row of the pair: values k-H .. k+1+H  (cols 8-H+2tx .. 9+H+2tx)
        const double* rowp = sl + (ty + H) * S3_PW + 2 * tx + 8 - H;
        double rk[2 * H + 2];
#pragma unroll
        for (int q = 0; q < H + 1; ++q) {
          const double2 v = *reinterpret_cast<const double2*>(rowp + 2 * q);
          rk[2 * q] = v.x;
          rk[2 * q + 1] = v.y;
        }
        // j column of the pair, accumulated over symmetric row pairs
        const double* colp = sl + (ty + H) * S3_PW + 8 + 2 * tx;
        double Dj0 = 0.0, Dj1 = 0.0, Lj0 = 0.0, Lj1 = 0.0;
        bool jwall = false, pin = false;
        if (JB) {
          const int j = j0 + ty;
          const int t = j < 6 ? j : (j >= n1 - 6 ? 6 + j - (n1 - 6) : -1);
          if (t >= 0) {  // closure rows: 12-point rows from the table
            jwall = true;
            pin = (j == 0 && a.wall[2]) || (j == n1 - 1 && a.wall[3]);
            const int base = t < 6 ? 0 : n1 - 12;  // global row of column 0
            const double* cb = sl + (base - (j0 - H)) * S3_PW + 8 + 2 * tx;
            double g0 = 0.0, g1 = 0.0, m0 = 0.0, m1 = 0.0;
#pragma unroll
            for (int q = 0; q < 12; ++q) {
              const double2 v = *reinterpret_cast<const double2*>(cb + q * S3_PW);
              const double G = c_jbG[t][q], M = c_jbM[t][q];
              g0 = fma(G, v.x, g0);
              g1 = fma(G, v.y, g1);
              m0 = fma(M, v.x, m0);
              m1 = fma(M, v.y, m1);
            }
            Dj0 = a.fsq[1] * g0;
            Dj1 = a.fsq[1] * g1;
            Lj0 = a.cc1 * m0;
            Lj1 = a.cc1 * m1;
          }
        }
        if (!jwall) {
          const double2 c = *reinterpret_cast<const double2*>(colp);
          Lj0 = a.fE[1][0] * c.x;
          Lj1 = a.fE[1][0] * c.y;
#pragma unroll
          for (int m = 1; m <= H; ++m) {
            const double2 lo = *reinterpret_cast<const double2*>(colp - m * S3_PW);
            const double2 hi = *reinterpret_cast<const double2*>(colp + m * S3_PW);
            Lj0 = fma(a.fE[1][m], hi.x + lo.x, Lj0);
            Lj1 = fma(a.fE[1][m], hi.y + lo.y, Lj1);
            if (m <= R) {
              Dj0 = fma(a.fC[1][m], hi.x - lo.x, Dj0);
              Dj1 = fma(a.fC[1][m], hi.y - lo.y, Dj1);
            }
          }
        }
        const double2 Av = STAGE == 1 ? *reinterpret_cast<const double2*>(colp)
                                      : (S3_REG ? cA : *reinterpret_cast<const double2*>(pt + own));
        double2 dtv2 = make_double2(0.0, 0.0), accv2 = make_double2(0.0, 0.0);
        if (STAGE > 1) {
          dtv2 = S3_REG ? cdt : *reinterpret_cast<const double2*>(pt + LY::PT + own);
          if (NEED_ACC) accv2 = S3_REG ? cacc : *reinterpret_cast<const double2*>(pt + 2 * LY::PT + own);
        }
        double o[2], ac[2], dtn[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double* ck = rk + H + e;  // centre of node e
          // axis 0 from the modular register windows:
          // p(i+m) = pw[(u+m) % NW], u(i+m) = uw[(u+m+R) % NW]
          auto u0 = [&](int m) -> double {
            const double2 v = uw[(u + m + R + 2 * NW) % NW];
            return e == 0 ? v.x : v.y;
          };
          double Dk = a.fC[2][1] * (ck[1] - ck[-1]);
#pragma unroll
          for (int m = 2; m <= R; ++m) Dk = fma(a.fC[2][m], ck[m] - ck[-m], Dk);
          const double Di = u0(0);
          const double pv = e == 0 ? pw[u % NW].x : pw[u % NW].y;
          const double Dj = e == 0 ? Dj0 : Dj1;
          double adv = Di * Di;
          adv = fma(Dj, Dj, adv);
          adv = fma(Dk, Dk, adv);
          double kv;
          if (EIK) {
            kv = 1.0 - adv;
          } else {
            // p_0 terms of k (composite); j's is in Lj; i is two-pass
            double lap = fma(a.fE[2][0], pv, e == 0 ? Lj0 : Lj1);
#pragma unroll
            for (int m = 1; m <= H; ++m) lap = fma(a.fE[2][m], ck[m] + ck[-m], lap);
#pragma unroll
            for (int m = 1; m <= R; ++m) lap = fma(a.fC[0][m], u0(m) - u0(-m), lap);
            kv = fma(a.eps * pv, lap, 1.0) - adv;
          }
          const double Ae = e == 0 ? Av.x : Av.y;
          if (STAGE == 1) {
            double den = a.fsq[0] * fabs(Di);
            den = fma(a.fsq[1], fabs(Dj), den);
            den = fma(a.fsq[2], fabs(Dk), den);
            if (!EIK) den = fma(2.0 * (a.eps * pv), a.sumS, den);
            const double dtv = fmin(s3_div(a.cfl, den + 1e-30), a.cflms);
            dtn[e] = dtv;
            ac[e] = kv;
            o[e] = pin ? 0.0 : fma(0.5 * dtv, kv, Ae);
          } else if (S3_LS && STAGE == 2) {  // k1 = (p1 - A) * 2 / dt
            const double dte = e == 0 ? dtv2.x : dtv2.y;
            const double k1 = (pv - Ae) * (2.0 * s3_rcp(dte));
            ac[e] = fma(2.0, kv, k1);
            o[e] = pin ? 0.0 : fma(0.5 * dte, kv, Ae);
          } else if (S3_LS && STAGE == 3) {
            const double dte = e == 0 ? dtv2.x : dtv2.y;
            o[e] = pin ? 0.0 : fma(dte, kv, Ae);
          } else if (STAGE == 2 || STAGE == 3) {
            const double dte = e == 0 ? dtv2.x : dtv2.y;
            const double acce = e == 0 ? accv2.x : accv2.y;
            ac[e] = fma(2.0, kv, acce);
            o[e] = pin ? 0.0 : fma(STAGE == 3 ? dte : 0.5 * dte, kv, Ae);
          } else if (S3_LS) {  // k3 = (p3 - A) / dt
            const double dte = e == 0 ? dtv2.x : dtv2.y;
            const double acce = e == 0 ? accv2.x : accv2.y;
            const double k3 = (pv - Ae) * s3_rcp(dte);
            o[e] = pin ? 0.0 : fma(dte * (1.0 / 6.0), fma(2.0, k3, acce) + kv, Ae);
          } else {
            const double dte = e == 0 ? dtv2.x : dtv2.y;
            const double acce = e == 0 ? accv2.x : accv2.y;
            o[e] = pin ? 0.0 : fma(dte * (1.0 / 6.0), acce + kv, Ae);
          }
        }
        const int idx = i * is0 + col;
        if (STAGE == 1) __stcs(reinterpret_cast<double2*>(a.dt + idx), make_double2(dtn[0], dtn[1]));
        if (S3_LS ? STAGE == 2 : STAGE <= 3)
          __stcs(reinterpret_cast<double2*>(a.acc + idx), make_double2(ac[0], ac[1]));
        __stcs(reinterpret_cast<double2*>(a.out + idx), make_double2(o[0], o[1]));
        // slab decomposition: boundary planes also land in the neighbours'
        // ghost planes (peer memory, NVLink stores; plane-uniform branch)
        if (PUSH) {
          if (i < a.push_l_end)
            __stcs(reinterpret_cast<double2*>(a.peer_l + (idx + a.push_shift)),
                   make_double2(o[0], o[1]));
          if (i >= a.push_r_beg)
            __stcs(reinterpret_cast<double2*>(a.peer_r + (idx - a.push_shift)),
                   make_double2(o[0], o[1]));
        }
      }
    }
    sb = sb + 1 == S3_SLOTS ? 0 : sb + 1;
  }
  s3_wait<0>();
}

}  // namespace wd
