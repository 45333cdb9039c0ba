// Fast E6 stage, interior tiles, two j rows per thread (k_f3_fast4).
//
// Same discretisation, operation order per node and data movement as
// k_f3_fast3 (wd_stage_fast.cuh: cp.async ring, register windows along
// axis 0, composite k / j stencils, low-storage RK4), but each of the 128
// threads owns a 2 (j) x 2 (k) block of the 32 x 16 column tile.  The j
// column of the two rows is one 14-row window (14 LDS.128) instead of 2 x 13,
// which takes ~20 % off the shared-memory traffic per node -- the resource
// that bounds k_f3_fast3 (ncu: short_scoreboard / mio_throttle, ~245 B of
// shared traffic per node).  Two 128-thread CTAs per SM (the register file
// holds the two rows' axis-0 windows).
#pragma once

#include "wd_stage_fast.cuh"

namespace wd {

#ifndef WD_S4_MINB
#define WD_S4_MINB 2
#endif
template <int R, bool EIK, int STAGE, bool PUSH = false>
__global__ void __launch_bounds__(128, WD_S4_MINB) k_f3_fast4(F3Args a, const int* tiles) {
  static_assert(S3_LS && !S3_REG, "k_f3_fast4 implements the low-storage, shared-memory variant");
  using LY = S3Layout<R>;
  constexpr int H = LY::H;
  constexpr int NW = H + 1;
  constexpr int NT = 128;
  constexpr int CPT = (LY::CHUNKS + NT - 1) / NT;
  if (a.st->state != WD_STATE_RUNNING) return;
  extern __shared__ double smem[];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;  // pair, row pair (rows 2ty, 2ty + 1)
  const int ntile = tiles[0];
  const int tile = tiles[1 + blockIdx.x % ntile];
  const int chunk_id = blockIdx.x / ntile;
  const int k0 = (tile % a.tiles_k) * S3_TK;
  const int j0 = (tile / a.tiles_k) * S3_TJ;
  const int i0 = a.i_lo + chunk_id * a.chunk;
  const int i1 = min(i0 + a.chunk, a.i_hi);
  if (i0 >= i1) return;
  const int n0 = a.n0, n1 = a.n1, n2 = a.n2;
  const int col0 = (j0 + 2 * ty) * n2 + k0 + 2 * tx;  // row 2ty; row 2ty+1 at + n2

  int coff[CPT];
  int cdst[CPT];
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int c = tid + NT * q;
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
  const int own0 = 2 * ty * S3_TK + 2 * tx;  // pointwise slot offset, row 2ty
  const int is0 = (int)a.s0;
  const int wrap0 = n0 * is0;
  constexpr bool NEED_ACC = STAGE == 4;
  auto issue = [&](int ip, int slot) {
    double* sl = smem + slot * LY::SLOT;
    if (ip < i1) {
      const int po = ip * is0;
#pragma unroll
      for (int q = 0; q < CPT; ++q)
        if (coff[q] != -2) s3_cp16(sl + cdst[q], a.p + (coff[q] >= 0 ? po + coff[q] : 0), coff[q] >= 0);
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int pl = po + col0 + r * n2;
        double* pt = sl + LY::PLANE + own0 + r * S3_TK;
        if (STAGE > 1) {
          s3_cp16(pt, a.A + pl, true);
          s3_cp16(pt + LY::PT, a.dt + pl, true);
          if (NEED_ACC) s3_cp16(pt + 2 * LY::PT, a.acc + pl, true);
        }
        int pw_off = pl + H * is0;
        bool wok = true;
        if (pw_off >= wrap0) {
          if (a.per0) pw_off -= wrap0;
          else wok = false;
        }
        s3_cp16(pt + 3 * LY::PT, a.p + (wok ? pw_off : 0), wok);
      }
    }
    s3_commit();
  };

  // axis-0 windows per row: p(i .. i+2R), u = sqrt(cc_0) D_0 p on u(i-R .. i+R)
  double2 pw[2][NW], uw[2][NW];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    double2 pp[2 * H];
#pragma unroll
    for (int s = 0; s < 2 * H; ++s) {
      int pos = i0 - H + s;
      bool ok = true;
      if (a.per0) pos = wrapm(pos, n0);
      else ok = pos >= 0 && pos < n0;
      pp[s] = ok ? *reinterpret_cast<const double2*>(a.p + (long long)pos * a.s0 + col0 + r * n2)
                 : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int s = 0; s < H; ++s) pw[r][s] = pp[H + s];
#pragma unroll
    for (int s = 0; s < H; ++s) {
      const int c = R + s;
      double2 v;
      v.x = a.fC[0][1] * (pp[c + 1].x - pp[c - 1].x);
      v.y = a.fC[0][1] * (pp[c + 1].y - pp[c - 1].y);
#pragma unroll
      for (int m = 2; m <= R; ++m) {
        v.x = fma(a.fC[0][m], pp[c + m].x - pp[c - m].x, v.x);
        v.y = fma(a.fC[0][m], pp[c + m].y - pp[c - m].y, v.y);
      }
      uw[r][s] = v;
    }
  }
#pragma unroll
  for (int d = 0; d < S3_D; ++d) issue(i0 + d, d);

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
        // j column of both rows: slot rows 2ty .. 2ty + 2H + 1 (14 for E6)
        double2 cj[2 * H + 2];
        {
          const double* cp = sl + 2 * ty * S3_PW + 8 + 2 * tx;
#pragma unroll
          for (int q = 0; q < 2 * H + 2; ++q) cj[q] = *reinterpret_cast<const double2*>(cp + q * S3_PW);
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          pw[r][(u + H) % NW] = *reinterpret_cast<const double2*>(pt + 3 * LY::PT + own0 + r * S3_TK);
          {
            auto P = [&](int m) -> const double2& { return pw[r][(u + m + 2 * NW) % NW]; };
            double2 v;
            v.x = a.fC[0][1] * (P(R + 1).x - P(R - 1).x);
            v.y = a.fC[0][1] * (P(R + 1).y - P(R - 1).y);
#pragma unroll
            for (int m = 2; m <= R; ++m) {
              v.x = fma(a.fC[0][m], P(R + m).x - P(R - m).x, v.x);
              v.y = fma(a.fC[0][m], P(R + m).y - P(R - m).y, v.y);
            }
            uw[r][(u + H) % NW] = v;
          }
          // k row: values k-H .. k+1+H of row 2ty + r
          const double* rowp = sl + (2 * ty + r + H) * S3_PW + 2 * tx + 8 - H;
          double rk[2 * H + 2];
#pragma unroll
          for (int q = 0; q < H + 1; ++q) {
            const double2 v = *reinterpret_cast<const double2*>(rowp + 2 * q);
            rk[2 * q] = v.x;
            rk[2 * q + 1] = v.y;
          }
          // j stencils of row r: centre cj[H + r], symmetric pairs
          const double2 cc = cj[H + r];
          double Lj0 = a.fE[1][0] * cc.x, Lj1 = a.fE[1][0] * cc.y;
          double Dj0 = 0.0, Dj1 = 0.0;
#pragma unroll
          for (int m = 1; m <= H; ++m) {
            const double2 lo = cj[H + r - m], hi = cj[H + r + m];
            Lj0 = fma(a.fE[1][m], hi.x + lo.x, Lj0);
            Lj1 = fma(a.fE[1][m], hi.y + lo.y, Lj1);
            if (m <= R) {
              Dj0 = fma(a.fC[1][m], hi.x - lo.x, Dj0);
              Dj1 = fma(a.fC[1][m], hi.y - lo.y, Dj1);
            }
          }
          const int own = own0 + r * S3_TK;
          const double2 Av = STAGE == 1 ? cc : *reinterpret_cast<const double2*>(pt + own);
          double2 dtv2 = make_double2(0.0, 0.0), accv2 = make_double2(0.0, 0.0);
          if (STAGE > 1) dtv2 = *reinterpret_cast<const double2*>(pt + LY::PT + own);
          if (NEED_ACC) accv2 = *reinterpret_cast<const double2*>(pt + 2 * LY::PT + own);
          double o[2], ac[2], dtn[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double* ck = rk + H + e;
            auto u0 = [&](int m) -> double {
              const double2 v = uw[r][(u + m + R + 2 * NW) % NW];
              return e == 0 ? v.x : v.y;
            };
            double Dk = a.fC[2][1] * (ck[1] - ck[-1]);
#pragma unroll
            for (int m = 2; m <= R; ++m) Dk = fma(a.fC[2][m], ck[m] - ck[-m], Dk);
            const double Di = u0(0);
            const double pv = e == 0 ? pw[r][u % NW].x : pw[r][u % NW].y;
            const double Dj = e == 0 ? Dj0 : Dj1;
            double adv = Di * Di;
            adv = fma(Dj, Dj, adv);
            adv = fma(Dk, Dk, adv);
            double kv;
            if (EIK) {
              kv = 1.0 - adv;
            } else {
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
              o[e] = fma(0.5 * dtv, kv, Ae);
            } else if (STAGE == 2) {
              const double dte = e == 0 ? dtv2.x : dtv2.y;
              const double k1 = (pv - Ae) * (2.0 * s3_rcp(dte));
              ac[e] = fma(2.0, kv, k1);
              o[e] = fma(0.5 * dte, kv, Ae);
            } else if (STAGE == 3) {
              const double dte = e == 0 ? dtv2.x : dtv2.y;
              o[e] = fma(dte, kv, Ae);
            } else {
              const double dte = e == 0 ? dtv2.x : dtv2.y;
              const double acce = e == 0 ? accv2.x : accv2.y;
              const double k3 = (pv - Ae) * s3_rcp(dte);
              o[e] = fma(dte * (1.0 / 6.0), fma(2.0, k3, acce) + kv, Ae);
            }
          }
          const int idx = i * is0 + col0 + r * n2;
          if (STAGE == 1) __stcs(reinterpret_cast<double2*>(a.dt + idx), make_double2(dtn[0], dtn[1]));
          if (STAGE == 2) __stcs(reinterpret_cast<double2*>(a.acc + idx), make_double2(ac[0], ac[1]));
          __stcs(reinterpret_cast<double2*>(a.out + idx), make_double2(o[0], o[1]));
          if (PUSH) {  // ghost push to the neighbours (wd_stage_fast.cuh)
            if (i < a.push_l_end)
              __stcs(reinterpret_cast<double2*>(a.peer_l + (idx + a.push_shift)),
                     make_double2(o[0], o[1]));
            if (i >= a.push_r_beg)
              __stcs(reinterpret_cast<double2*>(a.peer_r + (idx - a.push_shift)),
                     make_double2(o[0], o[1]));
          }
        }
      }
    }
    sb = sb + 1 == S3_SLOTS ? 0 : sb + 1;
  }
  s3_wait<0>();
}

}  // namespace wd
