// Fast-arithmetic E6 stage kernels (wd_stage_fast.cuh) in their own
// translation unit: launch helpers used by wd_fused.cu.
#include <cmath>
#include <vector>

#include "wd_stage_fast.cuh"
#include "wd_stage_fast4.cuh"

#include <cstdlib>

// interior tiles of stage s run k_f3_fast4 (two j rows per thread) when bit
// s-1 of WD_S4 is set.  A/B (same box, 512^3): stages 3 / 4 faster with
// fast4 (0.94 -> 0.84 / 1.04 -> 1.02 ms), stages 1 / 2 slower (1.00 -> 1.05,
// 1.01 -> 1.06 ms: dt quotient / k1 reciprocal at 8 warps per SM).
#ifndef WD_S4
#define WD_S4 12
#endif

namespace wd {

// fast interior tiles, E6: cp.async-pipelined stage (wd_stage_fast.cuh) with
// its own i-chunking (grid a multiple of the resident CTA slots)
// Closure rows of the E6 j derivative (wd_common.cuh:deriv_explicit_at,
// unit spacing) as a matrix D on a line of n = 24; G = D rows, M = D D.
// Rows 0-5 (low wall, columns from row 0) and n-6..n-1 (high wall, columns
// from row n-12) -> c_jbG / c_jbM.
static bool jb_tables() {
  const int n = 24;
  std::vector<double> D(n * n, 0.0);
  for (int i = 0; i < n; ++i) {
    double* r = &D[i * n];
    if (i < 2 || i > n - 3) {
      // e4_closure rows (wd_common.cuh) expressed on unit vectors
      if (i == 0) { r[0] = -25.0 / 12; r[1] = 48.0 / 12; r[2] = -36.0 / 12; r[3] = 16.0 / 12; r[4] = -3.0 / 12; }
      if (i == 1) { r[0] = -3.0 / 12; r[1] = -10.0 / 12; r[2] = 18.0 / 12; r[3] = -6.0 / 12; r[4] = 1.0 / 12; }
      if (i == n - 1) { r[n - 1] = 25.0 / 12; r[n - 2] = -48.0 / 12; r[n - 3] = 36.0 / 12; r[n - 4] = -16.0 / 12; r[n - 5] = 3.0 / 12; }
      if (i == n - 2) { r[n - 1] = 3.0 / 12; r[n - 2] = 10.0 / 12; r[n - 3] = -18.0 / 12; r[n - 4] = 6.0 / 12; r[n - 5] = -1.0 / 12; }
    } else if (i == 2 || i == n - 3) {
      r[i + 1] += E4_CA; r[i - 1] -= E4_CA; r[i + 2] += E4_CB; r[i - 2] -= E4_CB;
    } else {
      r[i + 1] += E6_CA; r[i - 1] -= E6_CA; r[i + 2] += E6_CB; r[i - 2] -= E6_CB;
      r[i + 3] += E6_CC; r[i - 3] -= E6_CC;
    }
  }
  double G[12][12] = {}, M[12][12] = {};
  for (int t = 0; t < 12; ++t) {
    const int i = t < 6 ? t : n - 12 + t;  // t >= 6: row n-6+(t-6)
    const int base = t < 6 ? 0 : n - 12;
    for (int q = 0; q < 12; ++q) {
      G[t][q] = D[i * n + base + q];
      double m = 0.0;
      for (int k = 0; k < n; ++k) m += D[i * n + k] * D[k * n + base + q];
      M[t][q] = m;
    }
  }
  return cudaMemcpyToSymbol(c_jbG, G, sizeof(G)) == cudaSuccess &&
         cudaMemcpyToSymbol(c_jbM, M, sizeof(M)) == cudaSuccess;
}

template <bool EIK>
bool fast3_prepare() {
  static const bool tables = jb_tables();
  if (!tables) return false;
  const int sm = (int)S3Layout<3>::SMEM;
  auto set = [&](const void* f) {
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) == cudaSuccess;
  };
  if (WD_S4 != 0 && !(set((const void*)k_f3_fast4<3, EIK, 1>) && set((const void*)k_f3_fast4<3, EIK, 2>) &&
                 set((const void*)k_f3_fast4<3, EIK, 3>) && set((const void*)k_f3_fast4<3, EIK, 4>)))
    return false;
  return set((const void*)k_f3_fast3<3, EIK, 1, false>) && set((const void*)k_f3_fast3<3, EIK, 2, false>) &&
         set((const void*)k_f3_fast3<3, EIK, 3, false>) && set((const void*)k_f3_fast3<3, EIK, 4, false>) &&
         set((const void*)k_f3_fast3<3, EIK, 1, true>) && set((const void*)k_f3_fast3<3, EIK, 2, true>) &&
         set((const void*)k_f3_fast3<3, EIK, 3, true>) && set((const void*)k_f3_fast3<3, EIK, 4, true>);
}

template <bool EIK, bool PUSH>
void launch_fast3_impl(int stage, F3Args a, int ntiles, const int* tiles, int chunks,
                       cudaStream_t s, bool jb) {
  const int ni = a.i_hi - a.i_lo;
  a.chunk = (ni + chunks - 1) / chunks;
  const int blocks = chunks * ntiles;
  const size_t sm = S3Layout<3>::SMEM;
  if (jb) {
    switch (stage) {
      case 1: k_f3_fast3<3, EIK, 1, true, PUSH><<<blocks, 256, sm, s>>>(a, tiles); break;
      case 2: k_f3_fast3<3, EIK, 2, true, PUSH><<<blocks, 256, sm, s>>>(a, tiles); break;
      case 3: k_f3_fast3<3, EIK, 3, true, PUSH><<<blocks, 256, sm, s>>>(a, tiles); break;
      default: k_f3_fast3<3, EIK, 4, true, PUSH><<<blocks, 256, sm, s>>>(a, tiles); break;
    }
    return;
  }
  if ((WD_S4 >> (stage - 1)) & 1) {
    switch (stage) {
      case 1: k_f3_fast4<3, EIK, 1, PUSH><<<blocks, 128, sm, s>>>(a, tiles); break;
      case 2: k_f3_fast4<3, EIK, 2, PUSH><<<blocks, 128, sm, s>>>(a, tiles); break;
      case 3: k_f3_fast4<3, EIK, 3, PUSH><<<blocks, 128, sm, s>>>(a, tiles); break;
      default: k_f3_fast4<3, EIK, 4, PUSH><<<blocks, 128, sm, s>>>(a, tiles); break;
    }
    return;
  }
  switch (stage) {
    case 1: k_f3_fast3<3, EIK, 1, false, PUSH><<<blocks, 256, sm, s>>>(a, tiles); break;
    case 2: k_f3_fast3<3, EIK, 2, false, PUSH><<<blocks, 256, sm, s>>>(a, tiles); break;
    case 3: k_f3_fast3<3, EIK, 3, false, PUSH><<<blocks, 256, sm, s>>>(a, tiles); break;
    default: k_f3_fast3<3, EIK, 4, false, PUSH><<<blocks, 256, sm, s>>>(a, tiles); break;
  }
}

// the peer-memory (PUSH) instantiations exist for HJ only
template <bool EIK>
void launch_fast3(int stage, F3Args a, int ntiles, const int* tiles, int chunks, cudaStream_t s,
                  bool jb) {
  if constexpr (!EIK) {
    if (a.peer_l != nullptr) {
      static const bool prepared = [] {
        const int sm = (int)S3Layout<3>::SMEM;
        auto set = [&](const void* f) {
          return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) ==
                 cudaSuccess;
        };
        return set((const void*)k_f3_fast3<3, false, 1, false, true>) &&
               set((const void*)k_f3_fast3<3, false, 2, false, true>) &&
               set((const void*)k_f3_fast3<3, false, 3, false, true>) &&
               set((const void*)k_f3_fast3<3, false, 4, false, true>) &&
               set((const void*)k_f3_fast3<3, false, 1, true, true>) &&
               set((const void*)k_f3_fast3<3, false, 2, true, true>) &&
               set((const void*)k_f3_fast3<3, false, 3, true, true>) &&
               set((const void*)k_f3_fast3<3, false, 4, true, true>) &&
               set((const void*)k_f3_fast4<3, false, 1, true>) &&
               set((const void*)k_f3_fast4<3, false, 2, true>) &&
               set((const void*)k_f3_fast4<3, false, 3, true>) &&
               set((const void*)k_f3_fast4<3, false, 4, true>);
      }();
      (void)prepared;
      launch_fast3_impl<false, true>(stage, a, ntiles, tiles, chunks, s, jb);
      return;
    }
  }
  a.peer_l = a.peer_r = nullptr;
  launch_fast3_impl<EIK, false>(stage, a, ntiles, tiles, chunks, s, jb);
}

// i-chunks for the fast3 grid: few partial waves over 2 CTAs / SM, long
// enough chunks that the 2R-plane window prologue stays cheap
int fast3_chunks(int ntiles, int ni) {
  if (const char* f = getenv("WD_F3_CHUNKS")) {  // A/B of the cost model below
    const int c = atoi(f);
    if (c >= 1 && c <= ni) return c;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const double slots = 2.0 * sms;
  // time ~ waves x (chunk length + window prologue, a 13-plane read worth
  // about 3 computed planes); more chunks = shorter tail, more re-reads
  int best = 1;
  double bc = 1e30;
  for (int c = 1; c <= 32; ++c) {
    const int len = (ni + c - 1) / c;
    if (len < 16 && c > 1) break;
    const double waves = std::ceil(ntiles * (double)c / slots);
    const double cost = waves * (len + 3.0);
    if (cost < bc - 1e-9) {
      bc = cost;
      best = c;
    }
  }
  return best;
}

int fast3_lowstorage() { return S3_LS ? 1 : 0; }

template bool fast3_prepare<true>();
template bool fast3_prepare<false>();
template void launch_fast3<true>(int, F3Args, int, const int*, int, cudaStream_t, bool);
template void launch_fast3<false>(int, F3Args, int, const int*, int, cudaStream_t, bool);

}  // namespace wd
