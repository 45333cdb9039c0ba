// Fast-arithmetic E6 stage kernels (wd_stage_fast.cuh) in their own
// translation unit: launch helpers used by wd_fused.cu.
#include <cmath>

#include "wd_stage_fast.cuh"

namespace wd {

// fast interior tiles, E6: cp.async-pipelined stage (wd_stage_fast.cuh) with
// its own i-chunking (grid a multiple of the resident CTA slots)
template <bool EIK>
bool fast3_prepare() {
  const int sm = (int)S3Layout<3>::SMEM;
  auto set = [&](const void* f) {
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, sm) == cudaSuccess;
  };
  return set((const void*)k_f3_fast3<3, EIK, 1>) && set((const void*)k_f3_fast3<3, EIK, 2>) &&
         set((const void*)k_f3_fast3<3, EIK, 3>) && set((const void*)k_f3_fast3<3, EIK, 4>);
}

template <bool EIK>
void launch_fast3(int stage, F3Args a, int ntiles, const int* tiles, int chunks, cudaStream_t s) {
  const int ni = a.i_hi - a.i_lo;
  a.chunk = (ni + chunks - 1) / chunks;
  const int blocks = chunks * ntiles;
  const size_t sm = S3Layout<3>::SMEM;
  switch (stage) {
    case 1: k_f3_fast3<3, EIK, 1><<<blocks, 256, sm, s>>>(a, tiles); break;
    case 2: k_f3_fast3<3, EIK, 2><<<blocks, 256, sm, s>>>(a, tiles); break;
    case 3: k_f3_fast3<3, EIK, 3><<<blocks, 256, sm, s>>>(a, tiles); break;
    default: k_f3_fast3<3, EIK, 4><<<blocks, 256, sm, s>>>(a, tiles); break;
  }
}

// i-chunks for the fast3 grid: few partial waves over 2 CTAs / SM, long
// enough chunks that the 2R-plane window prologue stays cheap
int fast3_chunks(int ntiles, int ni) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const double slots = 2.0 * sms;
  int best = 1;
  double bc = 1e30;
  for (int c = 1; c <= 32; ++c) {
    const int len = (ni + c - 1) / c;
    if (len < 16 && c > 1) break;
    const double waves = ntiles * (double)c / slots;
    const double cost = std::ceil(waves) / c * (len + 12.0);
    if (cost < bc - 1e-9) {
      bc = cost;
      best = c;
    }
  }
  return best;
}

template bool fast3_prepare<true>();
template bool fast3_prepare<false>();
template void launch_fast3<true>(int, F3Args, int, const int*, int, cudaStream_t);
template void launch_fast3<false>(int, F3Args, int, const int*, int, cudaStream_t);

}  // namespace wd
