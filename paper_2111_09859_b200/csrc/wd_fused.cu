// Specialised pseudo-step paths (see wd_fused.cuh).
//
// PATH_F3: 3-D, uniform Cartesian metrics, explicit E2/E4/E6, HJ or
// Eikonal, wall / periodic faces only (no far-field copies, no solid
// mask).  Covers BASELINE config 4 (512^3 channel) and 3-D wall-bounded
// boxes.  Everything else runs the generic kernels.
#include "wd_fused.cuh"
#include "wd_fused3d.cuh"
#include "wd_filter_sweep.cuh"
#include "wd_filter_scan.cuh"

#include <cmath>
#include <cstring>
#include <vector>

namespace wd {

// wd_stage_fast.cu
template <bool EIK> bool fast3_prepare();
template <bool EIK>
void launch_fast3(int stage, F3Args a, int ntiles, const int* tiles, int chunks, cudaStream_t s,
                  bool jb);
int fast3_chunks(int ntiles, int ni);

namespace {
constexpr int PATH_F3 = 1;

int grid_blocks(long long work, int threads) {
  long long b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  return (int)(b < 148LL * 32 ? b : 148LL * 32);
}

template <int R, bool EIK>
void launch_stage(int stage, const F3Args& a, int blocks, const int* tiles, bool fast,
                  cudaStream_t s) {
  const dim3 thr(F3_TK, F3_TJ);
  const size_t sm = F3_SMEM_DOUBLES * sizeof(double);
  if (fast && (a.n2 & 1)) {  // odd rows: 16-byte pairs would be misaligned
    const size_t smf = 2 * F3_PH * F3_PW * sizeof(double);
    switch (stage) {
      case 1: k_f3_fast<R, EIK, 1><<<blocks, thr, smf, s>>>(a, tiles); break;
      case 2: k_f3_fast<R, EIK, 2><<<blocks, thr, smf, s>>>(a, tiles); break;
      case 3: k_f3_fast<R, EIK, 3><<<blocks, thr, smf, s>>>(a, tiles); break;
      default: k_f3_fast<R, EIK, 4><<<blocks, thr, smf, s>>>(a, tiles); break;
    }
    return;
  }
  if (fast) {
    const dim3 thr2(16, F3_TJ);
    const size_t smf = 2 * F2_PH * F2_PW * sizeof(double);
    switch (stage) {
      case 1: k_f3_fast2<R, EIK, 1><<<blocks, thr2, smf, s>>>(a, tiles); break;
      case 2: k_f3_fast2<R, EIK, 2><<<blocks, thr2, smf, s>>>(a, tiles); break;
      case 3: k_f3_fast2<R, EIK, 3><<<blocks, thr2, smf, s>>>(a, tiles); break;
      default: k_f3_fast2<R, EIK, 4><<<blocks, thr2, smf, s>>>(a, tiles); break;
    }
    return;
  }
  switch (stage) {
    case 1: k_f3_stage<R, EIK, 1><<<blocks, thr, sm, s>>>(a, tiles); break;
    case 2: k_f3_stage<R, EIK, 2><<<blocks, thr, sm, s>>>(a, tiles); break;
    case 3: k_f3_stage<R, EIK, 3><<<blocks, thr, sm, s>>>(a, tiles); break;
    default: k_f3_stage<R, EIK, 4><<<blocks, thr, sm, s>>>(a, tiles); break;
  }
}

size_t sweep_smem(int n) {
  return (6 * (size_t)n + (size_t)((n + FB - 1) / FB) * 128 + 4 * 32 * 17) * sizeof(double);
}

void launch_sweep(const SweepArgs& w, cudaStream_t s) {
  const int per_row = ((w.axis == 2 ? w.n1 : w.n2) + 31) / 32;
  const long long outer = w.axis == 0 ? w.n1 : w.n0;
  const long long groups = outer * per_row;
  long long ctas = (groups + 3) / 4;
  if (ctas > 148LL * 8) ctas = 148LL * 8;
  if (w.axis == 2)
    k_filter_sweep<true><<<(int)ctas, 128, sweep_smem(w.n), s>>>(w);
  else
    k_filter_sweep<false><<<(int)ctas, 128, sweep_smem(w.n), s>>>(w);
}

// Tensor maps for the TMA tile loads of a strided sweep (wd_filter_scan.cuh).
// cuTensorMapEncodeTiled is resolved through the runtime (no libcuda link).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) ==
            cudaSuccess && qr == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
    cudaGetLastError();
  }
  return fn;
}

bool scan_tma_maps(const ScanArgs& a, ScanTma& tm) {
  // opt-in: measured slower than the per-thread cp.async staging on this
  // tile shape (128-byte rows, 522 row requests per tile through the SM's one
  // TMA unit): i / j sweeps 0.547 / 0.518 ms vs 0.499 / 0.460 ms at 512^3
  // (profiles/r02k_tma_ab.json); kept for wider-row tilings
  static const bool off = getenv("WD_TMA") == nullptr;
  EncodeTiledFn enc = encode_tiled();
  const int n = a.T.n;
  if (off || !enc || a.axis == 2 || (a.n2 % FS_L) != 0 || n / 2 > 256 || (n & 1) ||
      ((uintptr_t)a.in & 15))
    return false;
  const cuuint32_t es[3] = {1, 1, 1};
  void* base = const_cast<double*>(a.in);
  auto make = [&](CUtensorMap* m, int rows) {
    if (a.axis == 0) {  // (n0 rows) x (n1 n2 contiguous)
      const cuuint64_t dims[2] = {(cuuint64_t)a.n1 * a.n2, (cuuint64_t)a.n0};
      const cuuint64_t strides[1] = {(cuuint64_t)a.s0 * 8};
      const cuuint32_t box[2] = {(cuuint32_t)FS_L, (cuuint32_t)rows};
      return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    const cuuint64_t dims[3] = {(cuuint64_t)a.n2, (cuuint64_t)a.n1, (cuuint64_t)a.n0};
    const cuuint64_t strides[2] = {(cuuint64_t)a.n2 * 8, (cuuint64_t)a.s0 * 8};
    const cuuint32_t box[3] = {(cuuint32_t)FS_L, (cuuint32_t)rows, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  return make(&tm.main, n / 2) == CUDA_SUCCESS && make(&tm.ghost, FS_G) == CUDA_SUCCESS;
}

// fast arithmetic: segmented-scan filter (wd_filter_scan.cuh), persistent
// grid of resident CTAs
template <bool AX2, int MM, bool RED, bool TMA>
void scan_launch(const ScanArgs& a, const ScanTma& tm, long long groups, cudaStream_t s) {
  static int ctas = 0;
  const size_t smax = scan_smem(FS_NMAX);
  if (!ctas) {
    int dev = 0, sms = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_filter_scan<AX2, MM, RED, TMA>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_filter_scan<AX2, MM, RED, TMA>, FS_T,
                                                  smax);
    ctas = sms * (occ > 0 ? occ : 1);
  }
  const long long c = ctas < groups ? ctas : groups;
  k_filter_scan<AX2, MM, RED, TMA><<<(int)c, FS_T, scan_smem(a.T.n), s>>>(a, tm);
}

template <bool AX2, int MM, bool RED>
void scan_one(const ScanArgs& a, long long groups, cudaStream_t s) {
  ScanTma tm;
  std::memset(&tm, 0, sizeof(tm));
  if constexpr (!AX2 && MM > 0) {
    if (scan_tma_maps(a, tm)) {
      scan_launch<AX2, MM, RED, true>(a, tm, groups, s);
      return;
    }
  }
  scan_launch<AX2, MM, RED, false>(a, tm, groups, s);
}

// last sweep of the slab-decomposed step with the axis-0 correction fused
template <int MM>
void scan_fix(const ScanArgs& a, long long groups, cudaStream_t s) {
  ScanTma tm;
  std::memset(&tm, 0, sizeof(tm));
  static int ctas = 0;
  const size_t smax = scan_smem(FS_NMAX);
  if (!ctas) {
    int dev = 0, sms = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_filter_scan<true, MM, true, false, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ, k_filter_scan<true, MM, true, false, true>, FS_T, smax);
    ctas = sms * (occ > 0 ? occ : 1);
  }
  const long long c = ctas < groups ? ctas : groups;
  k_filter_scan<true, MM, true, false, true><<<(int)c, FS_T, scan_smem(a.T.n), s>>>(a, tm);
}

template <bool AX2, bool RED>
void scan_mm(const ScanArgs& a, long long groups, cudaStream_t s) {
  static const bool generic = getenv("WD_SCAN_GENERIC") != nullptr;  // A/B knob
  if constexpr (AX2 && RED) {
    if (a.fixc) {
      if (a.T.n == FS_S * FS_M && !generic) scan_fix<FS_M>(a, groups, s);
      else if (a.T.n == FS_S * 16 && !generic) scan_fix<16>(a, groups, s);
      else scan_fix<0>(a, groups, s);
      return;
    }
  }
  if (a.T.n == FS_S * FS_M && !generic) scan_one<AX2, FS_M, RED>(a, groups, s);
  else if (a.T.n == FS_S * 16 && !generic) scan_one<AX2, 16, RED>(a, groups, s);
  else scan_one<AX2, 0, RED>(a, groups, s);
}

bool scan_prepare() { return FS_NMAX > 0; }

void launch_scan(const SweepArgs& w, const ScanDev& T, cudaStream_t s) {
  ScanArgs a;
  a.in = w.in;
  a.out = w.out;
  a.axis = w.axis;
  a.n0 = w.n0;
  a.n1 = w.n1;
  a.n2 = w.n2;
  a.s0 = w.s0;
  a.per = w.per;
  a.T = T;
  a.fc = w.fc;
  a.A = w.A;
  a.st = w.st;
  a.fixc = w.axis == 2 && w.A ? w.fixc : nullptr;
  a.fixrow = w.fixrow;
  const long long inner = w.axis == 2 ? w.n1 : w.n2;
  const long long outer = w.axis == 0 ? w.n1 : w.n0;
  const long long groups = outer * ((inner + FS_L - 1) / FS_L);
  if (w.axis == 2) {
    if (w.A) scan_mm<true, true>(a, groups, s);
    else scan_mm<true, false>(a, groups, s);
  } else {
    if (w.A) scan_mm<false, true>(a, groups, s);
    else scan_mm<false, false>(a, groups, s);
  }
}

void stage_dispatch(int R, bool eik, int stage, const F3Args& a, int blocks, const int* tiles,
                    bool fast, cudaStream_t s) {
  if (R == 1) eik ? launch_stage<1, true>(stage, a, blocks, tiles, fast, s) : launch_stage<1, false>(stage, a, blocks, tiles, fast, s);
  else if (R == 2) eik ? launch_stage<2, true>(stage, a, blocks, tiles, fast, s) : launch_stage<2, false>(stage, a, blocks, tiles, fast, s);
  else eik ? launch_stage<3, true>(stage, a, blocks, tiles, fast, s) : launch_stage<3, false>(stage, a, blocks, tiles, fast, s);
}
}  // namespace

void fused_plan(FusedPlan& fp, const FusedInputs& in) {
  fp.active = 0;
  fp.in = in;
  const wd_grid_desc& gd = *in.gd;
  const wd_solver_desc& sd = *in.sd;
  if (const char* env = getenv("WD_DISABLE_FUSED")) {
    if (env[0] == '1') return;
  }
  if (gd.ndim != 3 || !gd.uniform || gd.solid_mask_dev != nullptr) return;
  if (sd.scheme != WD_E2 && sd.scheme != WD_E4 && sd.scheme != WD_E6) return;
  if (sd.kind != WD_HJ && sd.kind != WD_EIKONAL) return;
  for (int f = 0; f < 6; ++f)
    if (gd.face[f] == WD_FACE_FARFIELD) return;
  if (sd.use_filter) {
    for (int a = 0; a < 3; ++a)
      if (in.filt_swaps[a]) return;
    int nmax = 0;
    for (int a = 0; a < 3; ++a) nmax = in.g.n[a] > nmax ? in.g.n[a] : nmax;
    const int smem = (int)sweep_smem(nmax);
    if (cudaFuncSetAttribute(k_filter_sweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem) != cudaSuccess ||
        cudaFuncSetAttribute(k_filter_sweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem) != cudaSuccess)
      return;
  }
  fp.kind = PATH_F3;
  fp.active = 1;
  fp.use_fast3 = 0;
  if (sd.arith == 1 && sd.scheme == WD_E6 && (in.g.n[2] % 2) == 0 &&
      in.g.N < (1LL << 31) - (1LL << 24) && !getenv("WD_NO_FAST3"))
    fp.use_fast3 = sd.kind == WD_EIKONAL ? fast3_prepare<true>() : fast3_prepare<false>();
  fp.use_scan = 0;
  if (sd.use_filter && sd.arith == 1 && scan_prepare()) {
    fp.use_scan = 1;
    for (int a = 0; a < 3; ++a)
      if (in.scan[a].n != in.g.n[a]) fp.use_scan = 0;
  }
  fp.filt_order[0] = 0;
  fp.filt_order[1] = 1;
  fp.filt_order[2] = 2;
  if (const char* o = getenv("WD_FILTER_ORDER")) {  // experiments: e.g. "201"
    if (sd.arith == 1 && strlen(o) == 3)
      for (int a = 0; a < 3; ++a) fp.filt_order[a] = o[a] - '0';
  }
  fp.n_fast = fp.n_exact = 0;
  if (sd.arith == 1) {
    // interior tiles (every stencil inside or periodic) -> fast kernel
    const Geom& g = in.g;
    const int tk = (g.n[2] + F3_TK - 1) / F3_TK, tj = (g.n[1] + F3_TJ - 1) / F3_TJ;
    // fast: every stencil inside or periodic; jb: k interior, touching a
    // non-periodic j end (fast3 closure variant, else exact); exact: the rest
    std::vector<int> fastl(1, 0), jbl(1, 0), exactl(1, 0);
    for (int t = 0; t < tk * tj; ++t) {
      const int k0 = (t % tk) * F3_TK, j0 = (t / tk) * F3_TJ;
      const bool kf = g.per[2] ? (k0 + F3_TK <= g.n[2]) : (k0 >= F3_HP && k0 + F3_TK + F3_HP <= g.n[2]);
      const bool jf = g.per[1] ? (j0 + F3_TJ <= g.n[1]) : (j0 >= F3_HP && j0 + F3_TJ + F3_HP <= g.n[1]);
      const bool jb = kf && !jf && !g.per[1] && j0 + F3_TJ <= g.n[1] && g.n[1] >= 2 * F3_TJ;
      (kf && jf ? fastl : (jb ? jbl : exactl)).push_back(t);
    }
    fastl[0] = (int)fastl.size() - 1;
    jbl[0] = (int)jbl.size() - 1;
    exactl[0] = (int)exactl.size() - 1;
    fp.n_fast = fastl[0];
    fp.n_jb = jbl[0];
    fp.n_exact = exactl[0];
    const size_t nt = fastl.size() + jbl.size() + exactl.size();
    if (cudaMalloc(&fp.tiles_dev, nt * sizeof(int)) != cudaSuccess ||
        upload_sync(fp.tiles_dev, fastl.data(), fastl.size() * sizeof(int)) != cudaSuccess ||
        upload_sync(fp.tiles_dev + fastl.size(), jbl.data(), jbl.size() * sizeof(int)) !=
            cudaSuccess ||
        upload_sync(fp.tiles_dev + fastl.size() + jbl.size(), exactl.data(),
                    exactl.size() * sizeof(int)) != cudaSuccess) {
      fp.active = 0;
      return;
    }
    fp.fast_tiles = fp.tiles_dev;
    fp.jb_tiles = fp.tiles_dev + fastl.size();
    fp.exact_tiles = fp.tiles_dev + fastl.size() + jbl.size();
    if ((fp.n_exact || fp.n_jb) && fp.n_fast) {
      if (cudaStreamCreateWithFlags(&fp.side, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&fp.ev_fork, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&fp.ev_join, cudaEventDisableTiming) != cudaSuccess)
        fp.side = nullptr;
    }
    const size_t smf = 2 * F3_PH * F3_PW * sizeof(double);
    (void)smf;
  }
}

namespace {
// fast3 needs every updated plane 2R = 6 away from a non-periodic axis-0 end
bool fast3_ok(const FusedPlan& fp, const F3Args& a) {
  return fp.use_fast3 && (a.per0 || (a.i_lo >= 6 && a.i_hi <= a.n0 - 6));
}

// One RK stage over the tile lists of a fast-arithmetic plan: boundary
// tiles (exact kernel, or the fast3 j-wall variant) on the forked side
// stream so they overlap the interior tiles on `s`.
void stage_tiles(const FusedPlan& fp, int stage, const F3Args& a, int chunks, int R, bool eik,
                 cudaStream_t s) {
  const bool f3 = fast3_ok(fp, a);
  const bool side = fp.side != nullptr;
  const cudaStream_t ss = side ? fp.side : s;
  const bool any_side = fp.n_exact || fp.n_jb;
  if (any_side && side) {
    cudaEventRecord(fp.ev_fork, s);
    cudaStreamWaitEvent(fp.side, fp.ev_fork, 0);
  }
  const int c3 = f3 ? fast3_chunks(fp.n_fast + fp.n_jb, a.i_hi - a.i_lo) : 0;
  if (fp.n_jb) {
    if (f3) {
      if (eik) launch_fast3<true>(stage, a, fp.n_jb, fp.jb_tiles, c3, ss, true);
      else launch_fast3<false>(stage, a, fp.n_jb, fp.jb_tiles, c3, ss, true);
    } else {
      stage_dispatch(R, eik, stage, a, chunks * fp.n_jb, fp.jb_tiles, false, ss);
    }
  }
  if (fp.n_exact) stage_dispatch(R, eik, stage, a, chunks * fp.n_exact, fp.exact_tiles, false, ss);
  if (any_side && side) cudaEventRecord(fp.ev_join, fp.side);
  if (fp.n_fast) {
    if (f3) {
      if (eik) launch_fast3<true>(stage, a, fp.n_fast, fp.fast_tiles, c3, s, false);
      else launch_fast3<false>(stage, a, fp.n_fast, fp.fast_tiles, c3, s, false);
    } else {
      stage_dispatch(R, eik, stage, a, chunks * fp.n_fast, fp.fast_tiles, true, s);
    }
  }
  if (any_side && side) cudaStreamWaitEvent(s, fp.ev_join, 0);
}

F3Args f3_args(const FusedPlan& fp, const double* A, Status* st, int* blocks) {
  const FusedInputs& in = fp.in;
  const wd_grid_desc& gd = *in.gd;
  const wd_solver_desc& sd = *in.sd;
  const Geom& g = in.g;
  F3Args a;
  a.n0 = g.n[0];
  a.n1 = g.n[1];
  a.n2 = g.n[2];
  a.s0 = (long long)g.n[1] * g.n[2];
  a.per0 = g.per[0];
  a.per1 = g.per[1];
  a.per2 = g.per[2];
  for (int f = 0; f < 6; ++f) a.wall[f] = gd.face[f] == WD_FACE_WALL;
  a.c0 = gd.inv_spacing[0];
  a.c1 = gd.inv_spacing[1];
  a.c2 = gd.inv_spacing[2];
  a.eps = sd.epsilon;
  a.cfl = sd.cfl;
  a.sumS = in.sumS_c;
  a.cflms = in.cflms_c;
  a.A = A;
  a.dt = in.bufs[0];
  a.acc = in.bufs[1];
  a.st = st;
  a.tiles_k = (a.n2 + F3_TK - 1) / F3_TK;
  a.tiles_j = (a.n1 + F3_TJ - 1) / F3_TJ;
  const int tiles = a.tiles_k * a.tiles_j;
  // split the i-stream so the grid is several waves of 148 SMs
  a.i_lo = fp.i_lo;
  a.i_hi = fp.i_hi > 0 ? fp.i_hi : a.n0;
  const int ni = a.i_hi - a.i_lo;
  int chunks = 1;
  while ((long long)tiles * chunks < 148LL * 8 && ni / (chunks * 2) >= 32) chunks *= 2;
  a.chunk = (ni + chunks - 1) / chunks;
  *blocks = chunks;  // caller multiplies by its tile count
  // fast-mode coefficients (host doubles)
  const int R = sd.scheme == WD_E2 ? 1 : (sd.scheme == WD_E4 ? 2 : 3);
  double c[4] = {0.0, 0.0, 0.0, 0.0};
  if (R == 1) {
    c[1] = E2_CA;
  } else if (R == 2) {
    c[1] = E4_CA;
    c[2] = E4_CB;
  } else {
    c[1] = E6_CA;
    c[2] = E6_CB;
    c[3] = E6_CC;
  }
  for (int r = 0; r < 4; ++r) a.cr[r] = c[r];
  double e[7] = {0, 0, 0, 0, 0, 0, 0};
  for (int r = 1; r <= 3; ++r)
    for (int q = 1; q <= 3; ++q) {
      const double w = c[r] * c[q];
      e[r + q] += w;                          // p_{+(r+q)}
      if (r > q) e[r - q] -= w;               // -p_{r-q}
      else if (q > r) e[q - r] -= w;          // -p_{-(r-q)} (symmetric)
      else e[0] -= 2.0 * w;                   // r == q: -p_0 - p_0
    }
  for (int m = 0; m < 7; ++m) a.e[m] = e[m];
  a.cc0 = a.c0 * a.c0;
  a.cc1 = a.c1 * a.c1;
  a.cc2 = a.c2 * a.c2;
  const double cc[3] = {a.cc0, a.cc1, a.cc2};
  a.fE0 = 0.0;
  for (int l = 0; l < 3; ++l) {
    a.fsq[l] = std::sqrt(cc[l]);
    for (int m = 0; m < 4; ++m) a.fC[l][m] = a.fsq[l] * c[m];
    for (int m = 0; m < 7; ++m) a.fE[l][m] = cc[l] * e[m];
    a.fE0 += cc[l] * e[0];
  }
  return a;
}
}  // namespace

// kid 1..4: RK stages, 5..7: filter sweeps, 8: change reduction
void fused_launch(const FusedPlan& fp, int kid, const double* A, double* B, Status* st,
                  cudaStream_t s) {
  const FusedInputs& in = fp.in;
  const wd_solver_desc& sd = *in.sd;
  const Geom& g = in.g;
  double* bp = in.bufs[2];
  double* bk = in.bufs[3];
  double* tmp = in.bufs[4];
  int chunks = 0;
  F3Args a = f3_args(fp, A, st, &chunks);
  const int all_tiles = a.tiles_k * a.tiles_j;
  const int R = sd.scheme == WD_E2 ? 1 : (sd.scheme == WD_E4 ? 2 : 3);
  const bool eik = sd.kind == WD_EIKONAL;
  switch (kid) {
    case 1: a.p = A; a.out = bp; break;
    case 2: a.p = bp; a.out = bk; break;
    case 3: a.p = bk; a.out = bp; break;
    case 4: a.p = bp; a.out = sd.use_filter ? bk : B; break;
    default: break;
  }
  if (kid >= 1 && kid <= 4) {
    if (fp.fast_tiles) {
      stage_tiles(fp, kid, a, chunks, R, eik, s);
    } else {
      stage_dispatch(R, eik, kid, a, chunks * all_tiles, nullptr, false, s);
    }
  } else if (kid >= 5 && kid <= 7) {
    // position kid-5 in the sweep sequence -> axis (fast arithmetic may use
    // another axis order: the 1-D filters commute up to round-off)
    const int pos = kid - 5;
    const int ax = fp.filt_order[pos];
    const double* srcs[3] = {bk, tmp, bp};
    double* dsts[3] = {tmp, bp, B};
    SweepArgs w;
    w.in = srcs[pos];
    w.out = dsts[pos];
    w.n = g.n[ax];
    w.axis = ax;
    w.n0 = g.n[0];
    w.n1 = g.n[1];
    w.n2 = g.n[2];
    w.s0 = (long long)g.n[1] * g.n[2];
    w.per = g.per[ax];
    const TriDev& T = in.filt[ax];
    w.fact = T.fact;
    w.du = T.du;
    w.d = T.d;
    w.rinv = T.rinv;
    w.z = T.z;
    w.h = T.h;
    w.denom = T.denom;
    w.fc = in.fcoef;
    w.A = pos == 2 ? A : nullptr;
    w.st = st;
    if (fp.use_scan) launch_scan(w, in.scan[ax], s);
    else launch_sweep(w, s);
  } else if (kid == 8) {
    k_change<<<grid_blocks(g.N, 256), 256, 0, s>>>(B, A, nullptr, st, g.N);
  }
}

void fused_stage_ptrs(const FusedPlan& fp, int stage, const double* A, const double* p,
                      double* out, Status* st, cudaStream_t s) {
  const wd_solver_desc& sd = *fp.in.sd;
  int chunks = 0;
  F3Args a = f3_args(fp, A, st, &chunks);
  const int all_tiles = a.tiles_k * a.tiles_j;
  const int R = sd.scheme == WD_E2 ? 1 : (sd.scheme == WD_E4 ? 2 : 3);
  const bool eik = sd.kind == WD_EIKONAL;
  a.p = p;
  a.out = out;
  if (fp.peer_ws_l && fp.peer_ws_r && fast3_ok(fp, a) && !fp.n_exact) {
    const long long off = out - fp.ws_base;
    a.peer_l = fp.peer_ws_l + off;
    a.peer_r = fp.peer_ws_r + off;
    a.push_shift = (long long)fp.push_nl * a.s0;
    a.push_l_end = 2 * fp.push_G;
    a.push_r_beg = fp.push_nl;
  }
  if (fp.fast_tiles) {
    stage_tiles(fp, stage, a, chunks, R, eik, s);
  } else {
    stage_dispatch(R, eik, stage, a, chunks * all_tiles, nullptr, false, s);
  }
}

bool fused_can_push(const FusedPlan& fp) {
  return fp.active && fp.use_fast3 && fp.fast_tiles != nullptr && fp.n_exact == 0 &&
         fp.in.sd->kind == WD_HJ;
}

void fused_filter_any(const FusedPlan& fp, int axis, const double* in, double* out, int n0,
                      int n1, int n2, int per, const TriDev& T, const double* A, Status* st,
                      cudaStream_t s, const ScanDev* scan, const double* fixc,
                      const double* fixrow) {
  SweepArgs w;
  w.fixc = fixc;
  w.fixrow = fixrow;
  w.in = in;
  w.out = out;
  const int nn[3] = {n0, n1, n2};
  w.n = nn[axis];
  w.axis = axis;
  w.n0 = n0;
  w.n1 = n1;
  w.n2 = n2;
  w.s0 = (long long)n1 * n2;
  w.per = per;
  w.fact = T.fact;
  w.du = T.du;
  w.d = T.d;
  w.rinv = T.rinv;
  w.z = T.z;
  w.h = T.h;
  w.denom = T.denom;
  w.fc = fp.in.fcoef;
  w.A = A;
  w.st = st;
  if (scan && scan->n == w.n && scan_prepare()) launch_scan(w, *scan, s);
  else launch_sweep(w, s);
}

void fused_filter_prepare(int n) {
  const int smem = (int)sweep_smem(n);
  cudaFuncAttributes attr;
  if (cudaFuncGetAttributes(&attr, k_filter_sweep<true>) == cudaSuccess &&
      smem > attr.maxDynamicSharedSizeBytes)
    cudaFuncSetAttribute(k_filter_sweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (cudaFuncGetAttributes(&attr, k_filter_sweep<false>) == cudaSuccess &&
      smem > attr.maxDynamicSharedSizeBytes)
    cudaFuncSetAttribute(k_filter_sweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

void fused_step(const FusedPlan& fp, const double* A, double* B, Status* st, double* hist,
                cudaStream_t s) {
  const FusedInputs& in = fp.in;
  const wd_solver_desc& sd = *in.sd;
  for (int kid = 1; kid <= 4; ++kid) fused_launch(fp, kid, A, B, st, s);
  if (sd.use_filter)
    for (int kid = 5; kid <= 7; ++kid) fused_launch(fp, kid, A, B, st, s);  // 7 reduces
  else
    fused_launch(fp, 8, A, B, st, s);
  k_finalize<<<1, 1, 0, s>>>(st, hist, in.lref, sd.tol, 1e6 * in.lref);
}

void fused_release(FusedPlan& fp) {
  if (fp.side) {
    cudaStreamSynchronize(fp.side);
    cudaStreamDestroy(fp.side);
    cudaEventDestroy(fp.ev_fork);
    cudaEventDestroy(fp.ev_join);
    fp.side = nullptr;
  }
  if (fp.tiles_dev) cudaFree(fp.tiles_dev);
  fp.tiles_dev = nullptr;
  fp.active = 0;
}

}  // namespace wd
