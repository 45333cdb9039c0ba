// Specialised (fused) pseudo-step kernels.  A FusedPlan is built at
// context creation when the configuration matches a specialised path; the
// generic kernels of wd_kernels.cuh handle everything else.
#pragma once

#include <cstdlib>
#include "wd_kernels.cuh"

namespace wd {

// Fast-arithmetic filter in scan form (wd_filter_scan.cuh): 16 lines per
// CTA x 16 segments of <= 32 rows; 7 tables of n doubles per axis
// (f_{r-1}, P, 1/d, du/d, Q, z, h).
constexpr int FS_L = 16;
constexpr int FS_S = 16;
constexpr int FS_M = 32;
constexpr int FS_T = FS_L * FS_S;
constexpr int FS_NMAX = FS_S * FS_M;
constexpr int FS_G = 5;

struct ScanDev {
  int n = 0, m = 0;
  const double* tab = nullptr;
  double denom = 1.0;
};

struct FusedInputs {
  const wd_grid_desc* gd;
  const wd_solver_desc* sd;
  Geom g;
  Metric M;
  FilterCoef fcoef;
  TriDev filt[3];
  ScanDev scan[3];  // n = 0: no scan form for this axis
  int filt_swaps[3];
  double sumS_c, cflms_c, lref;
  double* bufs[6];  // dt, acc, p, k, tmp, tmp2 (N each)
};

struct FusedPlan {
  int active = 0;
  int kind = 0;          // which specialised path
  FusedInputs in;
  // fast arithmetic: interior tiles -> k_f3_fast, boundary tiles -> exact
  int* tiles_dev = nullptr;
  const int* fast_tiles = nullptr;
  const int* exact_tiles = nullptr;
  const int* jb_tiles = nullptr;  // k interior, touching a j wall
  int n_fast = 0, n_exact = 0, n_jb = 0;
  cudaStream_t side = nullptr;  // boundary tiles overlap the interior launch
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int i_lo = 0, i_hi = 0;  // axis-0 plane range updated by the stages (0,0 = all)
  int use_scan = 0;        // fast arithmetic: segmented-scan filter sweeps
  int use_fast3 = 0;       // fast arithmetic, E6: cp.async-pipelined stage kernel
  int filt_order[3] = {0, 1, 2};  // axis of each filter sweep (reference order 0, 1, 2)
  // peer-memory ghost push of the fast E6 stage kernels (wd_dist.cuh): the
  // neighbours' images of this rank's workspace; 0 = off
  const double* ws_base = nullptr;
  double* peer_ws_l = nullptr;
  double* peer_ws_r = nullptr;
  int push_nl = 0, push_G = 0;
};

// Decide whether a specialised path applies; fills fp (fp.active = 1).
void fused_plan(FusedPlan& fp, const FusedInputs& in);
// 1 when the fast E6 stage kernels run the low-storage RK4 (wd_stage_fast.cuh)
int fast3_lowstorage();
// One pseudo-step A -> B incl. change reduction and stop test.
void fused_step(const FusedPlan& fp, const double* A, double* B, Status* st, double* hist,
                cudaStream_t s);
void fused_release(FusedPlan& fp);
// Launch one kernel of the fused step (timing / profiling): kid 1..4 RK
// stages, 5..7 filter sweeps, 8 change reduction.
void fused_launch(const FusedPlan& fp, int kid, const double* A, double* B, Status* st,
                  cudaStream_t s);
// Distributed path: one RK stage with explicit buffers; a filter sweep on
// an arbitrary (n0, n1, n2) array with factor T (SweepArgs semantics).
void fused_stage_ptrs(const FusedPlan& fp, int stage, const double* A, const double* p,
                      double* out, Status* st, cudaStream_t s);
// the stage kernels of this plan can push ghost planes to peer memory
bool fused_can_push(const FusedPlan& fp);
void fused_filter_prepare(int n);  // opt in to the sweep's shared memory for length n
void fused_filter_any(const FusedPlan& fp, int axis, const double* in, double* out, int n0,
                      int n1, int n2, int per, const TriDev& T, const double* A, Status* st,
                      cudaStream_t s, const ScanDev* scan = nullptr, const double* fixc = nullptr,
                      const double* fixrow = nullptr);

}  // namespace wd
