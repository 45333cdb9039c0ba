// C ABI of libwd_b200.so: solver context, factor precomputation, pseudo-step
// enqueue (CUDA graphs), operator-level entry points.  See
// include/walldist_b200.h for the contract and the reference lines each
// entry point replaces.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <utility>
#include <vector>

#include "wd_kernels.cuh"
#include "wd_line_sweep.cuh"
#include "wd_fused.cuh"
#include "wd_metrics.cuh"
#include "wd_dist_filter0.cuh"
#include "wd_deriv_scan.cuh"
#include "wd_stage_explicit.cuh"
#include "wd_filter_long.cuh"

using namespace wd;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CK(expr)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (expr);                                                      \
    if (e_ != cudaSuccess)                                                        \
      return fail(WD_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr int kThreads = 256;
constexpr int kLineThreads = 64;

int nblocks(long long work, int threads) {
  long long b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  return (int)std::min<long long>(b, 148LL * 32);
}

// Launch with programmatic stream serialization (PDL, wd_common.cuh) when
// WD_PDL is set, else a plain launch.  Measured on the 2-D step (C1, 12 small
// kernels per step, CUDA-graph replay): 0.144 -> 0.177 ms per step WITH the
// programmatic edges (C3: 0.415 -> 0.428), i.e. slower than the plain
// kernel-to-kernel edges of the graph, so it is opt-in.
template <class... P, class... A>
void launch_pdl(void (*kern)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A&&... args) {
  static const bool off = getenv("WD_PDL") == nullptr;
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = off ? 0 : 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<P>(args)...);
}

int min_line(int scheme) {
  switch (scheme) {
    case WD_UW: return 3;
    case WD_E2: return 3;
    case WD_E4: return 5;
    default: return 7;  // E6, C4, C6
  }
}

const char* scheme_name(int s) {
  static const char* names[] = {"UW", "E2", "E4", "E6", "C4", "C6"};
  return (s >= 0 && s <= 5) ? names[s] : "?";
}

// ------------------------------------------------------------------ factors
// Host restatement of LAPACK dgtsv's elimination (oracle/wd.py:gtsv_factor);
// field-independent, so computed once per matrix.
struct HostFactor {
  int n = 0;
  int cyclic = 0;
  std::vector<double> fact, d, du, du2, swap, z, h;
  double vn = 0.0, denom = 1.0;
  int scan_m = 0;       // dist filters: scan-form tables appended at scan_off
  size_t scan_off = 0;
};

int gtsv_factor(int n, const double* lower, const double* diag, const double* upper,
                HostFactor& F) {
  F.n = n;
  F.d.assign(diag, diag + n);
  std::vector<double> dl(std::max(n - 1, 0)), du(std::max(n - 1, 0));
  for (int i = 0; i < n - 1; ++i) {
    dl[i] = lower[i + 1];
    du[i] = upper[i];
  }
  F.fact.assign(std::max(n, 1), 0.0);
  F.swap.assign(std::max(n, 1), 0.0);
  auto& d = F.d;
  for (int i = 0; i < n - 1; ++i) {
    double f;
    if (std::fabs(d[i]) >= std::fabs(dl[i])) {
      if (d[i] == 0.0) return fail(WD_ERR_ZERO_PIVOT, "zero pivot at row " + std::to_string(i + 1));
      f = dl[i] / d[i];
      d[i + 1] = d[i + 1] - f * du[i];
      dl[i] = 0.0;
    } else {
      f = d[i] / dl[i];
      d[i] = dl[i];
      double t = d[i + 1];
      d[i + 1] = du[i] - f * t;
      if (i < n - 2) {
        dl[i] = du[i + 1];
        du[i + 1] = -f * dl[i];
      }
      du[i] = t;
      F.swap[i] = 1.0;
    }
    F.fact[i] = f;
  }
  if (n > 0 && d[n - 1] == 0.0)
    return fail(WD_ERR_ZERO_PIVOT, "zero pivot at row " + std::to_string(n));
  F.du.assign(std::max(n, 1), 0.0);
  F.du2.assign(std::max(n, 1), 0.0);
  for (int i = 0; i < n - 1; ++i) F.du[i] = du[i];
  for (int i = 0; i < n - 2; ++i) F.du2[i] = dl[i];
  F.z.assign(std::max(n, 1), 0.0);
  return WD_OK;
}

void gtsv_apply_host(const HostFactor& F, std::vector<double>& x) {
  const int n = F.n;
  if (n == 1) {
    x[0] = x[0] / F.d[0];
    return;
  }
  for (int i = 0; i < n - 1; ++i) {
    const double f = F.fact[i];
    if (F.swap[i] != 0.0) {
      double t = x[i];
      double b1 = x[i + 1];
      x[i] = b1;
      x[i + 1] = t - f * b1;
    } else {
      x[i + 1] = x[i + 1] - f * x[i];
    }
  }
  x[n - 1] = x[n - 1] / F.d[n - 1];
  x[n - 2] = (x[n - 2] - F.du[n - 2] * x[n - 1]) / F.d[n - 2];
  for (int i = n - 3; i >= 0; --i) x[i] = ((x[i] - F.du[i] * x[i + 1]) - F.du2[i] * x[i + 2]) / F.d[i];
}

// EXTENSION: cyclic constant-coefficient tridiagonal by Sherman-Morrison
// (oracle/wd.py:cyclic_factor).
int cyclic_factor(double alpha, int n, HostFactor& F) {
  const double gamma = -1.0;
  std::vector<double> lower(n, alpha), upper(n, alpha), diag(n, 1.0);
  lower[0] = 0.0;
  upper[n - 1] = 0.0;
  diag[0] = 1.0 - gamma;
  diag[n - 1] = 1.0 - alpha * alpha / gamma;
  int rc = gtsv_factor(n, lower.data(), diag.data(), upper.data(), F);
  if (rc) return rc;
  std::vector<double> u(n, 0.0);
  u[0] = gamma;
  u[n - 1] = alpha;
  gtsv_apply_host(F, u);
  F.z = u;
  F.vn = alpha / gamma;
  std::vector<double> v(n, 0.0);
  v[0] = 1.0;
  v[n - 1] = F.vn;
  gtsv_apply_host(F, v);
  F.h = v;
  F.denom = 1.0 + (u[0] + F.vn * u[n - 1]);
  if (F.denom == 0.0) return fail(WD_ERR_ZERO_PIVOT, "singular cyclic system");
  F.cyclic = 1;
  return WD_OK;
}

int compact_factor(int scheme, int n, int periodic, HostFactor& F) {
  const double alpha = scheme == WD_C4 ? 0.25 : 1.0 / 3.0;
  if (periodic) return cyclic_factor(alpha, n, F);
  std::vector<double> lower(n, alpha), diag(n, 1.0), upper(n, alpha);
  lower[0] = 0.0;
  upper[0] = 3.0;
  upper[n - 1] = 0.0;
  lower[n - 1] = 3.0;
  if (scheme == WD_C6) {
    lower[1] = upper[1] = 0.25;
    lower[n - 2] = upper[n - 2] = 0.25;
  }
  return gtsv_factor(n, lower.data(), diag.data(), upper.data(), F);
}

// arith="fast": the same compact matrix factored WITHOUT interchanges
// (Thomas), the swap-free form the scan solve needs (wd_deriv_scan.cuh);
// periodic axes keep the cyclic factor (already swap-free).
int compact_factor_fast(int scheme, int n, int periodic, HostFactor& F) {
  const double alpha = scheme == WD_C4 ? 0.25 : 1.0 / 3.0;
  if (periodic) return cyclic_factor(alpha, n, F);
  std::vector<double> lower(n, alpha), diag(n, 1.0), upper(n, alpha);
  lower[0] = 0.0;
  upper[0] = 3.0;
  upper[n - 1] = 0.0;
  lower[n - 1] = 3.0;
  if (scheme == WD_C6) {
    lower[1] = upper[1] = 0.25;
    lower[n - 2] = upper[n - 2] = 0.25;
  }
  F = HostFactor();
  F.n = n;
  F.d = diag;
  F.fact.assign(n, 0.0);
  F.swap.assign(n, 0.0);
  F.du.assign(n, 0.0);
  F.du2.assign(n, 0.0);
  F.z.assign(n, 0.0);
  for (int i = 0; i < n - 1; ++i) {
    if (F.d[i] == 0.0) return fail(WD_ERR_ZERO_PIVOT, "zero pivot at row " + std::to_string(i + 1));
    const double f = lower[i + 1] / F.d[i];
    F.d[i + 1] = F.d[i + 1] - f * upper[i];
    F.fact[i] = f;
    F.du[i] = upper[i];
  }
  if (F.d[n - 1] == 0.0) return fail(WD_ERR_ZERO_PIVOT, "zero pivot at row " + std::to_string(n));
  return WD_OK;
}
int filter_factor(double af, int n, int periodic, HostFactor& F) {
  if (periodic) return cyclic_factor(af, n, F);
  std::vector<double> lower(n, af), diag(n, 1.0), upper(n, af);
  upper[0] = 0.0;
  lower[n - 1] = 0.0;
  return gtsv_factor(n, lower.data(), diag.data(), upper.data(), F);
}

// operators.py:269-295 coefficient expressions, folded as _filter_rhs_row
// (operators.py:298-302): hc[h][0] = a_0, hc[h][k] = 0.5 * a_k.
FilterCoef filter_coefs(double af) {
  FilterCoef c;
  std::memset(&c, 0, sizeof(c));
  double a[6][6] = {};
  a[1][0] = 0.5 + af;
  a[1][1] = 0.5 + af;
  a[2][0] = (5.0 + 6.0 * af) / 8.0;
  a[2][1] = (1.0 + 2.0 * af) / 2.0;
  a[2][2] = (-1.0 + 2.0 * af) / 8.0;
  a[3][0] = (11.0 + 10.0 * af) / 16.0;
  a[3][1] = (15.0 + 34.0 * af) / 32.0;
  a[3][2] = (-3.0 + 6.0 * af) / 16.0;
  a[3][3] = (1.0 - 2.0 * af) / 32.0;
  a[4][0] = (93.0 + 70.0 * af) / 128.0;
  a[4][1] = (7.0 + 18.0 * af) / 16.0;
  a[4][2] = (-7.0 + 14.0 * af) / 32.0;
  a[4][3] = (1.0 - 2.0 * af) / 16.0;
  a[4][4] = (-1.0 + 2.0 * af) / 128.0;
  a[5][0] = (193.0 + 126.0 * af) / 256.0;
  a[5][1] = (105.0 + 302.0 * af) / 256.0;
  a[5][2] = (-15.0 + 30.0 * af) / 64.0;
  a[5][3] = (45.0 - 90.0 * af) / 512.0;
  a[5][4] = (-5.0 + 10.0 * af) / 256.0;
  a[5][5] = (1.0 - 2.0 * af) / 512.0;
  for (int h = 1; h <= 5; ++h) {
    c.hc[h * 6] = a[h][0];
    for (int k = 1; k <= h; ++k) c.hc[h * 6 + k] = 0.5 * a[h][k];
  }
  return c;
}

// Device image of a HostFactor: 7 arrays of n doubles.
size_t factor_doubles(int n) { return (size_t)8 * std::max(n, 1); }

TriDev factor_view(const HostFactor& F, double* dev) {
  const size_t n = std::max(F.n, 1);
  TriDev T;
  T.n = F.n;
  T.cyclic = F.cyclic;
  T.fact = dev;
  T.d = dev + n;
  T.du = dev + 2 * n;
  T.du2 = dev + 3 * n;
  T.swap = dev + 4 * n;
  T.z = dev + 5 * n;
  T.rinv = dev + 6 * n;
  T.h = dev + 7 * n;
  T.vn = F.vn;
  T.denom = F.denom;
  return T;
}

void factor_pack(const HostFactor& F, std::vector<double>& out) {
  const size_t n = std::max(F.n, 1);
  out.assign(factor_doubles(F.n), 0.0);
  auto put = [&](int slot, const std::vector<double>& v) {
    std::copy(v.begin(), v.begin() + std::min(v.size(), n), out.begin() + slot * n);
  };
  put(0, F.fact);
  put(1, F.d);
  put(2, F.du);
  put(3, F.du2);
  put(4, F.swap);
  put(5, F.z);
  std::vector<double> rinv(n, 0.0);
  for (size_t i = 0; i < (size_t)F.n && i < F.d.size(); ++i) rinv[i] = 1.0 / F.d[i];
  put(6, rinv);
  put(7, F.h);
}

// Scan form of a swap-free factor for the fast filter (wd_filter_scan.cuh):
// y_r = rhs_r - fm_r y_{r-1}, x_r = y_r rinv_r - g_r x_{r+1}; per segment of
// m rows P_r = prod_{k=r0..r} (-fm_k), Q_r = prod_{k=r..r1-1} (-g_k).
int scan_pack(const HostFactor& F, std::vector<double>& out, int& m, int nseg = FS_S) {
  const int n = F.n;
  if (n < 12 || n > nseg * FS_M) return 0;
  for (int i = 0; i < n; ++i)
    if (F.swap[i] != 0.0) return 0;
  m = (n + nseg - 1) / nseg;
  // device layout: (fm, h)[n], (P, g)[n], (Q, z)[n] as double2, rinv[n]
  std::vector<double> fm(n), P(n), ri(n), g(n), Q(n), z(n, 0.0), h(n, 0.0);
  for (int r = 0; r < n; ++r) {
    fm[r] = r > 0 ? F.fact[r - 1] : 0.0;
    ri[r] = 1.0 / F.d[r];
    g[r] = r < n - 1 ? F.du[r] * ri[r] : 0.0;
    if (F.cyclic) {
      z[r] = F.z[r];
      h[r] = F.h[r];
    }
  }
  for (int r0 = 0; r0 < n; r0 += m) {
    const int r1 = std::min(n, r0 + m);
    P[r0] = -fm[r0];
    for (int r = r0 + 1; r < r1; ++r) P[r] = -fm[r] * P[r - 1];
    Q[r1 - 1] = -g[r1 - 1];
    for (int r = r1 - 2; r >= r0; --r) Q[r] = -g[r] * Q[r + 1];
  }
  out.assign((size_t)7 * n, 0.0);
  for (int r = 0; r < n; ++r) {
    out[2 * r] = fm[r];
    out[2 * r + 1] = h[r];
    out[2 * n + 2 * r] = P[r];
    out[2 * n + 2 * r + 1] = g[r];
    out[4 * n + 2 * r] = Q[r];
    out[4 * n + 2 * r + 1] = z[r];
    out[6 * n + r] = ri[r];
  }
  return 1;
}

Geom make_geom(int ndim, const int* dims, const int* face, const uint8_t* mask) {
  Geom g;
  std::memset(&g, 0, sizeof(g));
  g.nd = ndim;
  for (int a = 0; a < kMaxDim; ++a) g.n[a] = a < ndim ? dims[a] : 1;
  g.s[2] = 1;
  g.s[1] = g.n[2];
  g.s[0] = (long long)g.n[1] * g.n[2];
  g.N = (long long)g.n[0] * g.n[1] * g.n[2];
  for (int a = 0; a < kMaxDim; ++a) {
    g.fs[a] = fdiv_make((unsigned long long)std::max(g.s[a], 1LL));
    g.fn[a] = fdiv_make((unsigned long long)std::max(g.n[a], 1));
  }
  for (int f = 0; f < 2 * kMaxDim; ++f) g.face[f] = face ? face[f] : WD_FACE_NONE;
  for (int a = 0; a < kMaxDim; ++a)
    g.per[a] = a < ndim && face && face[2 * a] == WD_FACE_PERIODIC ? 1 : 0;
  g.mask = mask;
  return g;
}

}  // namespace

// ====================================================================== ctx

// Field workspaces are recycled across contexts: a cudaMalloc / cudaFree of
// the 7.5 GB workspace of a 512^3 solve took 2-170 ms (measured per call),
// which made one-shot solve_steady() times vary by up to ~2x.  Freed blocks
// of an exact size are kept (at most kWsCacheMax of them, LIFO) and handed
// to the next context that asks for that size; WD_NO_WS_CACHE disables it.
namespace {
constexpr size_t kWsCacheMax = 2;
std::mutex g_ws_mu;
struct WsBlock {
  int device;
  size_t bytes;
  void* ptr;
};
std::vector<WsBlock> g_ws_cache;  // keyed on (device, size): a block never crosses devices
int ws_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
cudaError_t ws_alloc(void** p, size_t bytes) {
  {
    const int dev = ws_device();
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (size_t i = g_ws_cache.size(); i-- > 0;)
      if (g_ws_cache[i].bytes == bytes && g_ws_cache[i].device == dev) {
        *p = g_ws_cache[i].ptr;
        g_ws_cache.erase(g_ws_cache.begin() + i);
        return cudaSuccess;
      }
  }
  return cudaMalloc(p, bytes);
}
void ws_free(void* p, size_t bytes) {
  if (!p) return;
  static const bool off = getenv("WD_NO_WS_CACHE") != nullptr;
  if (!off) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    if (g_ws_cache.size() < kWsCacheMax) {
      g_ws_cache.push_back(WsBlock{ws_device(), bytes, p});
      return;
    }
  }
  cudaFree(p);
}
}  // namespace

struct wd_dist;

struct wd_ctx {
  wd_dist* dist = nullptr;  // GENERIC slab-decomposed program (wd_dist.cuh): axis-0 hooks
  int concurrent = -1;      // independent line passes in one launch: -1 undecided, 0 no, 1 yes
  bool nopool = true;       // parked for reuse only when fully built and unmodified
  int device = 0;
  std::string env_sig;      // A/B environment knobs the plan was built under
  wd_grid_desc gd;
  wd_solver_desc sd;
  Geom g;
  Metric M;
  // M[l, m] not identically zero (generic path; see k_metric_nonzero)
  unsigned char mterm[9] = {1, 1, 1, 1, 1, 1, 1, 1, 1};
  cudaStream_t stream = nullptr;
  // factors
  HostFactor hcomp[3], hfilt[3];
  TriDev comp[3], filt[3];
  ScanDev scan[3];
  ScanDev cscan[3];  // fast compact derivatives (wd_deriv_scan.cuh), per axis
  ScanDev lscan[3];  // fast filter, 2-D lines of 513..2048 rows (wd_filter_long.cuh)
  double* factor_dev = nullptr;
  FilterCoef fcoef;
  // per-node metric sums (curvilinear) or scalars (uniform)
  double* sums_dev = nullptr;  // sumS | cflms | sqrtS[d]
  double sumS_c = 0, cflms_c = 0, sqrtS_c[3] = {0, 0, 0};
  // workspace
  double* ws = nullptr;
  double* ws_generic = nullptr;  // lazily allocated (ensure_generic)
  double* mk_dev = nullptr;      // compact metric terms (k-invariant grids, fast arithmetic)
  Metric Mk;                     // view of mk_dev (m == nullptr: none)
  double *p, *k, *acc, *dt, *lap, *tmp, *tmp2, *gam, *phiY;
  double *advf = nullptr, *gmf = nullptr;  // generic: advection, |grad phi|
  double* uabsf = nullptr;                 // generic: sum |U_hat| for the time step
  double *dphi[3], *U[3], *Uh[3], *nrm[3], *B[3], *F[3], *Ue[3];
  Status* st = nullptr;
  Status* st_scratch = nullptr;
  double* hist_scratch = nullptr;
  int* flag_dev = nullptr;
  // binding
  double* phi = nullptr;
  double* hist = nullptr;
  std::map<std::pair<int, int>, cudaGraphExec_t> graphs;
  long long enq = 0;  // host-side count of enqueued steps (buffer parity)
  FusedPlan fused;    // specialised kernels (wd_fused.cuh), if applicable
  // wd_fused_filter: filter factors for arbitrary (length, periodic)
  std::map<std::pair<int, int>, std::pair<HostFactor, double*>> dfilt;
};

namespace {

double lref(const wd_ctx* c) { return c->gd.ref_length; }

// axis-0 operators of a slab-decomposed context run on pencils (wd_dist.cuh)
void dist_deriv0(wd_ctx* c, const double* in, double* out, int scheme, const Epi& e,
                 const Status* st);
void dist_uw0(wd_ctx* c, const double* p, double* B, double* F, double* dphi, const Status* st);
void dist_d40(wd_ctx* c, const double* p, double* out, const Epi& e, const Status* st);
void dist_filter0_generic(wd_ctx* c, const double* cur, double* nxt, const Status* st);
void dist_reduce_status(wd_ctx* c);

Epi epi_plain() { return Epi{0, nullptr, nullptr, 0.0}; }

// coefficient M[l, m] as an epilogue source
Epi epi_metric(const wd_ctx* c, int l, int m, bool first, double* acc) {
  Epi e;
  e.mode = first ? 1 : 2;
  e.acc = acc;
  if (c->M.m) {
    e.cfield = c->M.m + (long long)(l * c->g.nd + m) * c->g.N;
    e.cscal = 0.0;
    if (c->Mk.m) {
      e.ccomp = c->Mk.m + (long long)(l * c->g.nd + m) * c->Mk.N;
      e.cdiv = c->Mk.kdiv;
    }
  } else {
    e.cfield = nullptr;
    e.cscal = l == m ? c->M.c[l] : 0.0;
  }
  return e;
}

// D_axis(in) with `scheme` (central) -> out via epilogue.  scratch is
// needed for compact schemes when the epilogue is not plain.
// generic line solves: parallel right-hand sides + warp-per-32-lines
// dgtsv recurrences (wd_line_sweep.cuh).  `scratch` holds rhs / y and must
// not alias `in`; it may equal `out` when the output does not read `out`.
bool line_solve_ok(int n) { return n >= 3 && line_solve_smem(n) <= kLineSolveMaxSmem; }
void line_solve_prepare() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(k_line_solve<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kLineSolveMaxSmem);
  cudaFuncSetAttribute(k_line_solve<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kLineSolveMaxSmem);
  cudaFuncSetAttribute(k_line_solve_t<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kLineSolveMaxSmem);
  cudaFuncSetAttribute(k_line_solve_t<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kLineSolveMaxSmem);
  cudaFuncSetAttribute(k_line_few<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kLineSolveMaxSmem);
  cudaFuncSetAttribute(k_line_few<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kLineSolveMaxSmem);
  done = true;
}
template <int JOB>
void launch_line_solve(const double* in, double* scratch, double* out, const Geom& g, int axis,
                       int per, double off, int scheme, const TriDev& T, const Epi& e,
                       const FilterCoef& fc, const uint8_t* pin, int use_geom_pin,
                       const Status* st, cudaStream_t s) {
  const int n = g.n[axis];
  const long long L = g.N / n;
  // few long lines (2-D grids): one chain thread per line out of shared
  // memory, right-hand side and epilogue in the same launch
  if (L <= 148LL * 2 * LF_MAXL && !getenv("WD_NO_LINE_FEW")) {
    int fl = (int)((L + 147) / 148);
    if (fl > LF_MAXL) fl = LF_MAXL;
    if (fl < 1) fl = 1;
    const size_t sm = line_few_smem(n, fl);
    if (sm <= kLineSolveMaxSmem) {
      const int blocks = (int)((L + fl - 1) / fl);
      launch_pdl(k_line_few<JOB>, dim3(blocks), dim3(LF_T), sm, s, in, out, g, axis, n, g.s[axis],
                 per, off, scheme, T, e, fc, pin, use_geom_pin, fl, st);
      return;
    }
  }
  if (g.s[axis] >= 32 && !getenv("WD_NO_RHS_SEG")) {
    const long long segs = L * ((n + RS_ROWS - 1) / RS_ROWS);
    k_line_rhs_seg<JOB><<<nblocks(segs, kThreads), kThreads, 0, s>>>(
        in, scratch, g.N, g.s[axis], n, per, off, scheme, fc, st);
  } else {
    k_line_rhs<JOB><<<nblocks(g.N, kThreads), kThreads, 0, s>>>(in, scratch, axis_geom(g, axis),
                                                                  per, off, scheme, fc, st);
  }
  const long long warps = (L + 31) / 32;
  const int blocks = (int)std::min<long long>((warps + LS_WARPS - 1) / LS_WARPS, 148LL * 8);
  // contiguous lines: transposed cp.async staging (coalesced); long strided
  // lines when there are too few of them to fill the GPU (C3's axis-0
  // filter: 513 lines of 1025, the chain runs from shared memory with the
  // next chunk in flight: 1.12 -> 1.04 ms per step; short lines (C2) lose)
  const bool few = warps < 148LL * 2 * LS_WARPS && n >= 512;
  if (line_solve_t_smem(n) <= kLineSolveMaxSmem &&
      ((g.s[axis] == 1 && axis == g.nd - 1) || (few && !getenv("WD_NO_TILED_FEW")))) {
    k_line_solve_t<JOB><<<blocks, LS_WARPS * 32, line_solve_t_smem(n), s>>>(
        in, scratch, out, g, axis, n, g.s[axis], T, e, pin, use_geom_pin, st);
    return;
  }
  k_line_solve<JOB><<<blocks, LS_WARPS * 32, line_solve_smem(n), s>>>(
      in, scratch, out, g, axis, n, g.s[axis], T, e, pin, use_geom_pin, st);
}

void launch_deriv(wd_ctx* c, const double* in, double* out, double* scratch, int axis, int scheme,
                  Epi e, const Status* st) {
  const Geom& g = c->g;
  if (c->dist && axis == 0) {
    dist_deriv0(c, in, out, scheme, e, st);
    return;
  }
  if ((scheme == WD_C4 || scheme == WD_C6) && c->cscan[axis].tab && scheme == c->sd.scheme) {
    // arith="fast": segmented-scan solve, epilogue fused (wd_deriv_scan.cuh)
    DScanArgs a;
    a.in = in;
    a.out = out;
    a.N = g.N;
    a.sa = g.s[axis];
    a.per = g.per[axis];
    a.scheme = scheme;
    a.T = c->cscan[axis];
    a.epi = e;
    a.st = st;
    const int n = g.n[axis];
    const long long lines = g.N / n;
    const DScanShape sh = dscan_shape(n, a.sa == 1);
    const long long groups = a.sa == 1 ? (lines + sh.NL - 1) / sh.NL
                                       : (g.N / (n * a.sa)) * ((a.sa + sh.NL - 1) / sh.NL);
    const int blocks = (int)std::min<long long>(groups, 148LL * (sh.TT == 256 ? 2 : 1));
    const DScanFn fn = dscan_kernel(n, a.sa == 1, a.per != 0, scheme == WD_C6);
    fn<<<blocks, sh.TT, dscan_smem(n, sh), c->stream>>>(a);
    return;
  }
  if (scheme == WD_C4 || scheme == WD_C6) {
    const long long L = g.N / g.n[axis];
    double* ys = (e.mode == 0 && out != in) ? out : scratch;
    if (line_solve_ok(g.n[axis]) && ys != in) {
      launch_line_solve<0>(in, ys, out, g, axis, g.per[axis], 0.0, scheme, c->comp[axis], e,
                           c->fcoef, nullptr, 0, st, c->stream);
      return;
    }
    double* scr = (e.mode == 0) ? out : scratch;
    k_deriv_compact<<<nblocks(L, kLineThreads), kLineThreads, 0, c->stream>>>(
        in, scr, out, g, axis, scheme, g.per[axis], 0.0, c->comp[axis], e, st);
  } else {
    k_deriv_explicit<<<nblocks(g.N, kThreads), kThreads, 0, c->stream>>>(
        in, out, axis_geom(g, axis), scheme, g.per[axis], 0.0, e, st);
  }
}

// Grids with few long lines (2-D configs, exact arithmetic): every compact
// pass is one dependency chain per line, ~25-100 us regardless of how little
// data it moves, and a tendency runs 10 of them back to back.  The passes of
// one phase are independent (the gradient's axes; the divergence's terms,
// which only meet in their sum), so they go into ONE launch
// (k_line_few_multi, blockIdx.y = pass) and the divergence terms are summed
// afterwards in the reference's order (k_div_combine): bit-identical to the
// serial chain.  (Forked streams -- parallel graph branches -- were measured
// 2x SLOWER than the serial launches: C2 1.23 -> 2.58 ms per step.)
bool concurrent_passes(wd_ctx* c) {
  if (c->concurrent >= 0) return c->concurrent != 0;
  c->concurrent = 0;
  const Geom& g = c->g;
  const int sc = c->sd.scheme;
  if ((sc != WD_C4 && sc != WD_C6) || c->dist || getenv("WD_NO_CONCURRENT")) return false;
  if (c->sd.arith == 1) return false;  // fast arithmetic: the scan kernels
  for (int a = 0; a < g.nd; ++a) {
    const long long L = g.N / g.n[a];
    if (!(L <= 148LL * 2 * LF_MAXL && line_solve_ok(g.n[a]) &&
          line_few_smem(g.n[a], LF_MAXL) <= kLineSolveMaxSmem))
      return false;
  }
  cudaFuncSetAttribute(k_line_few_multi, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kLineSolveMaxSmem);
  c->concurrent = 1;
  return true;
}

// up to 4 compact-derivative passes (plain epilogue) per launch
void launch_line_multi(wd_ctx* c, int count, const double* const* in, double* const* out,
                       const int* axis, const Status* st) {
  const Geom& g = c->g;
  for (int q0 = 0; q0 < count; q0 += 4) {
    LineFewJobs jobs;
    std::memset(&jobs, 0, sizeof(jobs));
    jobs.count = std::min(4, count - q0);
    long long lmax = 0;
    int nmax = 0;
    for (int q = 0; q < jobs.count; ++q) {
      const int a = axis[q0 + q];
      jobs.in[q] = in[q0 + q];
      jobs.out[q] = out[q0 + q];
      jobs.axis[q] = a;
      jobs.T[q] = c->comp[a];
      lmax = std::max(lmax, g.N / g.n[a]);
      nmax = std::max(nmax, g.n[a]);
    }
    int fl = (int)((lmax + 147) / 148);
    fl = std::max(1, std::min(fl, LF_MAXL));
    const dim3 grid((unsigned)((lmax + fl - 1) / fl), (unsigned)jobs.count);
    k_line_few_multi<<<grid, LF_T, line_few_smem(nmax, fl), c->stream>>>(jobs, g, c->sd.scheme,
                                                                        fl, st);
  }
}

// lap / kappa = sum_m sum_l M[l,m] D_l(V_m)  (formulations.py:135-143)
void launch_divergence(wd_ctx* c, double* const V[3], int csch, double* out, const Status* st) {
  const int nd = c->g.nd;
  if (csch == c->sd.scheme && concurrent_passes(c)) {
    DivTerms t;
    std::memset(&t, 0, sizeof(t));
    double* pool[9] = {c->B[0], c->B[1], c->B[2], c->F[0], c->F[1], c->F[2],
                       c->Ue[0], c->Ue[1], c->Ue[2]};  // UW-only fields: free here
    const double* src[9];
    for (int m = 0; m < nd; ++m)
      for (int l = 0; l < nd; ++l) {
        if (c->M.m == nullptr ? l != m : !c->mterm[l * nd + m]) continue;
        t.D[t.count] = pool[t.count];
        src[t.count] = V[m];
        t.l[t.count] = l;
        t.m[t.count] = m;
        ++t.count;
      }
    launch_line_multi(c, t.count, src, pool, t.l, st);
    const int nb = nblocks(c->g.N, kThreads);
    if (nd == 3) k_div_combine<3><<<nb, kThreads, 0, c->stream>>>(t, c->M, out, c->g.N, st);
    else k_div_combine<2><<<nb, kThreads, 0, c->stream>>>(t, c->M, out, c->g.N, st);
    return;
  }
  bool first = true;
  for (int m = 0; m < nd; ++m)
    for (int l = 0; l < nd; ++l) {
      if (c->M.m == nullptr ? l != m : !c->mterm[l * nd + m]) continue;  // exact zero terms
      launch_deriv(c, V[m], out, c->tmp, l, csch, epi_metric(c, l, m, first, out), st);
      first = false;
    }
}

void launch_assemble(wd_ctx* c, double* const d[3], double* const U[3], double* const Uh[3],
                     const Status* st, bool extras = false, bool uabs = false) {
  AsmExtra x;
  std::memset(&x, 0, sizeof(x));
  if (uabs) x.uabs = c->uabsf;
  if (extras) {  // central schemes: advection, |grad phi|, curvature normal
    x.adv = c->advf;
    if (c->sd.kind == WD_HJ_CURVATURE) {
      x.gm = c->gmf;
      for (int a = 0; a < 3; ++a) x.nrm.p[a] = c->nrm[a];
      x.eps0 = c->sd.eps0;
    }
  }
  Vec3 dv;
  MVec3 Uv, Uhv;
  for (int a = 0; a < 3; ++a) {
    dv.p[a] = d[a];
    Uv.p[a] = U[a];
    Uhv.p[a] = Uh ? Uh[a] : nullptr;
  }
  unsigned nzm = 0;
  for (int t = 0; t < c->g.nd * c->g.nd; ++t)
    if (c->M.m == nullptr || c->mterm[t]) nzm |= 1u << t;
  // the full metric fields even when a compact copy exists (c->Mk): measured
  // at 1024 x 512 x 256, this kernel runs 2.68 ms with the 16-byte loads of the
  // full terms and 3.81 ms with the broadcast loads of the compact ones
  // ... except the U-only instantiation (Poisson): at three times the
  // resident warps it gains from the five reads it drops, 1.70 -> 1.33 ms
  const bool uonly = Uhv.p[0] == nullptr && !x.adv && !x.uabs && !x.gm &&
                     !getenv("WD_NO_ASM_UONLY");
  const Metric& Mu = (c->Mk.m && (uonly || getenv("WD_ASM_COMPACT"))) ? c->Mk : c->M;
  const long long N = c->g.N;
  // two nodes per thread when the pairs are 16-byte aligned and, for compact
  // terms, never straddle two lines of the last axis
  uintptr_t al = (uintptr_t)Mu.m | (uintptr_t)x.adv | (uintptr_t)x.gm | (uintptr_t)x.uabs;
  for (int a = 0; a < c->g.nd; ++a)
    al |= (uintptr_t)dv.p[a] | (uintptr_t)Uv.p[a] | (uintptr_t)Uhv.p[a] | (uintptr_t)x.nrm.p[a];
  if (N % 2 == 0 && (al & 15) == 0 && (Mu.kdiv <= 1 || Mu.kdiv % 2 == 0) &&
      !getenv("WD_NO_ASM2")) {
    const int nb = nblocks(N / 2, 256);
    if (uonly && c->g.nd == 3) {
      if (nzm == 0x1FFu)
        k_assemble2<3, 0x1FFu, true><<<nb, 256, 0, c->stream>>>(dv, Mu, Uv, Uhv, N, nzm, x, st);
      else if (nzm == 0x11Bu)
        k_assemble2<3, 0x11Bu, true><<<nb, 256, 0, c->stream>>>(dv, Mu, Uv, Uhv, N, nzm, x, st);
      else
        k_assemble2<3, 0u, true><<<nb, 256, 0, c->stream>>>(dv, Mu, Uv, Uhv, N, nzm, x, st);
      return;
    }
    if (c->g.nd == 3) {
      if (nzm == 0x1FFu)
        k_assemble2<3, 0x1FFu><<<nb, 256, 0, c->stream>>>(dv, Mu, Uv, Uhv, N, nzm, x, st);
      else if (nzm == 0x11Bu)  // extruded grids: the four cross terms with the last axis vanish
        k_assemble2<3, 0x11Bu><<<nb, 256, 0, c->stream>>>(dv, Mu, Uv, Uhv, N, nzm, x, st);
      else
        k_assemble2<3, 0u><<<nb, 256, 0, c->stream>>>(dv, Mu, Uv, Uhv, N, nzm, x, st);
    } else {
      if (nzm == 0xFu) k_assemble2<2, 0xFu><<<nb, 256, 0, c->stream>>>(dv, Mu, Uv, Uhv, N, nzm, x, st);
      else k_assemble2<2, 0u><<<nb, 256, 0, c->stream>>>(dv, Mu, Uv, Uhv, N, nzm, x, st);
    }
    return;
  }
  if (c->g.nd == 3)
    k_assemble<3><<<nblocks(N, kThreads), kThreads, 0, c->stream>>>(dv, Mu, Uv, Uhv, N, 3, nzm, x, st);
  else
    k_assemble<2><<<nblocks(N, kThreads), kThreads, 0, c->stream>>>(dv, c->M, Uv, Uhv, N, 2, nzm, x, st);
}

// directional derivatives of p with the run's scheme -> dphi (+B, F for UW)
void launch_dphi(wd_ctx* c, const double* p, const Status* st) {
  if (c->sd.scheme != WD_UW && concurrent_passes(c)) {
    const double* in3[3] = {p, p, p};
    const int ax3[3] = {0, 1, 2};
    launch_line_multi(c, c->g.nd, in3, c->dphi, ax3, st);
    return;
  }
  for (int l = 0; l < c->g.nd; ++l) {
    if (c->sd.scheme == WD_UW && c->dist && l == 0)
      dist_uw0(c, p, c->B[l], c->F[l], c->dphi[l], st);
    else if (c->sd.scheme == WD_UW)
      k_uw_bf<<<nblocks(c->g.N, kThreads), kThreads, 0, c->stream>>>(p, c->B[l], c->F[l],
                                                                      c->dphi[l],
                                                                      axis_geom(c->g, l),
                                                                      c->g.per[l], st);
    else
      launch_deriv(c, p, c->dphi[l], c->tmp, l, c->sd.scheme, epi_plain(), st);
  }
}

void launch_gamma_lad(wd_ctx* c, const double* p, const Status* st) {
  const Geom& g = c->g;
  for (int l = 0; l < g.nd; ++l) {
    Epi e;
    e.mode = l == 0 ? 1 : 2;
    e.acc = c->tmp2;
    e.cfield = c->sums_dev ? c->sums_dev + (2 + l) * g.N : nullptr;
    e.cscal = c->sqrtS_c[l];
    if (c->dist && l == 0) {
      dist_d40(c, p, c->tmp2, e, st);
      continue;
    }
    k_d4<<<nblocks(g.N, kThreads), kThreads, 0, c->stream>>>(p, c->tmp2, axis_geom(g, l), g.per[l], e, st);
  }
  k_gamma_lad<<<nblocks(g.N, kThreads), kThreads, 0, c->stream>>>(p, c->tmp2, c->gam, g.N,
                                                                   c->sd.epsilon, c->sd.lad_c, st);
}

// tendency(p) -> k   (formulations.py:232-252).  `fresh`: dphi / U / Uh
// (and gamma for LAD) already hold the values for this p -- the time step of
// the same pseudo-iteration computed them from the same field with the same
// kernels, so recomputing would reproduce them bit for bit.
void enqueue_tendency(wd_ctx* c, const double* p, double* k, const Status* st,
                      bool fresh = false, ResidualArgs* defer = nullptr) {
  const int kind = c->sd.kind, scheme = c->sd.scheme, nd = c->g.nd;
  const int csch = scheme == WD_UW ? WD_E2 : scheme;
  ResidualArgs a;
  std::memset(&a, 0, sizeof(a));
  a.kind = kind;
  a.scheme = scheme;
  a.nd = nd;
  a.eps = c->sd.epsilon;
  a.p = p;
  a.lap = c->lap;
  a.gam = c->gam;
  a.kappa = c->tmp2;
  for (int l = 0; l < 3; ++l) {
    a.U.p[l] = c->U[l];
    a.Uh.p[l] = c->Uh[l];
    a.dphi.p[l] = c->dphi[l];
    a.B.p[l] = c->B[l];
    a.F.p[l] = c->F[l];
  }
  if (kind == WD_POISSON) {
    for (int l = 0; l < nd; ++l) launch_deriv(c, p, c->dphi[l], c->tmp, l, csch, epi_plain(), st);
    launch_assemble(c, c->dphi, c->U, nullptr, st);
    launch_divergence(c, c->U, csch, c->lap, st);
  } else {
    // central schemes: the assemble kernel also leaves adv, |grad phi| and
    // the curvature normal (bit-identical, k_assemble); UW keeps its own
    const bool ext = scheme != WD_UW && !getenv("WD_NO_ASM_EXTRA");
    if (!fresh) {
      launch_dphi(c, p, st);
      // with the extras nothing downstream reads U_hat: not written
      launch_assemble(c, c->dphi, c->U, ext ? nullptr : c->Uh, st, ext);
    }
    if (ext) {
      a.adv = c->advf;
      if (kind == WD_HJ_CURVATURE) a.gm = c->gmf;
    }
    if (kind != WD_EIKONAL) {
      double* const* Ul = c->U;
      if (scheme == WD_UW) {
        for (int l = 0; l < nd; ++l)
          launch_deriv(c, p, c->nrm[l], c->tmp, l, WD_E2, epi_plain(), st);
        launch_assemble(c, c->nrm, c->Ue, nullptr, st);
        Ul = c->Ue;
        for (int l = 0; l < 3; ++l) a.U.p[l] = c->Ue[l];
      }
      launch_divergence(c, Ul, csch, c->lap, st);
      if (kind == WD_HJ_LAD && !fresh) launch_gamma_lad(c, p, st);
      if (kind == WD_HJ_CURVATURE) {
        Vec3 uv;
        MVec3 nv;
        for (int l = 0; l < 3; ++l) {
          uv.p[l] = Ul[l];
          nv.p[l] = c->nrm[l];
        }
        if (!ext)
          k_normal<<<nblocks(c->g.N, kThreads), kThreads, 0, c->stream>>>(uv, nv, c->g.N, nd,
                                                                           c->sd.eps0, st);
        launch_divergence(c, c->nrm, csch, c->tmp2, st);
      }
    }
  }
  if (defer) {  // the caller fuses the residual into its own kernel (k_tend_rk)
    *defer = a;
    return;
  }
  k_tendency<<<nblocks(c->g.N, kThreads), kThreads, 0, c->stream>>>(a, k, c->g.N, st);
}

// local_timestep(p) -> dt   (solver.py:160-180)
void enqueue_timestep(wd_ctx* c, const double* p, double* dt, const Status* st) {
  DtArgs a;
  std::memset(&a, 0, sizeof(a));
  a.kind = c->sd.kind;
  a.nd = c->g.nd;
  a.eps = c->sd.epsilon;
  a.cfl = c->sd.cfl;
  a.p = p;
  a.gam = c->gam;
  for (int l = 0; l < 3; ++l) a.Uh.p[l] = c->Uh[l];
  a.sumS = c->sums_dev;
  a.sumS_c = c->sumS_c;
  a.cflms = c->sums_dev ? c->sums_dev + c->g.N : nullptr;
  a.cflms_c = c->cflms_c;
  if (c->sd.kind != WD_POISSON) {
    launch_dphi(c, p, st);
    // extras for the stage-1 tendency of the same iteration (fresh)
    const bool ext = c->sd.scheme != WD_UW && !getenv("WD_NO_ASM_EXTRA");
    launch_assemble(c, c->dphi, c->U, ext ? nullptr : c->Uh, st, ext, ext);
    if (ext) a.uabs = c->uabsf;
    if (c->sd.kind == WD_HJ_LAD) launch_gamma_lad(c, p, st);
  }
  k_timestep<<<nblocks(c->g.N, kThreads), kThreads, 0, c->stream>>>(a, dt, c->g.N, st);
}

// filter all axes + BC: x (BC'd RK4 output, clobbered) -> out
// (solver.py:208-212)
void enqueue_filter_bc(wd_ctx* c, double* x, double* out, const Status* st,
                       const double* change_vs = nullptr) {
  const Geom& g = c->g;
  double* cur = x;
  double* bufs[2] = {c->tmp2, x};
  for (int a = 0; a < g.nd; ++a) {
    double* nxt = bufs[a & 1];
    const long long L = g.N / g.n[a];
    if (c->dist && a == 0) {
      dist_filter0_generic(c, cur, nxt, st);
      cur = nxt;
      continue;
    }
    // arith="fast", no solid mask, lines of 12..512 rows: the segmented-scan sweep
    // (wd_filter_scan.cuh).  It does not restore pinned nodes, which is
    // exact here: the input is BC'd (walls are 0), a wall of this axis is a
    // line end (identity row) and a wall of another axis holds whole lines
    // of zeros, which the linear sweep maps to zeros.
    if (st && c->sd.arith == 1 && g.mask == nullptr && c->scan[a].tab &&
        !getenv("WD_NO_GEN_SCANF")) {
      FusedPlan fp;
      fp.in.fcoef = c->fcoef;
      if (g.nd == 3)
        fused_filter_any(fp, a, cur, nxt, g.n[0], g.n[1], g.n[2], g.per[a], c->filt[a], nullptr,
                         const_cast<Status*>(st), c->stream, &c->scan[a]);
      else  // 2-D (n0, n1) swept as the (1, n0, n1) array: axes 0, 1 -> 1, 2
        fused_filter_any(fp, a + 1, cur, nxt, 1, g.n[0], g.n[1], g.per[a], c->filt[a], nullptr,
                         const_cast<Status*>(st), c->stream, &c->scan[a]);
      cur = nxt;
      continue;
    }
    // the same for the few long lines of a 2-D grid (wd_filter_long.cuh)
    if (st && c->sd.arith == 1 && g.mask == nullptr && g.nd == 2 && c->lscan[a].tab &&
        !getenv("WD_NO_GEN_SCANF")) {
      LongScanArgs la;
      la.in = cur;
      la.out = nxt;
      la.L = L;
      la.rstride = g.s[a];
      la.lstride = g.s[1 - a];
      la.per = g.per[a];
      la.T = c->lscan[a];
      la.fc = c->fcoef;
      la.st = st;
      launch_filter_long(la, c->stream);
      cur = nxt;
      continue;
    }
    if (line_solve_ok(g.n[a])) {
      launch_line_solve<1>(cur, nxt, nxt, g, a, g.per[a], 0.0, 0, c->filt[a], epi_plain(),
                           c->fcoef, nullptr, 1, st, c->stream);
    } else {
      k_filter<<<nblocks(L, kLineThreads), kLineThreads, 0, c->stream>>>(
          cur, nxt, g, a, g.per[a], c->fcoef, c->filt[a], nullptr, 1, st);
    }
    cur = nxt;
  }
  if (change_vs)  // the step's convergence reduction rides on the BC pass
    launch_pdl(k_bc_change, dim3(nblocks(g.N, kThreads)), dim3(kThreads), 0, c->stream, cur, out,
               change_vs, g, const_cast<Status*>(st));
  else
    k_bc<<<nblocks(g.N, kThreads), kThreads, 0, c->stream>>>(cur, out, g, st);
}

void rk_stage(int nd, int nb, cudaStream_t s, int stage, const double* phi, const double* dt,
              const double* k, double* acc, double* out, const Geom& g, const Status* st) {
  if (nd == 3) k_rk_stage<3><<<nb, kThreads, 0, s>>>(stage, phi, dt, k, acc, out, g, st);
  else k_rk_stage<2><<<nb, kThreads, 0, s>>>(stage, phi, dt, k, acc, out, g, st);
}

// one RK4 step A -> B given dt already in c->dt (solver.py:183-212)
void enqueue_rk4(wd_ctx* c, const double* A, double* B, const Status* st,
                 bool dt_fresh = false, bool fuse_change = false) {
  const Geom& g = c->g;
  const int nb = nblocks(g.N, kThreads);
  // stage 1 evaluates the tendency at A, where enqueue_timestep just left
  // dphi / U / Uh (/ gamma) -- except for Poisson, whose time step is static.
  // The residual itself is evaluated inside the stage update (k_tend_rk).
  // Stage fields ping-pong p -> k -> p -> k: the update reads the stage input
  // (eps phi in the residual) at its source node, so it cannot be in place.
  auto stage = [&](int sidx, const double* pin, double* outp, bool fresh) {
    ResidualArgs ra;
    enqueue_tendency(c, pin, nullptr, st, fresh, &ra);
    if (c->g.nd == 3)
      k_tend_rk<3><<<nb, kThreads, 0, c->stream>>>(sidx, ra, A, c->dt, c->acc, outp, g, st);
    else
      k_tend_rk<2><<<nb, kThreads, 0, c->stream>>>(sidx, ra, A, c->dt, c->acc, outp, g, st);
  };
  stage(1, A, c->p, dt_fresh && c->sd.kind != WD_POISSON);
  stage(2, c->p, c->k, false);
  stage(3, c->k, c->p, false);
  if (c->sd.use_filter) {
    stage(4, c->p, c->k, false);
    enqueue_filter_bc(c, c->k, B, st, fuse_change ? A : nullptr);
  } else {
    stage(4, c->p, B, false);
  }
}

// Generic-path workspace (27 fields), allocated the first time a generic
// kernel sequence is enqueued; the fused path never needs it.
int ensure_generic(wd_ctx* c) {
  if (c->ws_generic) return WD_OK;
  const long long N = c->g.N;
  if (ws_alloc((void**)&c->ws_generic, (size_t)27 * N * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    return fail(WD_ERR_CUDA, "generic workspace allocation failed (" +
                                 std::to_string(27.0 * N * 8 / 1e9) + " GB)");
  }
  if (c->M.m && !getenv("WD_NO_ZERO_SKIP")) {
    const int nt = c->g.nd * c->g.nd;
    int* fl = nullptr;
    int hf[9] = {0};
    if (cudaMalloc(&fl, nt * sizeof(int)) != cudaSuccess) {
      cudaGetLastError();
      return fail(WD_ERR_CUDA, "metric flag allocation failed");
    }
    cudaMemsetAsync(fl, 0, nt * sizeof(int), c->stream);
    k_metric_nonzero<<<dim3(148 * 2, nt), kThreads, 0, c->stream>>>(c->M.m, c->g.N, fl);
    cudaMemcpyAsync(hf, fl, nt * sizeof(int), cudaMemcpyDeviceToHost, c->stream);
    const cudaError_t e = cudaStreamSynchronize(c->stream);
    cudaFree(fl);
    if (e != cudaSuccess) return fail(WD_ERR_CUDA, std::string("metric scan: ") + cudaGetErrorString(e));
    for (int t = 0; t < nt; ++t) c->mterm[t] = hf[t] != 0;
  }
  // fast arithmetic, 3-D: metric terms constant along the last axis are kept
  // once per (i, j) for the scan derivatives and the assemble kernel
  if (c->M.m && c->sd.arith == 1 && c->g.nd == 3 && c->g.n[2] > 1 && N <= 0xffffffffLL &&
      !c->mk_dev && !getenv("WD_NO_KMETRIC")) {
    const int nt = 9, n2 = c->g.n[2];
    int* fl = nullptr;
    int hv = 1;
    if (cudaMalloc(&fl, sizeof(int)) == cudaSuccess) {
      cudaMemsetAsync(fl, 0, sizeof(int), c->stream);
      k_metric_kvar<<<148 * 4, kThreads, 0, c->stream>>>(c->M.m, N, n2, nt, fl);
      cudaMemcpyAsync(&hv, fl, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
      if (cudaStreamSynchronize(c->stream) != cudaSuccess) hv = 1;
      cudaFree(fl);
    }
    cudaGetLastError();
    const long long Nk = N / n2;
    if (hv == 0 && cudaMalloc(&c->mk_dev, (size_t)nt * Nk * sizeof(double)) == cudaSuccess) {
      k_metric_kgather<<<nblocks(nt * Nk, kThreads), kThreads, 0, c->stream>>>(c->M.m, c->mk_dev,
                                                                              N, n2, nt);
      c->Mk = c->M;
      c->Mk.m = c->mk_dev;
      c->Mk.N = Nk;
      c->Mk.kdiv = n2;
    }
    cudaGetLastError();
  }
  double* w = c->ws_generic;
  auto take = [&]() {
    double* r = w;
    w += N;
    return r;
  };
  c->lap = take();
  c->gam = take();
  take();
  c->advf = take();
  c->gmf = take();
  c->uabsf = take();
  for (int a = 0; a < 3; ++a) {
    c->dphi[a] = take();
    c->U[a] = take();
    c->Uh[a] = take();
    c->nrm[a] = take();
    c->B[a] = take();
    c->F[a] = take();
    c->Ue[a] = take();
  }
  return WD_OK;
}

// 2-D explicit central schemes, Eikonal / HJ: two kernels per RK stage
// (wd_stage_explicit.cuh), bit-identical to the multi-kernel sequence below
bool explicit_stage_ok(const wd_ctx* c) {
  const int sc = c->sd.scheme;
  return c->g.nd == 2 && (sc == WD_E2 || sc == WD_E4 || sc == WD_E6) &&
         (c->sd.kind == WD_EIKONAL || c->sd.kind == WD_HJ) && !c->dist &&
         !getenv("WD_NO_STAGE_EXPLICIT");
}

void enqueue_step_explicit(wd_ctx* c, const double* A, double* B) {
  ExArgs a;
  std::memset(&a, 0, sizeof(a));
  a.A = A;
  a.dt = c->dt;
  a.acc = c->acc;
  a.g = c->g;
  a.M = c->M;
  for (int t = 0; t < c->g.nd * c->g.nd; ++t)
    if (c->M.m == nullptr || c->mterm[t]) a.nzm |= 1u << t;
  a.scheme = c->sd.scheme;
  a.kind = c->sd.kind;
  a.eps = c->sd.epsilon;
  a.cfl = c->sd.cfl;
  a.sumS = c->sums_dev;
  a.sumS_c = c->sumS_c;
  a.cflms = c->sums_dev ? c->sums_dev + c->g.N : nullptr;
  a.cflms_c = c->cflms_c;
  a.st = c->st;
  a.U[0] = c->U[0];
  a.U[1] = c->U[1];
  a.adv = c->advf;
  const int nb = nblocks(c->g.N, 256);
  double* last = c->sd.use_filter ? c->k : B;
  a.p = A;
  a.out = c->p;
  launch_pdl(k_ex_grad<2, true>, dim3(nb), dim3(256), 0, c->stream, a);
  launch_pdl(k_ex_update<2, 1>, dim3(nb), dim3(256), 0, c->stream, a);
  a.p = c->p;
  a.out = c->k;
  launch_pdl(k_ex_grad<2, false>, dim3(nb), dim3(256), 0, c->stream, a);
  launch_pdl(k_ex_update<2, 2>, dim3(nb), dim3(256), 0, c->stream, a);
  a.p = c->k;
  a.out = c->p;
  launch_pdl(k_ex_grad<2, false>, dim3(nb), dim3(256), 0, c->stream, a);
  launch_pdl(k_ex_update<2, 3>, dim3(nb), dim3(256), 0, c->stream, a);
  a.p = c->p;
  a.out = last;
  launch_pdl(k_ex_grad<2, false>, dim3(nb), dim3(256), 0, c->stream, a);
  launch_pdl(k_ex_update<2, 4>, dim3(nb), dim3(256), 0, c->stream, a);
  if (c->sd.use_filter)
    enqueue_filter_bc(c, c->k, B, c->st, A);
  else
    k_change<<<nblocks(c->g.N, kThreads), kThreads, 0, c->stream>>>(B, A, c->g.mask, c->st,
                                                                     c->g.N);
  launch_pdl(k_finalize, dim3(1), dim3(1), 0, c->stream, c->st, c->hist, lref(c), c->sd.tol,
             1e6 * lref(c));
}

void enqueue_step(wd_ctx* c, const double* A, double* B) {
  if (c->fused.active) {
    fused_step(c->fused, A, B, c->st, c->hist, c->stream);
    return;
  }
  if (explicit_stage_ok(c)) {
    enqueue_step_explicit(c, A, B);
    return;
  }
  enqueue_timestep(c, A, c->dt, c->st);
  // filtered steps end with a BC pass: the convergence reduction rides on it
  const bool fuse = c->sd.use_filter && !getenv("WD_NO_BC_CHANGE");
  enqueue_rk4(c, A, B, c->st, true, fuse);
  if (!fuse)
    k_change<<<nblocks(c->g.N, kThreads), kThreads, 0, c->stream>>>(B, A, c->g.mask, c->st,
                                                                     c->g.N);
  if (c->dist) dist_reduce_status(c);
  k_finalize<<<1, 1, 0, c->stream>>>(c->st, c->hist, lref(c), c->sd.tol, 1e6 * lref(c));
}

int validate(const wd_grid_desc* gd, const wd_solver_desc* sd) {
  if (gd->ndim != 2 && gd->ndim != 3) return fail(WD_ERR_INVALID, "ndim must be 2 or 3");
  if (sd->scheme < WD_UW || sd->scheme > WD_C6) return fail(WD_ERR_INVALID, "unknown scheme");
  if (sd->kind < WD_EIKONAL || sd->kind > WD_POISSON)
    return fail(WD_ERR_INVALID, "unknown formulation");
  if (!(sd->cfl > 0.0)) return fail(WD_ERR_INVALID, "cfl must be positive");
  if (!(sd->tol > 0.0)) return fail(WD_ERR_INVALID, "tol must be positive");
  if (sd->epsilon < 0.0) return fail(WD_ERR_INVALID, "epsilon must be non-negative");
  if (sd->lad_c < 0.0) return fail(WD_ERR_INVALID, "lad_c must be non-negative");
  if (!(sd->eps0 > 0.0)) return fail(WD_ERR_INVALID, "eps0 must be positive");
  if (sd->use_filter && !(sd->alpha_f >= 0.40 && sd->alpha_f <= 0.5))
    return fail(WD_ERR_INVALID, "alpha_f must lie in [0.40, 0.5]");
  if (!(gd->ref_length > 0.0)) return fail(WD_ERR_INVALID, "ref_length must be positive");
  if (sd->arith != 0 && sd->arith != 1) return fail(WD_ERR_INVALID, "arith must be 0 (exact) or 1 (fast)");
  for (int a = 0; a < gd->ndim; ++a) {
    const int lo = gd->face[2 * a], hi = gd->face[2 * a + 1];
    if ((lo == WD_FACE_PERIODIC) != (hi == WD_FACE_PERIODIC))
      return fail(WD_ERR_INVALID, "periodic faces must come in lo/hi pairs");
    const int n = gd->dims[a];
    const bool per = lo == WD_FACE_PERIODIC;
    if (n < 1) return fail(WD_ERR_INVALID, "bad dims");
    const int need = per ? 5 : min_line(sd->scheme);
    if (n < need)
      return fail(WD_ERR_LINE_TOO_SHORT, std::string(scheme_name(sd->scheme)) +
                                             " derivative needs at least " +
                                             std::to_string(need) + " points, got " +
                                             std::to_string(n));
    if ((sd->kind == WD_HJ_LAD) && n < 5)
      return fail(WD_ERR_LINE_TOO_SHORT, "fourth derivative needs at least 5 points");
    if (sd->scheme == WD_UW && sd->kind != WD_EIKONAL && n < 3)
      return fail(WD_ERR_LINE_TOO_SHORT, "E2 derivative needs at least 3 points");
    if (per && sd->use_filter && sd->scheme != WD_UW && sd->alpha_f >= 0.5)
      return fail(WD_ERR_INVALID, "periodic filter needs alpha_f < 0.5");
  }
  if (!gd->uniform && gd->metrics_dev == nullptr)
    return fail(WD_ERR_INVALID, "metrics required for a non-uniform grid");
  return WD_OK;
}

}  // namespace

// Parked contexts.  A solve_steady() call builds a context, runs, and
// destroys it; for the same grid and scheme the next call would redo the
// factorisation, ~10 small cudaMalloc / cudaFree (each a device-wide
// synchronisation), the stream and event creation, the tile-list uploads and
// the CUDA-graph instantiation -- 10-140 ms of jitter on a 0.15-0.4 s
// one-shot solve.  Contexts whose descriptors hold no
// caller-owned device pointers (uniform grid, no solid mask) are parked on
// wd_destroy (at most kCtxPoolMax, oldest evicted) and handed back by
// wd_create for an equal descriptor; tol / max_iters may differ (they only
// invalidate the captured graphs).  WD_NO_CTX_POOL disables it.
namespace {
constexpr size_t kCtxPoolMax = 2;
std::mutex g_pool_mu;
std::vector<wd_ctx*> g_ctx_pool;

std::string env_signature() {
  static const char* knobs[] = {"WD_DISABLE_FUSED", "WD_NO_FAST3", "WD_FILTER_ORDER", "WD_NO_DSCAN",
                                "WD_SCAN_GENERIC", "WD_NO_GEN_SCANF", "WD_NO_ZERO_SKIP",
                                "WD_NO_ASM_EXTRA", "WD_NO_RHS_SEG", "WD_NO_TILED_FEW"};
  std::string sig;
  for (const char* k : knobs) {
    const char* v = getenv(k);
    sig += v ? v : "-";
    sig += '|';
  }
  return sig;
}
bool ctx_poolable(const wd_grid_desc& gd) {
  static const bool off = getenv("WD_NO_CTX_POOL") != nullptr;
  return !off && gd.uniform && gd.metrics_dev == nullptr && gd.solid_mask_dev == nullptr;
}
bool same_desc(const wd_ctx* c, const wd_grid_desc& gd, const wd_solver_desc& sd, bool use_filter) {
  const wd_grid_desc& a = c->gd;
  if (a.ndim != gd.ndim || a.uniform != gd.uniform || a.ref_length != gd.ref_length) return false;
  for (int k = 0; k < 3; ++k)
    if (k < gd.ndim && (a.dims[k] != gd.dims[k] || a.inv_spacing[k] != gd.inv_spacing[k]))
      return false;
  for (int k = 0; k < 2 * gd.ndim; ++k)
    if (a.face[k] != gd.face[k]) return false;
  const wd_solver_desc& b = c->sd;
  return b.scheme == sd.scheme && b.kind == sd.kind && b.epsilon == sd.epsilon &&
         b.lad_c == sd.lad_c && b.eps0 == sd.eps0 && (b.use_filter != 0) == use_filter &&
         (!use_filter || b.alpha_f == sd.alpha_f) && b.cfl == sd.cfl && b.arith == sd.arith;
}
}  // namespace

extern "C" {

int wd_version(void) { return 100; }

const char* wd_last_error(void) { return g_last_error.c_str(); }

int wd_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int wd_create(const wd_grid_desc* gd, const wd_solver_desc* sd, void* stream, wd_ctx** out) {
  line_solve_prepare();
  if (!gd || !sd || !out) return fail(WD_ERR_INVALID, "null argument");
  int rc = validate(gd, sd);
  if (rc) return rc;
  if (ctx_poolable(*gd)) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    const int dev = ws_device();
    const bool uf = sd->use_filter && sd->scheme != WD_UW;
    for (size_t i = g_ctx_pool.size(); i-- > 0;) {
      wd_ctx* p = g_ctx_pool[i];
      if (p->device != dev || !same_desc(p, *gd, *sd, uf) || p->env_sig != env_signature())
        continue;
      g_ctx_pool.erase(g_ctx_pool.begin() + i);
      if (p->sd.tol != sd->tol || p->sd.max_iters != sd->max_iters) {
        for (auto& kv : p->graphs) cudaGraphExecDestroy(kv.second);  // tol is a graph argument
        p->graphs.clear();
        p->sd.tol = sd->tol;
        p->sd.max_iters = sd->max_iters;
      }
      p->fused.i_lo = p->fused.i_hi = 0;
      p->enq = 0;
      p->nopool = false;
      *out = p;
      return WD_OK;
    }
  }
  wd_ctx* c = new wd_ctx();
  c->device = ws_device();
  c->env_sig = env_signature();
  c->gd = *gd;
  c->sd = *sd;
  c->sd.use_filter = sd->use_filter && sd->scheme != WD_UW;
  c->g = make_geom(gd->ndim, gd->dims, gd->face, gd->solid_mask_dev);
  const Geom& g = c->g;
  c->M.m = gd->uniform ? nullptr : gd->metrics_dev;
  c->M.N = g.N;
  c->M.nd = g.nd;
  c->M.kdiv = 0;
  for (int a = 0; a < 3; ++a) c->M.c[a] = gd->uniform ? gd->inv_spacing[a] : 0.0;
  (void)stream;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return fail(WD_ERR_CUDA, "stream create failed");
  }
  // factors
  std::vector<double> packed, all;
  size_t off_comp[3] = {0, 0, 0}, off_filt[3] = {0, 0, 0}, off_scan[3] = {0, 0, 0};
  size_t off_cscan[3] = {0, 0, 0};
  int scan_m[3] = {0, 0, 0}, cscan_m[3] = {0, 0, 0}, lscan_m[3] = {0, 0, 0};
  size_t off_lscan[3] = {0, 0, 0};
  HostFactor cfast[3];
  for (int a = 0; a < g.nd; ++a) {
    if (sd->scheme == WD_C4 || sd->scheme == WD_C6) {
      rc = compact_factor(sd->scheme, g.n[a], g.per[a], c->hcomp[a]);
      if (rc) {
        wd_destroy(c);
        return rc;
      }
      factor_pack(c->hcomp[a], packed);
      off_comp[a] = all.size();
      all.insert(all.end(), packed.begin(), packed.end());
      if (sd->arith == 1 && !getenv("WD_NO_DSCAN") &&
          compact_factor_fast(sd->scheme, g.n[a], g.per[a], cfast[a]) == WD_OK &&
          scan_pack(cfast[a], packed, cscan_m[a], dscan_segments(g.n[a]))) {
        off_cscan[a] = all.size();
        all.insert(all.end(), packed.begin(), packed.end());
      } else {
        cscan_m[a] = 0;
      }
    }
    if (c->sd.use_filter && g.n[a] >= 3) {
      rc = filter_factor(sd->alpha_f, g.n[a], g.per[a], c->hfilt[a]);
      if (rc) {
        wd_destroy(c);
        return rc;
      }
      factor_pack(c->hfilt[a], packed);
      off_filt[a] = all.size();
      all.insert(all.end(), packed.begin(), packed.end());
      if (sd->arith == 1 && scan_pack(c->hfilt[a], packed, scan_m[a])) {
        off_scan[a] = all.size();
        all.insert(all.end(), packed.begin(), packed.end());
      } else {
        scan_m[a] = 0;
        if (sd->arith == 1 && g.nd == 2 && g.n[a] > FS_NMAX &&
            scan_pack(c->hfilt[a], packed, lscan_m[a], FL_S)) {
          off_lscan[a] = all.size();
          all.insert(all.end(), packed.begin(), packed.end());
        } else {
          lscan_m[a] = 0;
        }
      }
    }
  }
  if (c->sd.use_filter) c->fcoef = filter_coefs(sd->alpha_f);
  if (!all.empty()) {
    if (cudaMalloc(&c->factor_dev, all.size() * sizeof(double)) != cudaSuccess ||
        upload_sync(c->factor_dev, all.data(), all.size() * sizeof(double)) != cudaSuccess) {
      wd_destroy(c);
      return fail(WD_ERR_CUDA, "factor upload failed");
    }
    for (int a = 0; a < g.nd; ++a) {
      if (c->hcomp[a].n) c->comp[a] = factor_view(c->hcomp[a], c->factor_dev + off_comp[a]);
      if (c->hfilt[a].n) c->filt[a] = factor_view(c->hfilt[a], c->factor_dev + off_filt[a]);
      if (cscan_m[a]) {
        c->cscan[a].n = cfast[a].n;
        c->cscan[a].m = cscan_m[a];
        c->cscan[a].tab = c->factor_dev + off_cscan[a];
        c->cscan[a].denom = cfast[a].cyclic ? cfast[a].denom : 1.0;
      }
      if (scan_m[a]) {
        c->scan[a].n = c->hfilt[a].n;
        c->scan[a].m = scan_m[a];
        c->scan[a].tab = c->factor_dev + off_scan[a];
        c->scan[a].denom = c->hfilt[a].cyclic ? c->hfilt[a].denom : 1.0;
      }
      if (lscan_m[a]) {
        c->lscan[a].n = c->hfilt[a].n;
        c->lscan[a].m = lscan_m[a];
        c->lscan[a].tab = c->factor_dev + off_lscan[a];
        c->lscan[a].denom = c->hfilt[a].cyclic ? c->hfilt[a].denom : 1.0;
      }
    }
  }
  // workspace: the 7 fields every path uses; the generic path's 24 more
  // (derivatives, U, U_hat, ...) are allocated on first use (ensure_generic)
  const int ncore = 7;
  if (ws_alloc((void**)&c->ws, (size_t)ncore * g.N * sizeof(double)) != cudaSuccess) {
    wd_destroy(c);
    return fail(WD_ERR_CUDA, "workspace allocation failed (" +
                                 std::to_string((double)ncore * g.N * 8 / 1e9) + " GB)");
  }
  {
    double* w = c->ws;
    c->p = w;
    c->k = w + g.N;
    c->acc = w + 2 * g.N;
    c->dt = w + 3 * g.N;
    c->tmp = w + 4 * g.N;
    c->tmp2 = w + 5 * g.N;
    c->phiY = w + 6 * g.N;
  }
  if (cudaMalloc(&c->st, 2 * sizeof(Status)) != cudaSuccess ||
      cudaMalloc(&c->hist_scratch, 8 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&c->flag_dev, sizeof(int)) != cudaSuccess) {
    wd_destroy(c);
    return fail(WD_ERR_CUDA, "status allocation failed");
  }
  c->st_scratch = c->st + 1;
  // metric sums
  if (gd->uniform) {
    double tot = 0.0, ms = 0.0;
    for (int l = 0; l < g.nd; ++l) {
      const double S = gd->inv_spacing[l] * gd->inv_spacing[l];
      tot = l == 0 ? S : tot + S;
      const double sq = std::sqrt(S);
      const double sp = 1.0 / sq;
      ms = l == 0 ? sp : std::min(ms, sp);
      c->sqrtS_c[l] = sq;
    }
    c->sumS_c = tot;
    c->cflms_c = sd->cfl * ms;
  } else {
    if (cudaMalloc(&c->sums_dev, (size_t)(2 + g.nd) * g.N * sizeof(double)) != cudaSuccess) {
      wd_destroy(c);
      return fail(WD_ERR_CUDA, "metric-sum allocation failed");
    }
    k_metric_sums<<<nblocks(g.N, kThreads), kThreads, 0, c->stream>>>(
        c->M, c->sums_dev, c->sums_dev + g.N, c->sums_dev + 2 * g.N, sd->cfl, g.N, g.nd);
  }
  {
    FusedInputs fi;
    fi.gd = &c->gd;
    fi.sd = &c->sd;
    fi.g = c->g;
    fi.M = c->M;
    fi.fcoef = c->fcoef;
    for (int a = 0; a < 3; ++a) {
      fi.filt[a] = c->filt[a];
      fi.scan[a] = c->scan[a];
      fi.filt_swaps[a] = 0;
      for (double sw : c->hfilt[a].swap) fi.filt_swaps[a] |= sw != 0.0;
    }
    fi.sumS_c = c->sumS_c;
    fi.cflms_c = c->cflms_c;
    fi.lref = c->gd.ref_length;
    fi.bufs[0] = c->dt;
    fi.bufs[1] = c->acc;
    fi.bufs[2] = c->p;
    fi.bufs[3] = c->k;
    fi.bufs[4] = c->tmp;
    fi.bufs[5] = c->tmp2;
    fused_plan(c->fused, fi);
  }
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) {
    wd_destroy(c);
    return fail(WD_ERR_CUDA, "context setup failed");
  }
  c->nopool = false;
  *out = c;
  return WD_OK;
}

int wd_destroy(wd_ctx* c) {
  if (!c) return WD_OK;
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->stream && c->ws && c->st && !c->nopool && !c->dist && ctx_poolable(c->gd)) {
    wd_ctx* evict = nullptr;
    {
      std::lock_guard<std::mutex> lk(g_pool_mu);
      g_ctx_pool.push_back(c);
      if (g_ctx_pool.size() > kCtxPoolMax) {
        evict = g_ctx_pool.front();
        g_ctx_pool.erase(g_ctx_pool.begin());
      }
    }
    if (!evict) return WD_OK;
    c = evict;
    c->nopool = true;  // really destroy the evicted one
  }
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
  fused_release(c->fused);
  for (auto& kv : c->dfilt) cudaFree(kv.second.second);
  cudaFree(c->factor_dev);
  cudaFree(c->mk_dev);
  cudaFree(c->sums_dev);
  ws_free(c->ws, (size_t)7 * c->g.N * sizeof(double));
  ws_free(c->ws_generic, (size_t)27 * c->g.N * sizeof(double));
  cudaFree(c->st);
  cudaFree(c->hist_scratch);
  cudaFree(c->flag_dev);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return WD_OK;
}

int wd_bind(wd_ctx* c, double* phi, double* hist) {
  if (!c || !phi || !hist) return fail(WD_ERR_INVALID, "null argument");
  CK(cudaDeviceSynchronize());
  if (phi != c->phi || hist != c->hist) {
    for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
    c->graphs.clear();
  }
  c->phi = phi;
  c->hist = hist;
  c->enq = 0;
  Status s;
  std::memset(&s, 0, sizeof(s));
  s.state = c->sd.max_iters > 0 ? WD_STATE_RUNNING : WD_STATE_MAXITERS;
  s.max_iters = c->sd.max_iters;
  CK(cudaMemcpyAsync(c->st, &s, sizeof(s), cudaMemcpyHostToDevice, c->stream));
  k_bc<<<nblocks(c->g.N, kThreads), kThreads, 0, c->stream>>>(phi, c->tmp, c->g, nullptr);
  CK(cudaMemcpyAsync(phi, c->tmp, c->g.N * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return WD_OK;
}

int wd_steps(wd_ctx* c, int k) {
  if (!c || !c->phi) return fail(WD_ERR_INVALID, "context not bound");
  if (k <= 0) return WD_OK;
  if (!c->fused.active) {
    const int rc = ensure_generic(c);
    if (rc) return rc;
  }
  const int parity = (int)(c->enq & 1);
  if (getenv("WD_NO_GRAPH")) {  // plain launches (debugging, per-kernel profiling)
    for (int s = 0; s < k; ++s) {
      const bool even = ((parity + s) & 1) == 0;
      enqueue_step(c, even ? c->phi : c->phiY, even ? c->phiY : c->phi);
    }
    CK(cudaGetLastError());
    c->enq += k;
    return WD_OK;
  }
  auto key = std::make_pair(k, parity);
  auto it = c->graphs.find(key);
  if (it == c->graphs.end()) {
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    for (int s = 0; s < k; ++s) {
      const bool even = ((parity + s) & 1) == 0;
      enqueue_step(c, even ? c->phi : c->phiY, even ? c->phiY : c->phi);
    }
    CK(cudaStreamEndCapture(c->stream, &graph));
    cudaGraphExec_t exec;
    cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(WD_ERR_CUDA, std::string("graph: ") + cudaGetErrorString(e));
    it = c->graphs.emplace(key, exec).first;
  }
  CK(cudaGraphLaunch(it->second, c->stream));
  c->enq += k;
  return WD_OK;
}

int wd_read_status(wd_ctx* c, wd_status* out) {
  if (!c || !out) return fail(WD_ERR_INVALID, "null argument");
  Status s;
  CK(cudaMemcpyAsync(&s, c->st, sizeof(s), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  out->state = s.state;
  out->iters = s.iters;
  out->max_iters = s.max_iters;
  out->diverged_iter = s.diverged_iter;
  return WD_OK;
}

int wd_status_async(wd_ctx* c, wd_status* out) {
  if (!c || !out) return fail(WD_ERR_INVALID, "null argument");
  // wd_status is the leading 4 ints of Status
  CK(cudaMemcpyAsync(out, c->st, sizeof(wd_status), cudaMemcpyDeviceToHost, c->stream));
  return WD_OK;
}

int wd_finish(wd_ctx* c) {
  wd_status s;
  int rc = wd_read_status(c, &s);
  if (rc) return rc;
  // step t (1-based) writes phiY when t is odd; frozen steps write nothing
  if (s.state != WD_STATE_DIVERGED && (s.iters & 1))
    CK(cudaMemcpyAsync(c->phi, c->phiY, c->g.N * sizeof(double), cudaMemcpyDeviceToDevice,
                       c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return WD_OK;
}

void* wd_get_stream(wd_ctx* c) { return c ? (void*)c->stream : nullptr; }

int wd_fused_active(wd_ctx* c) { return c && c->fused.active ? 1 : 0; }

int wd_time_kernel(wd_ctx* c, int kid, int reps, double* avg_ms) {
  if (!c || !c->phi || !avg_ms || reps < 1) return fail(WD_ERR_INVALID, "bad arguments");
  if (!c->fused.active) return fail(WD_ERR_INVALID, "no fused path for this configuration");
  if (kid < 1 || kid > 8 || (kid >= 5 && kid <= 7 && !c->sd.use_filter))
    return fail(WD_ERR_INVALID, "bad kernel id");
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  fused_launch(c->fused, kid, c->phi, c->phiY, c->st, c->stream);  // warm
  CK(cudaEventRecord(e0, c->stream));
  for (int r = 0; r < reps; ++r) fused_launch(c->fused, kid, c->phi, c->phiY, c->st, c->stream);
  CK(cudaEventRecord(e1, c->stream));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *avg_ms = ms / reps;
  return WD_OK;
}

int wd_kernel_words(wd_ctx* c, int kid) {
  if (!c || !c->fused.active || kid < 1 || kid > 8) return 0;
  // stages 1-4, filters along axes (sweep order) 0, 1, 2 (+ reduction), change
  static const int classic[9] = {0, 4, 6, 6, 5, 2, 2, 3, 2};
  static const int low[9] = {0, 3, 5, 4, 5, 2, 2, 3, 2};
  return (c->fused.use_fast3 && fast3_lowstorage()) ? low[kid] : classic[kid];
}

int wd_tendency(wd_ctx* c, const double* phi, double* k) {
  if (!c) return fail(WD_ERR_INVALID, "null ctx");
  if (const int rc = ensure_generic(c)) return rc;
  CK(cudaDeviceSynchronize());
  enqueue_tendency(c, phi, k, nullptr);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));
  return WD_OK;
}

int wd_local_timestep(wd_ctx* c, const double* phi, double* dt) {
  if (!c) return fail(WD_ERR_INVALID, "null ctx");
  if (const int rc = ensure_generic(c)) return rc;
  CK(cudaDeviceSynchronize());
  enqueue_timestep(c, phi, dt, nullptr);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));
  return WD_OK;
}

int wd_apply_bc(wd_ctx* c, double* phi) {
  if (!c) return fail(WD_ERR_INVALID, "null ctx");
  CK(cudaDeviceSynchronize());
  k_bc<<<nblocks(c->g.N, kThreads), kThreads, 0, c->stream>>>(phi, c->tmp, c->g, nullptr);
  CK(cudaMemcpyAsync(phi, c->tmp, c->g.N * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return WD_OK;
}

int wd_rk4_step(wd_ctx* c, const double* phi, const double* dt, double* out, int* diverged) {
  if (!c) return fail(WD_ERR_INVALID, "null ctx");
  if (const int rc = ensure_generic(c)) return rc;
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpyAsync(c->dt, dt, c->g.N * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  enqueue_rk4(c, phi, out, nullptr);
  Status s;
  std::memset(&s, 0, sizeof(s));
  s.max_iters = 1 << 30;
  CK(cudaMemcpyAsync(c->st_scratch, &s, sizeof(s), cudaMemcpyHostToDevice, c->stream));
  k_change<<<nblocks(c->g.N, kThreads), kThreads, 0, c->stream>>>(out, phi, c->g.mask,
                                                                   c->st_scratch, c->g.N);
  k_finalize<<<1, 1, 0, c->stream>>>(c->st_scratch, c->hist_scratch, lref(c), 0.0,
                                     1e6 * lref(c));
  CK(cudaMemcpyAsync(&s, c->st_scratch, sizeof(s), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (diverged) *diverged = s.state == WD_STATE_DIVERGED;
  return WD_OK;
}

int wd_poisson_post(wd_ctx* c, const double* pp, double* phi) {
  return wd_poisson_map(c, pp, phi, 1);
}

int wd_poisson_map(wd_ctx* c, const double* pp, double* phi, int apply_bc) {
  if (!c) return fail(WD_ERR_INVALID, "null ctx");
  if (const int rc = ensure_generic(c)) return rc;
  CK(cudaDeviceSynchronize());
  const Geom& g = c->g;
  const int csch = c->sd.scheme == WD_UW ? WD_E2 : c->sd.scheme;
  const int nb = nblocks(g.N, kThreads);
  k_poisson_clip<<<nb, kThreads, 0, c->stream>>>(pp, c->p, g.N);
  for (int l = 0; l < g.nd; ++l) launch_deriv(c, c->p, c->dphi[l], c->tmp, l, csch, epi_plain(), nullptr);
  launch_assemble(c, c->dphi, c->U, nullptr, nullptr);
  CK(cudaMemsetAsync(c->flag_dev, 0, sizeof(int), c->stream));
  Vec3 uv;
  for (int l = 0; l < 3; ++l) uv.p[l] = c->U[l];
  k_poisson_map<<<nb, kThreads, 0, c->stream>>>(c->p, uv, c->tmp, g.N, g.nd, c->flag_dev);
  int neg = 0;
  CK(cudaMemcpyAsync(&neg, c->flag_dev, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  if (apply_bc)
    k_bc<<<nb, kThreads, 0, c->stream>>>(c->tmp, phi, g, nullptr);
  else
    CK(cudaMemcpyAsync(phi, c->tmp, g.N * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (neg) return fail(WD_ERR_NEGATIVE_RADICAND, "negative radicand in the Poisson map");
  return WD_OK;
}

int wd_derivative(const double* in, double* out, int ndim, const int* dims, int axis, int scheme,
                  int periodic, double offset, void* stream) {
  if (!in || !out || !dims || ndim < 1 || ndim > 3 || axis < 0 || axis >= ndim)
    return fail(WD_ERR_INVALID, "bad arguments");
  if (scheme == WD_UW || scheme < 0 || scheme > WD_C6)
    return fail(WD_ERR_INVALID, "use upwind_front_derivative for the UW scheme");
  const int n = dims[axis];
  const int need = periodic ? 5 : min_line(scheme);
  if (n < need)
    return fail(WD_ERR_LINE_TOO_SHORT, std::string(scheme_name(scheme)) +
                                           " derivative needs at least " + std::to_string(need) +
                                           " points, got " + std::to_string(n));
  int face[6] = {0, 0, 0, 0, 0, 0};
  if (periodic) face[2 * axis] = face[2 * axis + 1] = WD_FACE_PERIODIC;
  Geom g = make_geom(ndim, dims, face, nullptr);
  cudaStream_t s = (cudaStream_t)stream;
  if (scheme == WD_C4 || scheme == WD_C6) {
    HostFactor F;
    int rc = compact_factor(scheme, n, periodic, F);
    if (rc) return rc;
    std::vector<double> packed;
    factor_pack(F, packed);
    double* dev = nullptr;
    CK(cudaMallocAsync(&dev, packed.size() * sizeof(double), s));
    CK(cudaMemcpyAsync(dev, packed.data(), packed.size() * sizeof(double), cudaMemcpyHostToDevice,
                       s));
    const long long L = g.N / n;
    line_solve_prepare();
    if (line_solve_ok(n) && in != out)
      launch_line_solve<0>(in, out, out, g, axis, periodic, offset, scheme, factor_view(F, dev),
                           epi_plain(), FilterCoef{}, nullptr, 0, nullptr, s);
    else
      k_deriv_compact<<<nblocks(L, kLineThreads), kLineThreads, 0, s>>>(
          in, out, out, g, axis, scheme, periodic, offset, factor_view(F, dev), epi_plain(),
          nullptr);
    CK(cudaFreeAsync(dev, s));
    CK(cudaStreamSynchronize(s));
  } else {
    k_deriv_explicit<<<nblocks(g.N, kThreads), kThreads, 0, s>>>(in, out, axis_geom(g, axis), scheme,
                                                                   periodic, offset, epi_plain(),
                                                                   nullptr);
  }
  CK(cudaGetLastError());
  return WD_OK;
}

int wd_fourth_derivative(const double* in, double* out, int ndim, const int* dims, int axis,
                         int periodic, void* stream) {
  if (!in || !out || !dims || ndim < 1 || ndim > 3 || axis < 0 || axis >= ndim)
    return fail(WD_ERR_INVALID, "bad arguments");
  if (dims[axis] < 5)
    return fail(WD_ERR_LINE_TOO_SHORT, "fourth derivative needs at least 5 points, got " +
                                           std::to_string(dims[axis]));
  int face[6] = {0, 0, 0, 0, 0, 0};
  if (periodic) face[2 * axis] = face[2 * axis + 1] = WD_FACE_PERIODIC;
  Geom g = make_geom(ndim, dims, face, nullptr);
  k_d4<<<nblocks(g.N, kThreads), kThreads, 0, (cudaStream_t)stream>>>(in, out, axis_geom(g, axis), periodic,
                                                                       epi_plain(), nullptr);
  CK(cudaGetLastError());
  return WD_OK;
}

int wd_filter(const double* in, double* out, const unsigned char* pinned, int ndim,
              const int* dims, int axis, double alpha_f, int periodic, void* stream) {
  if (!in || !out || in == out || !dims || ndim < 1 || ndim > 3 || axis < 0 || axis >= ndim)
    return fail(WD_ERR_INVALID, "bad arguments");
  if (!(alpha_f >= 0.40 && alpha_f <= 0.5))
    return fail(WD_ERR_INVALID, "alpha_f must lie in [0.40, 0.5]");
  const int n = dims[axis];
  if (periodic && alpha_f >= 0.5) return fail(WD_ERR_INVALID, "periodic filter needs alpha_f < 0.5");
  if (periodic && n < 5) return fail(WD_ERR_LINE_TOO_SHORT, "periodic filter needs 5 points");
  int face[6] = {0, 0, 0, 0, 0, 0};
  if (periodic) face[2 * axis] = face[2 * axis + 1] = WD_FACE_PERIODIC;
  Geom g = make_geom(ndim, dims, face, nullptr);
  cudaStream_t s = (cudaStream_t)stream;
  HostFactor F;
  TriDev T;
  std::memset(&T, 0, sizeof(T));
  double* dev = nullptr;
  if (n >= 3 || periodic) {
    int rc = filter_factor(alpha_f, n, periodic, F);
    if (rc) return rc;
    std::vector<double> packed;
    factor_pack(F, packed);
    CK(cudaMallocAsync(&dev, packed.size() * sizeof(double), s));
    CK(cudaMemcpyAsync(dev, packed.data(), packed.size() * sizeof(double), cudaMemcpyHostToDevice,
                       s));
    T = factor_view(F, dev);
  }
  const long long L = g.N / n;
  line_solve_prepare();
  if (line_solve_ok(n))
    launch_line_solve<1>(in, out, out, g, axis, periodic, 0.0, 0, T, epi_plain(),
                         filter_coefs(alpha_f), pinned, 0, nullptr, s);
  else
    k_filter<<<nblocks(L, kLineThreads), kLineThreads, 0, s>>>(in, out, g, axis, periodic,
                                                                 filter_coefs(alpha_f), T, pinned,
                                                                 0, nullptr);
  CK(cudaGetLastError());
  if (dev) CK(cudaFreeAsync(dev, s));
  CK(cudaStreamSynchronize(s));
  return WD_OK;
}

}  // extern "C"

namespace {
__global__ void k_tri_lines(double* x, Geom g, int axis, TriDev T) {
  const long long sa = pick(g.s, axis);
  const int n = pick(g.n, axis);
  const long long L = g.N / n;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < L;
       q += (long long)gridDim.x * blockDim.x)
    tri_solve_line(x + line_base(g, axis, q), sa, T);
}
}  // namespace

extern "C" {

int wd_solve_tridiagonal(const double* lower, const double* diag, const double* upper,
                         double* rhs, int n, int nrhs, void* stream) {
  if (!lower || !diag || !upper || !rhs || n < 1 || nrhs < 1)
    return fail(WD_ERR_INVALID, "bad arguments");
  HostFactor F;
  if (n == 1) {
    if (diag[0] == 0.0) return fail(WD_ERR_ZERO_PIVOT, "1x1 tridiagonal system with zero diagonal");
    F.n = 1;
    F.d.assign(1, diag[0]);
    F.fact.assign(1, 0.0);
    F.du.assign(1, 0.0);
    F.du2.assign(1, 0.0);
    F.swap.assign(1, 0.0);
    F.z.assign(1, 0.0);
  } else {
    int rc = gtsv_factor(n, lower, diag, upper, F);
    if (rc) return rc;
  }
  int dims[2] = {n, nrhs};
  Geom g = make_geom(2, dims, nullptr, nullptr);
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<double> packed;
  factor_pack(F, packed);
  double* dev = nullptr;
  CK(cudaMallocAsync(&dev, packed.size() * sizeof(double), s));
  CK(cudaMemcpyAsync(dev, packed.data(), packed.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  k_tri_lines<<<nblocks(nrhs, kLineThreads), kLineThreads, 0, s>>>(rhs, g, 0, factor_view(F, dev));
  CK(cudaGetLastError());
  CK(cudaFreeAsync(dev, s));
  CK(cudaStreamSynchronize(s));
  return WD_OK;
}

int wd_compute_metrics(const double* coords, double* metrics, double* jac, int ndim,
                       const int* dims, int scheme, const int* periodic, const double* periods,
                       void* stream) {
  if (!coords || !metrics || !jac || !dims || (ndim != 2 && ndim != 3))
    return fail(WD_ERR_INVALID, "bad arguments");
  const int csch = scheme == WD_UW ? WD_E2 : scheme;
  int face[6] = {0, 0, 0, 0, 0, 0};
  for (int a = 0; a < ndim; ++a)
    if (periodic && periodic[a]) face[2 * a] = face[2 * a + 1] = WD_FACE_PERIODIC;
  Geom g = make_geom(ndim, dims, face, nullptr);
  cudaStream_t s = (cudaStream_t)stream;
  double* fwd = nullptr;
  CK(cudaMallocAsync(&fwd, (size_t)ndim * ndim * g.N * sizeof(double), s));
  int rc = WD_OK;
  for (int m = 0; m < ndim && rc == WD_OK; ++m)
    for (int l = 0; l < ndim && rc == WD_OK; ++l) {
      const double off = periods ? periods[l * ndim + m] : 0.0;
      rc = wd_derivative(coords + (long long)m * g.N, fwd + (long long)(m * ndim + l) * g.N, ndim,
                         dims, l, csch, g.per[l], off, stream);
    }
  int* flag = nullptr;
  if (rc == WD_OK) {
    CK(cudaMallocAsync(&flag, sizeof(int), s));
    CK(cudaMemsetAsync(flag, 0, sizeof(int), s));
    k_metric_invert<<<nblocks(g.N, kThreads), kThreads, 0, s>>>(fwd, metrics, jac, g.N, ndim,
                                                                  flag);
    int h = 0;
    CK(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (h) rc = fail(WD_ERR_SINGULAR_METRIC, "metric matrix is singular at a node");
    cudaFreeAsync(flag, s);
  }
  cudaFreeAsync(fwd, s);
  CK(cudaStreamSynchronize(s));
  return rc;
}

int wd_linf_delta(const double* a, const double* b, const unsigned char* mask, long long n,
                  double* out, void* stream) {
  if (!a || !b || !out) return fail(WD_ERR_INVALID, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* dev = nullptr;
  CK(cudaMallocAsync(&dev, sizeof(unsigned long long), s));
  CK(cudaMemsetAsync(dev, 0, sizeof(unsigned long long), s));
  k_linf<<<nblocks(n, kThreads), kThreads, 0, s>>>(a, b, mask, dev, n);
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, dev, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(dev, s));
  CK(cudaStreamSynchronize(s));
  double v;
  std::memcpy(&v, &h, sizeof(v));
  *out = v;
  return WD_OK;
}

int wd_sampled_wall_distance(const double* pts, long long n, const double* wall, long long m,
                             int d, double* out, void* stream) {
  if (!pts || !wall || !out || n < 0 || m < 1 || d < 1 || d > 3)
    return fail(WD_ERR_INVALID, "bad arguments");
  if (n == 0) return WD_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const long long per_cta = (long long)MP_T * MP_PTS;
  const int blocks = (int)((n + per_cta - 1) / per_cta);
  if (d == 1) k_sampled_distance<1><<<blocks, MP_T, 0, s>>>(pts, n, wall, m, out);
  else if (d == 2) k_sampled_distance<2><<<blocks, MP_T, 0, s>>>(pts, n, wall, m, out);
  else k_sampled_distance<3><<<blocks, MP_T, 0, s>>>(pts, n, wall, m, out);
  CK(cudaGetLastError());
  return WD_OK;
}

int wd_l2_norm(const double* phi, const double* exact, const double* jac, double jac_const,
               long long n, double* out, void* stream) {
  if (!phi || !exact || !out || n < 1) return fail(WD_ERR_INVALID, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  double* dev = nullptr;
  CK(cudaMallocAsync(&dev, (L2_B + 1) * sizeof(double), s));
  const int nb = (int)std::min<long long>(L2_B, (n + L2_T - 1) / L2_T);
  k_l2_partial<<<nb, L2_T, 0, s>>>(phi, exact, jac, jac_const, n, dev + 1);
  k_l2_final<<<1, L2_T, 0, s>>>(dev + 1, nb, dev);
  CK(cudaMemcpyAsync(out, dev, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(dev, s));
  CK(cudaStreamSynchronize(s));
  return WD_OK;
}

int wd_gradient_magnitude(wd_ctx* c, const double* phi, double* out) {
  if (!c || !phi || !out) return fail(WD_ERR_INVALID, "bad arguments");
  int rc = ensure_generic(c);
  if (rc != WD_OK) return rc;
  CK(cudaDeviceSynchronize());
  launch_dphi(c, phi, nullptr);
  launch_assemble(c, c->dphi, c->U, c->Uh, nullptr);
  MVec3 U;
  for (int a = 0; a < 3; ++a) U.p[a] = c->U[a];
  k_gradmag<<<nblocks(c->g.N, kThreads), kThreads, 0, c->stream>>>(U, c->g.N, c->g.nd, out);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));
  return WD_OK;
}

int wd_levelset_step(wd_ctx* c, const double* p0, double* out, double F, double dt,
                     double source) {
  if (!c || !p0 || !out || p0 == out) return fail(WD_ERR_INVALID, "bad arguments");
  int rc = ensure_generic(c);
  if (rc != WD_OK) return rc;
  CK(cudaDeviceSynchronize());
  const Geom& g = c->g;
  const int nb = nblocks(g.N, kThreads);
  MVec3 U;
  for (int a = 0; a < 3; ++a) U.p[a] = c->U[a];
  // rate(p) -> k (levelset.py:185-188)
  auto rate = [&](const double* p, double* k) {
    launch_dphi(c, p, nullptr);
    launch_assemble(c, c->dphi, c->U, c->Uh, nullptr);
    k_ls_rate<<<nb, kThreads, 0, c->stream>>>(U, g.N, g.nd, F, source, k);
  };
  // classical RK4 with the Neumann (far-field) BC on every stage
  // (levelset.py:190-199): the solver's stage kernels with dt as a field
  k_fill<<<nb, kThreads, 0, c->stream>>>(c->dt, dt, g.N);
  rate(p0, c->acc);
  rk_stage(c->g.nd, nb, c->stream, 1, p0, c->dt, c->acc, c->acc, c->p, g, nullptr);
  rate(c->p, c->k);
  rk_stage(c->g.nd, nb, c->stream, 2, p0, c->dt, c->k, c->acc, c->p, g, nullptr);
  rate(c->p, c->k);
  rk_stage(c->g.nd, nb, c->stream, 3, p0, c->dt, c->k, c->acc, c->p, g, nullptr);
  rate(c->p, c->k);
  rk_stage(c->g.nd, nb, c->stream, 4, p0, c->dt, c->k, c->acc, out, g, nullptr);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));
  return WD_OK;
}

}  // extern "C"

#include "wd_dist.cuh"
