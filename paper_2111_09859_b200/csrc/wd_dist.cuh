// Slab-decomposed pseudo-time solve; included at the end of
// wd_capi.cu.  One process per GPU owns the planes [rank nl, (rank + 1) nl) of
// the periodic axis 0.  Two step programs share this object:
//
// FUSED (uniform 3-D E2/E4/E6 HJ/Eikonal, BASELINE config 4): the slab is
//   stored with G ghost planes per side; per RK stage the stage input's
//   ghost planes are exchanged on a side stream while the fused stage kernel
//   runs on the planes whose stencils stay inside the rank, then the 2 G
//   boundary planes; the axis-0 filter is the partitioned solve of
//   wd_dist_filter0.cuh (fast arithmetic: one kernel, one all_gather of 3
//   doubles per line, one fix-up) or a slab <-> pencil transpose pair (exact
//   arithmetic: bit-identical to one GPU); axes 1, 2 are filtered locally,
//   the last sweep accumulating the local maxima; one all_reduce(max) of
//   three words feeds the stop test, identical on every rank.
// GENERIC (curvilinear / compact / LAD / curvature / Poisson / UW / masks,
//   BASELINE config 5): the rank's context works on its (nl, n1[, n2]) slab;
//   every operator ALONG axis 0 -- explicit or compact derivative, one-sided
//   differences, 4th derivative, filter -- is evaluated on pencils
//   (n0, n1 / P[, n2]) between two all_to_all transposes ("solve the
//   undecomposed directions locally and transpose for the decomposed one"),
//   with the derivative epilogue (metric contraction, accumulation) and the
//   pinned-node restore applied while unpacking.  Every line sees exactly
//   the single-GPU operations, so the decomposed solve is bit-identical.
//
// With an NCCL communicator k steps are captured into one CUDA graph
// (collectives included) with the in-device freeze-on-stop.
#pragma once

#include <unistd.h>

#include "wd_comm.cuh"

struct wd_dist {
  wd_comm* comm = nullptr;
  wd_ctx* c = nullptr;
  int nd = 3, n0 = 0, n1 = 0, n2 = 1, nl = 0, G = 0, P = 1, rank = 0, m1 = 0;
  int fused = 0;     // 1: FUSED program, 0: GENERIC
  int filter0 = 0;   // fused: 0 partitioned, 1 transpose
  int overlap = 0;
  int rc = WD_OK;    // first error raised inside an enqueue hook
  long long plane = 0, Nl = 0, Ng = 0;  // nodes per plane, per slab, per ghosted slab
  // fused program
  double* A = nullptr;  // ghosted state (B = c->phiY, Pa = c->p, Pb = c->k)
  double *mine = nullptr, *all = nullptr, *coef2 = nullptr;
  const double* fixc = nullptr;  // this step's filtered correction planes, if fused
  wd::F0Tables f0;
  double* f0_dev = nullptr;
  // transposes / pencils
  double *send = nullptr, *recv = nullptr, *pscr = nullptr;
  Geom gp;                  // pencil geometry (n0, m1[, n2]), axis 0 periodic
  HostFactor hfilt0, hcomp0;
  TriDev filt0, comp0;
  ScanDev scan0, cscan0;
  double* fac0_dev = nullptr;
  long long* stats = nullptr;
  // peer-memory ghost push (p2p = 1): neighbours' images of c->ws and of the
  // barrier flags, opened through CUDA IPC (same-process ranks: the pointers)
  int p2p = 0;
  double *peer_ws_l = nullptr, *peer_ws_r = nullptr;
  unsigned long long* xflags = nullptr;  // [0] written by the left rank, [1] by the right, [2] epoch
  unsigned long long *xflag_l = nullptr, *xflag_r = nullptr;  // my slots in the neighbours
  void* ipc_open[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaStream_t cs = nullptr;  // communication stream (ghost planes)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  double* phi = nullptr;      // caller's (nl, n1, n2) state
  double* hist = nullptr;
  long long enq = 0;
  std::map<std::pair<int, int>, cudaGraphExec_t> graphs;
};

namespace {

int dfail(wd_dist* d, int code, const std::string& msg) {
  if (d && d->rc == WD_OK) d->rc = code;
  return fail(code, msg);
}

#define DCK(d, expr)                                                                   \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return dfail(d, WD_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

int comm_rc(wd_dist* d, int rc) {
  if (rc != WD_OK) return dfail(d, rc, d->comm->err);
  return WD_OK;
}

// slab (nl, n1, n2) -> all_to_all buffer (P, nl, n1/P, n2)
__global__ void k_pack_slab(const double* __restrict__ slab, double* __restrict__ buf, int nl,
                            int n1, int n2, int P, const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  const int m1 = n1 / P;
  const long long N = (long long)nl * n1 * n2;
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < N;
       o += (long long)gridDim.x * blockDim.x) {
    long long t = o;
    const int k = (int)(t % n2);
    t /= n2;
    const int jj = (int)(t % m1);
    t /= m1;
    const int i = (int)(t % nl);
    const int q = (int)(t / nl);
    buf[o] = slab[((long long)i * n1 + (long long)q * m1 + jj) * n2 + k];
  }
}
// all_to_all buffer (P, nl, n1/P, n2) -> slab; MODE 0: the derivative
// epilogue e (D, c D or acc + c D, exactly Epi::apply of the local kernels),
// MODE 1: pinned nodes of the slab keep `orig` (apply_filter's restore,
// operators.py:349-351)
template <int MODE>
__global__ void k_unpack_slab(const double* __restrict__ buf, double* slab, int nl, int n1, int n2,
                              int P, Epi e, Geom g, const double* __restrict__ orig,
                              const Status* st) {
  if (st && st->state != WD_STATE_RUNNING) return;
  const int m1 = n1 / P;
  const long long N = (long long)nl * n1 * n2;
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < N;
       o += (long long)gridDim.x * blockDim.x) {
    long long t = o;
    const int k = (int)(t % n2);
    t /= n2;
    const int jj = (int)(t % m1);
    t /= m1;
    const int i = (int)(t % nl);
    const int q = (int)(t / nl);
    const long long idx = ((long long)i * n1 + (long long)q * m1 + jj) * n2 + k;
    double v = buf[o];
    if (MODE == 0) {
      v = e.apply(v, idx);
    } else if (orig) {
      int cc[kMaxDim];
      node_coords(g, idx, cc);
      if (is_pinned(g, idx, cc)) v = orig[idx];
    }
    slab[idx] = v;
  }
}
__global__ void k_stats_out(const Status* st, long long* out) {
  out[0] = (long long)st->max_delta_bits;
  out[1] = (long long)st->max_abs_bits;
  out[2] = st->nonfinite;
}
__global__ void k_stats_in(Status* st, const long long* in) {
  st->max_delta_bits = (unsigned long long)in[0];
  st->max_abs_bits = (unsigned long long)in[1];
  st->nonfinite = (int)in[2];
}

// Neighbour barrier of the peer-memory path: every rank runs the same
// sequence of these, so a per-rank epoch counter names the barrier.  Thread 0
// publishes the epoch into both neighbours' flag slots (release, system
// scope: the stage kernel's ghost-plane stores precede it in stream order)
// and spins until both of its own slots have reached the epoch (acquire).
__global__ void k_xbar(unsigned long long* mine, unsigned long long* at_left,
                       unsigned long long* at_right) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned long long e = mine[2] + 1;
  mine[2] = e;
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(at_left + 1), "l"(e) : "memory");
  asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(at_right), "l"(e) : "memory");
  for (int side = 0; side < 2; ++side) {
    unsigned long long v;
    do {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(mine + side) : "memory");
    } while (v < e);
  }
}

// All neighbours' ghost pushes of the kernels enqueued so far have landed
// (and theirs into mine): device flags with NCCL ranks, a host barrier with
// the callback communicators (tests), nothing for a rank running alone.
int dist_xbar(wd_dist* d) {
  wd_ctx* c = d->c;
  if (d->comm->kind == 2 || d->P == 1) return WD_OK;
  if (d->comm->kind == 1) {
    DCK(d, cudaStreamSynchronize(c->stream));
    return comm_rc(d, d->comm->allreduce_max(d->stats + 8, 1, c->stream));
  }
  k_xbar<<<1, 32, 0, c->stream>>>(d->xflags, d->xflag_l, d->xflag_r);
  return WD_OK;
}

// ---- transposes -------------------------------------------------------
int dist_to_pencil(wd_dist* d, const double* slab, double* pencil, const Status* st) {
  wd_ctx* c = d->c;
  k_pack_slab<<<nblocks(d->Nl, kThreads), kThreads, 0, c->stream>>>(slab, d->send, d->nl, d->n1,
                                                                    d->n2, d->P, st);
  return comm_rc(d, d->comm->alltoall(d->send, pencil, (size_t)(d->Nl / d->P), c->stream));
}
// pencil -> all_to_all buffer d->recv (unpacked by the caller)
int dist_from_pencil(wd_dist* d, const double* pencil) {
  return comm_rc(d, d->comm->alltoall(pencil, d->recv, (size_t)(d->Nl / d->P), d->c->stream));
}
void dist_unpack_epi(wd_dist* d, double* out, const Epi& e, const Status* st) {
  k_unpack_slab<0><<<nblocks(d->Nl, kThreads), kThreads, 0, d->c->stream>>>(
      d->recv, out, d->nl, d->n1, d->n2, d->P, e, d->c->g, nullptr, st);
}

// ---- axis-0 operators of the GENERIC program (hooks of the enqueue code) ----
// central derivative along axis 0 with epilogue e -> out
void dist_deriv0(wd_ctx* c, const double* in, double* out, int scheme, const Epi& e,
                 const Status* st) {
  wd_dist* d = c->dist;
  double* pin = d->pscr;   // pencil input
  double* pout = d->send;  // pencil output (the pack buffer is free again)
  if (dist_to_pencil(d, in, pin, st)) return;
  const Geom& gp = d->gp;
  if ((scheme == WD_C4 || scheme == WD_C6) && d->cscan0.tab && scheme == c->sd.scheme) {
    DScanArgs a;
    a.in = pin;
    a.out = pout;
    a.N = gp.N;
    a.sa = gp.s[0];
    a.per = 1;
    a.scheme = scheme;
    a.T = d->cscan0;
    a.epi = epi_plain();
    a.st = st;
    const int n = gp.n[0];
    const DScanShape sh = dscan_shape(n, a.sa == 1);
    const long long lines = gp.N / n;
    const long long groups = a.sa == 1 ? (lines + sh.NL - 1) / sh.NL : (a.sa + sh.NL - 1) / sh.NL;
    const int blocks = (int)std::min<long long>(groups, 148LL * (sh.TT == 256 ? 2 : 1));
    const DScanFn fn = dscan_kernel(n, a.sa == 1, true, scheme == WD_C6);
    fn<<<blocks, sh.TT, dscan_smem(n, sh), c->stream>>>(a);
  } else if (scheme == WD_C4 || scheme == WD_C6) {
    if (line_solve_ok(gp.n[0])) {
      launch_line_solve<0>(pin, pout, pout, gp, 0, 1, 0.0, scheme, d->comp0, epi_plain(), c->fcoef,
                           nullptr, 0, st, c->stream);
    } else {
      const long long L = gp.N / gp.n[0];
      k_deriv_compact<<<nblocks(L, kLineThreads), kLineThreads, 0, c->stream>>>(
          pin, pout, pout, gp, 0, scheme, 1, 0.0, d->comp0, epi_plain(), st);
    }
  } else {
    k_deriv_explicit<<<nblocks(gp.N, kThreads), kThreads, 0, c->stream>>>(
        pin, pout, axis_geom(gp, 0), scheme, 1, 0.0, epi_plain(), st);
  }
  if (dist_from_pencil(d, pout)) return;
  dist_unpack_epi(d, out, e, st);
}

// one-sided differences + front derivative along axis 0 (UW scheme)
void dist_uw0(wd_ctx* c, const double* p, double* B, double* F, double* dphi, const Status* st) {
  wd_dist* d = c->dist;
  // three pencil outputs: B and F share the generic workspace's spare
  // pencils (tmp, tmp2 are free while the one-sided differences are taken)
  double* pin = d->pscr;
  if (dist_to_pencil(d, p, pin, st)) return;
  double* pB = c->tmp;
  double* pF = c->tmp2;
  double* pD = d->send;
  k_uw_bf<<<nblocks(d->gp.N, kThreads), kThreads, 0, c->stream>>>(pin, pB, pF, pD,
                                                                  axis_geom(d->gp, 0), 1, st);
  double* outs[3] = {B, F, dphi};
  const double* pens[3] = {pB, pF, pD};
  for (int t = 0; t < 3; ++t) {
    if (dist_from_pencil(d, pens[t])) return;
    dist_unpack_epi(d, outs[t], epi_plain(), st);
  }
}

// 4th derivative along axis 0 with epilogue e -> e.acc / out (LAD sensor)
void dist_d40(wd_ctx* c, const double* p, double* out, const Epi& e, const Status* st) {
  wd_dist* d = c->dist;
  double* pin = d->pscr;
  double* pout = d->send;
  if (dist_to_pencil(d, p, pin, st)) return;
  k_d4<<<nblocks(d->gp.N, kThreads), kThreads, 0, c->stream>>>(pin, pout, axis_geom(d->gp, 0), 1,
                                                               epi_plain(), st);
  if (dist_from_pencil(d, pout)) return;
  dist_unpack_epi(d, out, e, st);
}

// implicit filter along axis 0: cur -> nxt, pinned nodes restored
void dist_filter0_generic(wd_ctx* c, const double* cur, double* nxt, const Status* st) {
  wd_dist* d = c->dist;
  double* pin = d->pscr;
  double* pout = d->send;
  if (dist_to_pencil(d, cur, pin, st)) return;
  const Geom& gp = d->gp;
  const bool scan = st && c->sd.arith == 1 && c->g.nd == 3 && c->g.mask == nullptr && d->scan0.tab &&
                    !getenv("WD_NO_GEN_SCANF");
  if (scan) {
    FusedPlan fp;
    fp.in.fcoef = c->fcoef;
    fused_filter_any(fp, 0, pin, pout, gp.n[0], gp.n[1], gp.n[2], 1, d->filt0, nullptr,
                     const_cast<Status*>(st), c->stream, &d->scan0);
  } else if (line_solve_ok(gp.n[0])) {
    launch_line_solve<1>(pin, pout, pout, gp, 0, 1, 0.0, 0, d->filt0, epi_plain(), c->fcoef,
                         nullptr, 0, st, c->stream);
  } else {
    const long long L = gp.N / gp.n[0];
    k_filter<<<nblocks(L, kLineThreads), kLineThreads, 0, c->stream>>>(
        pin, pout, gp, 0, 1, c->fcoef, d->filt0, nullptr, 0, st);
  }
  if (dist_from_pencil(d, pout)) return;
  k_unpack_slab<1><<<nblocks(d->Nl, kThreads), kThreads, 0, c->stream>>>(
      d->recv, nxt, d->nl, d->n1, d->n2, d->P, epi_plain(), c->g, scan ? nullptr : cur, st);
}

// local maxima of the status word -> max over the ranks (before k_finalize)
void dist_reduce(wd_dist* d) {
  wd_ctx* c = d->c;
  if (d->P == 1 && !d->comm->nccl) return;
  k_stats_out<<<1, 1, 0, c->stream>>>(c->st, d->stats);
  if (comm_rc(d, d->comm->allreduce_max(d->stats, 3, c->stream))) return;
  k_stats_in<<<1, 1, 0, c->stream>>>(c->st, d->stats);
}
void dist_reduce_status(wd_ctx* c) { dist_reduce(c->dist); }

// ---- FUSED program -----------------------------------------------------
int dist_stage_range(wd_dist* d, int stage, const double* A, const double* p, double* out, int lo,
                     int hi) {
  wd_ctx* c = d->c;
  c->fused.i_lo = lo;
  c->fused.i_hi = hi;
  fused_stage_ptrs(c->fused, stage, A, p, out, c->st, c->stream);
  return WD_OK;
}

int dist_f0_tables(wd_dist* d) {
  wd_ctx* c = d->c;
  // solo communicator: the slab wraps onto itself, so its rows ARE a cyclic
  // line of nl rows (one block); the all_gather still moves P slots
  const bool solo = d->comm->kind == 2;
  const int n0 = solo ? d->nl : d->n0, nl = d->nl, P = solo ? 1 : d->P;
  const int lo = solo ? 0 : d->rank * nl;
  HostFactor F;
  int rc = filter_factor(c->sd.alpha_f, n0, 1, F);
  if (rc) return rc;
  for (double sw : F.swap)
    if (sw != 0.0) return fail(WD_ERR_INVALID, "filter factor with interchanges");
  std::vector<double> fm(n0), ri(n0), g(n0), h(n0), z(n0);
  for (int r = 0; r < n0; ++r) {
    fm[r] = r > 0 ? F.fact[r - 1] : 0.0;
    ri[r] = 1.0 / F.d[r];
    g[r] = r < n0 - 1 ? F.du[r] * ri[r] : 0.0;
    h[r] = F.cyclic ? F.h[r] : 0.0;
    z[r] = F.cyclic ? F.z[r] : 0.0;
  }
  // segments: exactly MM rows each when nl = S * MM with MM in {4, 8, 16}
  int m = 0, S = 0;
  for (int mm : {16, 8, 4})
    if (!m && nl % mm == 0 && nl / mm <= F0_SMAX && nl / mm >= 1 &&
        (mm == 16 || nl / mm <= 16)) {
      m = mm;
      S = nl / mm;
    }
  if (!m || getenv("WD_F0_GENERIC")) {
    S = 16;
    m = (nl + S - 1) / S;
    if (m > 32) return fail(WD_ERR_INVALID, "slab too thick for the partitioned axis-0 filter");
    S = (nl + m - 1) / m;
    d->f0.m = -m;  // runtime rows per segment (generic kernel)
  } else {
    d->f0.m = m;
  }
  d->f0.S = S;
  std::vector<double> tab((size_t)9 * nl + 3 * P);
  double* tfm = tab.data();
  double* th = tfm + nl;
  double* tPs = th + nl;
  double* tg = tPs + nl;
  double* tri = tg + nl;
  double* tQs = tri + nl;
  double* tW = tQs + nl;
  double* tQp = tW + nl;
  double* tz = tQp + nl;
  for (int r = 0; r < nl; ++r) {
    tfm[r] = fm[lo + r];
    th[r] = h[lo + r];
    tg[r] = g[lo + r];
    tri[r] = ri[lo + r];
    tz[r] = z[lo + r];
  }
  for (int r0 = 0; r0 < nl; r0 += m) {
    const int r1 = std::min(nl, r0 + m);
    tPs[r0] = -tfm[r0];
    for (int r = r0 + 1; r < r1; ++r) tPs[r] = -tfm[r] * tPs[r - 1];
    tQs[r1 - 1] = -tg[r1 - 1];
    for (int r = r1 - 2; r >= r0; --r) tQs[r] = -tg[r] * tQs[r + 1];
  }
  // rank-level rows of every rank q: Pp, W, Qp; this rank's go to the table
  double* blk = tab.data() + 9 * nl;
  for (int q = 0; q < P; ++q) {
    const int b = q * nl;
    std::vector<double> Pp(nl), W(nl), Qp(nl);
    double pp = 1.0;
    for (int r = 0; r < nl; ++r) {
      pp *= -fm[b + r];
      Pp[r] = pp;
    }
    double w = 0.0, qq = 1.0;
    for (int r = nl - 1; r >= 0; --r) {
      w = Pp[r] * ri[b + r] - g[b + r] * w;
      W[r] = w;
      qq *= -g[b + r];
      Qp[r] = qq;
    }
    blk[3 * q] = Pp[nl - 1];
    blk[3 * q + 1] = Qp[0];
    blk[3 * q + 2] = W[0];
    if (q == (solo ? 0 : d->rank))
      for (int r = 0; r < nl; ++r) {
        tW[r] = W[r];
        tQp[r] = Qp[r];
      }
  }
  CK(cudaMalloc(&d->f0_dev, tab.size() * sizeof(double)));
  CK(upload_sync(d->f0_dev, tab.data(), tab.size() * sizeof(double)));
  d->f0.tab = d->f0_dev;
  d->f0.blk = d->f0_dev + 9 * nl;
  d->f0.P = P;
  d->f0.rank = solo ? 0 : d->rank;
  d->f0.nl = nl;
  d->f0.rden = F.cyclic ? 1.0 / F.denom : 0.0;
  return WD_OK;
}

template <int MM>
void f0_launch(const F0Args& a, int threads, bool generic, cudaStream_t s) {
  static int ctas = 0;
  static size_t smax = 0;
  const size_t sm = f0_smem_bytes(a.T.nl, generic);
  if (!ctas || sm > smax) {
    int dev = 0, sms = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_f0_local<MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_f0_local<MM>, threads, sm);
    ctas = sms * (occ > 0 ? occ : 1);
    smax = sm;
  }
  const long long groups = (long long)a.n1 * ((a.n2 + F0_L - 1) / F0_L);
  k_f0_local<MM><<<(int)std::min<long long>(groups, ctas), threads, sm, s>>>(a);
}

// axis-0 filter of the ghosted stage-4 output Pb -> T1 (interior layout)
int dist_filter0_fused(wd_dist* d, double* Pb, double* T1) {
  wd_ctx* c = d->c;
  cudaStream_t s = c->stream;
  if (d->p2p) {
    if (int rc = dist_xbar(d)) return rc;  // stage 4 pushed Pb's ghost planes
  }
  if (d->filter0 == 0) {
    if (!d->p2p)
      if (int rc = comm_rc(d, d->comm->halo(Pb, d->plane, d->nl, d->G, s))) return rc;
    F0Args a;
    a.in = Pb;
    a.out = T1;
    a.mine = d->mine;
    a.n1 = d->n1;
    a.n2 = d->n2;
    a.G = d->G;
    a.T = d->f0;
    a.fc = c->fcoef;
    a.st = c->st;
    const int m = d->f0.m;
    a.T.m = m < 0 ? -m : m;
    const int threads = F0_L * d->f0.S;
    if (m == 16) f0_launch<16>(a, threads, false, s);
    else if (m == 8) f0_launch<8>(a, threads, false, s);
    else if (m == 4) f0_launch<4>(a, threads, false, s);
    else f0_launch<0>(a, threads, true, s);
    if (int rc = comm_rc(d, d->comm->allgather(d->mine, d->all, (size_t)3 * d->plane, s)))
      return rc;
    k_f0_carry<<<nblocks(d->plane, 256), 256, 0, s>>>(d->all, d->mine, d->plane, d->f0, c->st);
    // The correction cf W_i + cb Qp_i - f z_i is separable (per-line
    // coefficient x per-plane factor) and the j / k sweeps are linear, so
    // the sweeps can run on x' and the correction be added at the end with
    // the coefficient PLANES filtered instead: two tiny sweeps over 3 planes
    // and three L2-resident loads in the last sweep's store replace a
    // 2-word pass over the slab.
    // Measured at 512^3 (ncu, P = 1): the last sweep grows from 712 to 1044 us
    // with the three coefficient loads per node, the 318 us pass goes away:
    // no net gain, so the separate pass stays the default (WD_F0_FIX_FUSED=1
    // selects the fused form; tests/test_gpu_dist.py runs both).
    static const bool fusedfix = getenv("WD_F0_FIX_FUSED") != nullptr;
    if (fusedfix && d->coef2 && c->scan[1].tab && c->scan[2].tab) {
      fused_filter_any(c->fused, 1, d->mine, d->coef2, 3, d->n1, d->n2, c->g.per[1], c->filt[1],
                       nullptr, c->st, s, &c->scan[1]);
      fused_filter_any(c->fused, 2, d->coef2, d->mine, 3, d->n1, d->n2, c->g.per[2], c->filt[2],
                       nullptr, c->st, s, &c->scan[2]);
      d->fixc = d->mine;
      return WD_OK;
    }
    d->fixc = nullptr;
    const dim3 fg((unsigned)((d->plane + 255) / 256), (unsigned)((d->nl + F0_FR - 1) / F0_FR));
    k_f0_fix<<<fg, 256, 0, s>>>(T1, d->mine, d->nl, d->plane, d->f0, c->st);
    return WD_OK;
  }
  // slab -> pencil, sweep, pencil -> slab: every line sees the single-GPU sweep
  const double* x = Pb + (long long)d->G * d->plane;
  if (int rc = dist_to_pencil(d, x, d->pscr, c->st)) return rc;
  fused_filter_any(c->fused, 0, d->pscr, d->send, d->n0, d->m1, d->n2, 1, d->filt0, nullptr, c->st,
                   s, d->scan0.tab ? &d->scan0 : nullptr);
  if (int rc = dist_from_pencil(d, d->send)) return rc;
  dist_unpack_epi(d, T1, epi_plain(), c->st);
  return WD_OK;
}

// one pseudo-step X -> Y on the ghosted slabs
int dist_step_fused(wd_dist* d, double* X, double* Y) {
  wd_ctx* c = d->c;
  cudaStream_t s = c->stream;
  const int G = d->G, nl = d->nl;
  double* Pa = c->p;
  double* Pb = c->k;
  double* T1 = c->tmp;
  double* T2 = c->tmp2;
  double* ins[4] = {X, Pa, Pb, Pa};
  double* outs[4] = {Pa, Pb, Pa, Pb};
  for (int st = 0; st < 4; ++st) {
    if (d->p2p && st > 0) {
      // the previous stage pushed its boundary planes into the neighbours'
      // ghost planes as it wrote them: no exchange, one neighbour barrier
      if (int rc = dist_xbar(d)) return rc;
      dist_stage_range(d, st + 1, X, ins[st], outs[st], G, G + nl);
      continue;
    }
    if (d->overlap) {
      // planes [2G, nl): every stencil reach (<= G planes) stays inside the
      // rank's own planes, so they run while the ghost planes are in flight
      DCK(d, cudaEventRecord(d->ev_fork, s));
      DCK(d, cudaStreamWaitEvent(d->cs, d->ev_fork, 0));
      if (int rc = comm_rc(d, d->comm->halo(ins[st], d->plane, nl, G, d->cs))) return rc;
      DCK(d, cudaEventRecord(d->ev_join, d->cs));
      dist_stage_range(d, st + 1, X, ins[st], outs[st], 2 * G, nl);
      DCK(d, cudaStreamWaitEvent(s, d->ev_join, 0));
      dist_stage_range(d, st + 1, X, ins[st], outs[st], G, 2 * G);
      dist_stage_range(d, st + 1, X, ins[st], outs[st], nl, nl + G);
    } else {
      if (int rc = comm_rc(d, d->comm->halo(ins[st], d->plane, nl, G, s))) return rc;
      dist_stage_range(d, st + 1, X, ins[st], outs[st], G, G + nl);
    }
  }
  c->fused.i_lo = G;
  c->fused.i_hi = G + nl;
  d->fixc = nullptr;
  if (int rc = dist_filter0_fused(d, Pb, T1)) return rc;
  const long long go = (long long)G * d->plane;
  fused_filter_any(c->fused, 1, T1, T2, nl, d->n1, d->n2, c->g.per[1], c->filt[1], nullptr, c->st, s,
                   c->scan[1].tab ? &c->scan[1] : nullptr);
  fused_filter_any(c->fused, 2, T2, Y + go, nl, d->n1, d->n2, c->g.per[2], c->filt[2], X + go,
                   c->st, s, c->scan[2].tab ? &c->scan[2] : nullptr, d->fixc,
                   d->fixc ? d->f0.tab + 6 * nl : nullptr);
  dist_reduce(d);
  k_finalize<<<1, 1, 0, s>>>(c->st, d->hist, lref(c), c->sd.tol, 1e6 * lref(c));
  DCK(d, cudaGetLastError());
  return d->rc;
}

int dist_enqueue(wd_dist* d, int k, int parity) {
  wd_ctx* c = d->c;
  for (int t = 0; t < k; ++t) {
    const bool even = ((parity + t) & 1) == 0;
    if (d->fused) {
      if (int rc = dist_step_fused(d, even ? d->A : c->phiY, even ? c->phiY : d->A)) return rc;
    } else {
      enqueue_step(c, even ? c->phi : c->phiY, even ? c->phiY : c->phi);
      if (d->rc) return d->rc;
    }
  }
  return WD_OK;
}

// Peer-memory setup: every rank publishes (pid, raw pointers, IPC handles) of
// its workspace and flag allocations; each opens its two neighbours'.
int dist_p2p_setup(wd_dist* d) {
  wd_ctx* c = d->c;
  wd_comm* cm = d->comm;
  if (cudaMalloc(&d->xflags, 64) != cudaSuccess) return fail(WD_ERR_CUDA, "flag allocation failed");
  CK(memset_sync(d->xflags, 0, 64));
  if (cm->kind == 2 || d->P == 1) {  // alone: the slab wraps onto itself
    d->peer_ws_l = d->peer_ws_r = c->ws;
    d->xflag_l = d->xflag_r = d->xflags;
  } else {
    constexpr int W = 20;  // doubles per rank: pid, ws ptr, flag ptr, 2 x 64-byte handles
    struct Pub {
      long long pid;
      unsigned long long ws, fl;
      cudaIpcMemHandle_t hws, hfl;
    } me, *all;
    static_assert(sizeof(Pub) <= W * sizeof(double), "Pub does not fit");
    std::memset(&me, 0, sizeof(me));
    me.pid = (long long)getpid();
    me.ws = (unsigned long long)(uintptr_t)c->ws;
    me.fl = (unsigned long long)(uintptr_t)d->xflags;
    CK(cudaIpcGetMemHandle(&me.hws, c->ws));
    CK(cudaIpcGetMemHandle(&me.hfl, d->xflags));
    double *dm = nullptr, *da = nullptr;
    CK(cudaMalloc(&dm, W * sizeof(double)));
    CK(cudaMalloc(&da, (size_t)W * d->P * sizeof(double)));
    std::vector<double> hostm(W, 0.0), hosta((size_t)W * d->P);
    std::memcpy(hostm.data(), &me, sizeof(me));
    CK(upload_sync(dm, hostm.data(), W * sizeof(double)));
    int rc = cm->allgather(dm, da, W, c->stream);
    if (rc == WD_OK && cudaStreamSynchronize(c->stream) != cudaSuccess) rc = WD_ERR_CUDA;
    if (rc == WD_OK)
      CK(cudaMemcpy(hosta.data(), da, hosta.size() * sizeof(double), cudaMemcpyDeviceToHost));
    cudaFree(dm);
    cudaFree(da);
    if (rc) return fail(rc, "peer handle exchange failed: " + cm->err);
    auto open = [&](int q, int slot, double** ws, unsigned long long** fl) -> int {
      std::memcpy(&me, hosta.data() + (size_t)q * W, sizeof(me));  // reuse as scratch
      all = &me;
      if (all->pid == (long long)getpid()) {  // a logical rank of this process
        *ws = (double*)(uintptr_t)all->ws;
        *fl = (unsigned long long*)(uintptr_t)all->fl;
        return WD_OK;
      }
      void *pw = nullptr, *pf = nullptr;
      CK(cudaIpcOpenMemHandle(&pw, all->hws, cudaIpcMemLazyEnablePeerAccess));
      CK(cudaIpcOpenMemHandle(&pf, all->hfl, cudaIpcMemLazyEnablePeerAccess));
      d->ipc_open[2 * slot] = pw;
      d->ipc_open[2 * slot + 1] = pf;
      *ws = (double*)pw;
      *fl = (unsigned long long*)pf;
      return WD_OK;
    };
    if (int r2 = open(cm->left(), 0, &d->peer_ws_l, &d->xflag_l)) return r2;
    if (cm->right() == cm->left()) {  // two ranks: one neighbour on both sides
      d->peer_ws_r = d->peer_ws_l;
      d->xflag_r = d->xflag_l;
    } else if (int r3 = open(cm->right(), 1, &d->peer_ws_r, &d->xflag_r)) {
      return r3;
    }
  }
  c->fused.ws_base = c->ws;
  c->fused.peer_ws_l = d->peer_ws_l;
  c->fused.peer_ws_r = d->peer_ws_r;
  c->fused.push_nl = d->nl;
  c->fused.push_G = d->G;
  c->nopool = true;  // the plan now points into other ranks' memory
  d->p2p = 1;
  return WD_OK;
}

int dist_pencil_factors(wd_dist* d) {
  wd_ctx* c = d->c;
  const int n0 = d->n0;
  std::vector<double> all, packed;
  size_t off_f = 0, off_fs = 0, off_c = 0, off_cs = 0;
  int fs_m = 0, cs_m = 0;
  HostFactor cfast;
  const int sch = c->sd.scheme;
  if (c->sd.use_filter) {
    if (int rc = filter_factor(c->sd.alpha_f, n0, 1, d->hfilt0)) return rc;
    factor_pack(d->hfilt0, packed);
    off_f = all.size();
    all.insert(all.end(), packed.begin(), packed.end());
    if (c->sd.arith == 1 && scan_pack(d->hfilt0, packed, fs_m)) {
      off_fs = all.size();
      all.insert(all.end(), packed.begin(), packed.end());
    } else {
      fs_m = 0;
    }
  }
  if (sch == WD_C4 || sch == WD_C6) {
    if (int rc = compact_factor(sch, n0, 1, d->hcomp0)) return rc;
    factor_pack(d->hcomp0, packed);
    off_c = all.size();
    all.insert(all.end(), packed.begin(), packed.end());
    if (c->sd.arith == 1 && !getenv("WD_NO_DSCAN") &&
        compact_factor_fast(sch, n0, 1, cfast) == WD_OK &&
        scan_pack(cfast, packed, cs_m, dscan_segments(n0))) {
      off_cs = all.size();
      all.insert(all.end(), packed.begin(), packed.end());
    } else {
      cs_m = 0;
    }
  }
  if (all.empty()) return WD_OK;
  CK(cudaMalloc(&d->fac0_dev, all.size() * sizeof(double)));
  CK(upload_sync(d->fac0_dev, all.data(), all.size() * sizeof(double)));
  if (d->hfilt0.n) d->filt0 = factor_view(d->hfilt0, d->fac0_dev + off_f);
  if (d->hcomp0.n) d->comp0 = factor_view(d->hcomp0, d->fac0_dev + off_c);
  if (fs_m) {
    d->scan0.n = n0;
    d->scan0.m = fs_m;
    d->scan0.tab = d->fac0_dev + off_fs;
    d->scan0.denom = d->hfilt0.cyclic ? d->hfilt0.denom : 1.0;
    fused_filter_prepare(n0);
  }
  if (cs_m) {
    d->cscan0.n = n0;
    d->cscan0.m = cs_m;
    d->cscan0.tab = d->fac0_dev + off_cs;
    d->cscan0.denom = cfast.cyclic ? cfast.denom : 1.0;
  }
  if (d->hfilt0.n) fused_filter_prepare(n0);
  return WD_OK;
}

}  // namespace

extern "C" {

int wd_comm_unique_id(void* id_out) {
  if (!id_out) return fail(WD_ERR_INVALID, "null argument");
  std::string err;
  NcclApi* api = nccl_api(err);
  if (!api) return fail(WD_ERR_CUDA, err);
  NcclUniqueId id;
  const int rc = api->GetUniqueId(&id);
  if (rc) return fail(WD_ERR_CUDA, std::string("ncclGetUniqueId: ") + api->GetErrorString(rc));
  std::memcpy(id_out, &id, sizeof(id));
  return WD_OK;
}

int wd_comm_init(const void* nccl_id, int rank, int nranks, int decomposition, wd_comm** out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(WD_ERR_INVALID, "bad communicator arguments");
  if (decomposition != WD_DECOMP_SLAB0)
    return fail(WD_ERR_INVALID, "only the axis-0 slab decomposition is implemented");
  wd_comm* cm = new wd_comm();
  cm->rank = rank;
  cm->P = nranks;
  cm->kind = 0;
  cm->decomposition = decomposition;
  // WD_NCCL_SELF: a one-rank communicator still goes through NCCL (self
  // send/recv, all_gather, all_reduce inside the captured graph): exercises
  // the loader, the ABI constants and the capture on a single GPU
  const bool self = nranks == 1 && getenv("WD_NCCL_SELF") != nullptr;
  if (nranks > 1 || self) {
    if (!nccl_id && !self) {
      delete cm;
      return fail(WD_ERR_INVALID, "nccl_id is required for more than one rank");
    }
    std::string err;
    cm->api = nccl_api(err);
    if (!cm->api) {
      delete cm;
      return fail(WD_ERR_CUDA, err);
    }
    NcclUniqueId id;
    if (self) {
      const int rc0 = cm->api->GetUniqueId(&id);
      if (rc0) {
        const std::string msg = std::string("ncclGetUniqueId: ") + cm->api->GetErrorString(rc0);
        delete cm;
        return fail(WD_ERR_CUDA, msg);
      }
    } else {
      std::memcpy(&id, nccl_id, sizeof(id));
    }
    const int rc = cm->api->CommInitRank(&cm->nccl, nranks, id, rank);
    if (rc) {
      const std::string msg = std::string("ncclCommInitRank: ") + cm->api->GetErrorString(rc);
      delete cm;
      return fail(WD_ERR_CUDA, msg);
    }
  }
  *out = cm;
  return WD_OK;
}

int wd_comm_init_callbacks(const wd_comm_callbacks* cb, int rank, int nranks, wd_comm** out) {
  if (!out || !cb || nranks < 1 || rank < 0 || rank >= nranks || !cb->halo || !cb->allgather ||
      !cb->alltoall || !cb->allreduce_max)
    return fail(WD_ERR_INVALID, "bad communicator arguments");
  wd_comm* cm = new wd_comm();
  cm->rank = rank;
  cm->P = nranks;
  cm->kind = 1;
  cm->cb = *cb;
  *out = cm;
  return WD_OK;
}

int wd_comm_init_solo(int rank, int nranks, wd_comm** out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(WD_ERR_INVALID, "bad communicator arguments");
  wd_comm* cm = new wd_comm();
  cm->rank = rank;
  cm->P = nranks;
  cm->kind = 2;
  *out = cm;
  return WD_OK;
}

int wd_comm_allgather(wd_comm* cm, const double* mine, double* all, long long count,
                      void* stream) {
  if (!cm || !mine || !all || count < 0) return fail(WD_ERR_INVALID, "bad arguments");
  const int rc = cm->allgather(mine, all, (size_t)count, (cudaStream_t)stream);
  return rc ? fail(rc, cm->err) : WD_OK;
}

int wd_comm_destroy(wd_comm* cm) {
  if (!cm) return WD_OK;
  if (cm->nccl && cm->api) cm->api->CommDestroy(cm->nccl);
  delete cm;
  return WD_OK;
}

int wd_dist_destroy(wd_dist* d) {
  if (!d) return WD_OK;
  if (d->c && d->c->stream) cudaStreamSynchronize(d->c->stream);
  if (d->cs) cudaStreamSynchronize(d->cs);
  for (auto& kv : d->graphs) cudaGraphExecDestroy(kv.second);
  if (d->c) {
    d->c->dist = nullptr;
    wd_destroy(d->c);
  }
  for (void* p : d->ipc_open)
    if (p) cudaIpcCloseMemHandle(p);
  cudaFree(d->xflags);
  ws_free(d->A, (size_t)d->Ng * sizeof(double));
  cudaFree(d->mine);
  cudaFree(d->coef2);
  cudaFree(d->all);
  cudaFree(d->f0_dev);
  cudaFree(d->send);
  cudaFree(d->recv);
  cudaFree(d->pscr);
  cudaFree(d->fac0_dev);
  cudaFree(d->stats);
  if (d->cs) cudaStreamDestroy(d->cs);
  if (d->ev_fork) cudaEventDestroy(d->ev_fork);
  if (d->ev_join) cudaEventDestroy(d->ev_join);
  delete d;
  return WD_OK;
}

int wd_dist_create(wd_comm* cm, const wd_grid_desc* gd, const wd_solver_desc* sd, int filter0,
                   int overlap, wd_dist** out) {
  if (!cm || !gd || !sd || !out) return fail(WD_ERR_INVALID, "null argument");
  const int P = cm->P, nd = gd->ndim;
  if (nd != 2 && nd != 3) return fail(WD_ERR_INVALID, "ndim must be 2 or 3");
  if (gd->face[0] != WD_FACE_PERIODIC || gd->face[1] != WD_FACE_PERIODIC)
    return fail(WD_ERR_INVALID, "slab decomposition needs a periodic axis 0");
  const int n0 = gd->dims[0], n1 = gd->dims[1], n2 = nd == 3 ? gd->dims[2] : 1;
  if (n0 % P) return fail(WD_ERR_INVALID, "axis 0 must divide evenly over the ranks");
  if (P > 8) return fail(WD_ERR_INVALID, "at most 8 ranks (one NVSwitch box)");
  if (int rc = validate(gd, sd)) return rc;
  wd_dist* d = new wd_dist();
  d->comm = cm;
  d->P = P;
  d->rank = cm->rank;
  d->nd = nd;
  d->n0 = n0;
  d->n1 = n1;
  d->n2 = n2;
  d->nl = n0 / P;
  d->plane = (long long)n1 * n2;
  d->Nl = d->plane * d->nl;
  // FUSED when the single-GPU plan would be (decided on the global geometry)
  bool fusedok = nd == 3 && gd->uniform && !gd->solid_mask_dev && sd->use_filter &&
                 (sd->scheme == WD_E2 || sd->scheme == WD_E4 || sd->scheme == WD_E6) &&
                 (sd->kind == WD_HJ || sd->kind == WD_EIKONAL) && !getenv("WD_DIST_GENERIC");
  for (int f = 0; f < 6; ++f)
    if (gd->face[f] == WD_FACE_FARFIELD) fusedok = false;
  {
    const char* env = getenv("WD_DISABLE_FUSED");
    if (env && env[0] == '1') fusedok = false;
  }
  const int G = 7;  // >= 4 + R (exact axis-0 windows) and >= 2R (fast), R <= 3
  if (fusedok && d->nl < G) fusedok = false;
  d->fused = fusedok ? 1 : 0;
  d->filter0 = filter0 < 0 ? (sd->arith == 1 ? 0 : 1) : filter0;
  if (d->fused && d->filter0 == 0 && sd->arith != 1) {
    delete d;
    return fail(WD_ERR_INVALID, "the partitioned axis-0 filter is a fast-arithmetic path");
  }
  const bool need_pencil = !d->fused || d->filter0 == 1;
  if (need_pencil && n1 % P) {
    delete d;
    return fail(WD_ERR_INVALID, "axis 1 must divide evenly over the ranks (pencil transposes)");
  }
  d->m1 = n1 / P;
  if (cm->kind == 2 && !(d->fused && d->filter0 == 0)) {
    delete d;
    return fail(WD_ERR_INVALID, "the solo communicator times the fused partitioned program only");
  }
  // local context
  wd_grid_desc lg = *gd;
  if (d->fused) {
    d->G = G;
    lg.dims[0] = d->nl + 2 * G;
    lg.face[0] = lg.face[1] = WD_FACE_NONE;  // ghosts carry the wrap
  } else {
    d->G = 0;
    lg.dims[0] = d->nl;
    if (d->nl < 5 && P > 1) {
      delete d;
      return fail(WD_ERR_INVALID, "slab thinner than 5 planes");
    }
  }
  d->Ng = (long long)lg.dims[0] * d->plane;
  int rc = wd_create(&lg, sd, nullptr, &d->c);
  if (rc) {
    delete d;
    return rc;
  }
  wd_ctx* c = d->c;
  auto bail = [&](int code) {
    wd_dist_destroy(d);
    return code;
  };
  if (d->fused && !c->fused.active) return bail(fail(WD_ERR_INVALID, "configuration is not on the fused 3-D path"));
  if (!d->fused) c->nopool = true;  // fused plan released / axis-0 hooks: not reusable
  if (!d->fused && c->fused.active) fused_release(c->fused);
  if (cudaMalloc(&d->stats, 16 * sizeof(long long)) != cudaSuccess)
    return bail(fail(WD_ERR_CUDA, "allocation failed"));
  d->overlap = overlap && d->fused && P > 1 && d->nl >= 2 * G + 8 &&
               !getenv("WD_DIST_NO_OVERLAP");
  if (d->fused) {
    if (ws_alloc((void**)&d->A, (size_t)d->Ng * sizeof(double)) != cudaSuccess)
      return bail(fail(WD_ERR_CUDA, "slab allocation failed"));
    if (d->filter0 == 0) {
      if (cudaMalloc(&d->coef2, (size_t)3 * d->plane * sizeof(double)) != cudaSuccess ||
          cudaMalloc(&d->mine, (size_t)3 * d->plane * sizeof(double)) != cudaSuccess ||
          cudaMalloc(&d->all, (size_t)3 * P * d->plane * sizeof(double)) != cudaSuccess)
        return bail(fail(WD_ERR_CUDA, "carry buffer allocation failed"));
      if ((rc = dist_f0_tables(d))) return bail(rc);
    }
    if (getenv("WD_DIST_P2P") && fused_can_push(c->fused))
      if ((rc = dist_p2p_setup(d))) return bail(rc);
    if (cudaStreamCreateWithFlags(&d->cs, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&d->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d->ev_join, cudaEventDisableTiming) != cudaSuccess)
      return bail(fail(WD_ERR_CUDA, "stream create failed"));
  }
  if (need_pencil) {
    if (cudaMalloc(&d->send, (size_t)d->Nl * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&d->recv, (size_t)d->Nl * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&d->pscr, (size_t)d->Nl * sizeof(double)) != cudaSuccess)
      return bail(fail(WD_ERR_CUDA, "pencil buffer allocation failed"));
    int pd[3] = {n0, d->m1, n2};
    int pf[6] = {WD_FACE_PERIODIC, WD_FACE_PERIODIC, 0, 0, 0, 0};
    d->gp = make_geom(nd, pd, pf, nullptr);
    if ((rc = dist_pencil_factors(d))) return bail(rc);
  }
  if (!d->fused) {
    c->dist = d;
    if ((rc = ensure_generic(c))) return bail(rc);
    // identically-zero metric terms decide which line passes (and hence
    // which collectives) run: the flags must agree on every rank
    if (c->M.m && P > 1) {
      long long hf[9] = {0};
      for (int t = 0; t < 9; ++t) hf[t] = c->mterm[t];
      if (upload_sync(d->stats, hf, sizeof(hf)) != cudaSuccess)
        return bail(fail(WD_ERR_CUDA, "flag upload failed"));
      if ((rc = cm->allreduce_max(d->stats, 9, c->stream))) return bail(fail(rc, cm->err));
      if (cudaMemcpyAsync(hf, d->stats, sizeof(hf), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
          cudaStreamSynchronize(c->stream) != cudaSuccess)
        return bail(fail(WD_ERR_CUDA, "flag download failed"));
      for (int t = 0; t < 9; ++t) c->mterm[t] = hf[t] != 0;
    }
  }
  *out = d;
  return WD_OK;
}

int wd_dist_bind(wd_dist* d, double* phi, double* hist) {
  if (!d || !phi || !hist) return fail(WD_ERR_INVALID, "null argument");
  wd_ctx* c = d->c;
  CK(cudaDeviceSynchronize());
  if (phi != d->phi || hist != d->hist) {
    for (auto& kv : d->graphs) cudaGraphExecDestroy(kv.second);
    d->graphs.clear();
  }
  d->phi = phi;
  d->hist = hist;
  d->enq = 0;
  d->rc = WD_OK;
  if (!d->fused) return wd_bind(c, phi, hist);
  // ghosted state: interior <- phi, then the local BCs (walls) + status reset
  CK(cudaMemsetAsync(d->A, 0, (size_t)d->Ng * sizeof(double), c->stream));
  CK(cudaMemcpyAsync(d->A + (long long)d->G * d->plane, phi, (size_t)d->Nl * sizeof(double),
                     cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return wd_bind(c, d->A, hist);
}

int wd_dist_steps(wd_dist* d, int k) {
  if (!d || !d->phi) return fail(WD_ERR_INVALID, "context not bound");
  if (k <= 0) return WD_OK;
  wd_ctx* c = d->c;
  const int parity = (int)(d->enq & 1);
  if (!d->comm->capturable() || getenv("WD_DIST_NO_GRAPH")) {
    const int rc = dist_enqueue(d, k, parity);
    if (rc) return rc;
    CK(cudaGetLastError());
    d->enq += k;
    return WD_OK;
  }
  auto key = std::make_pair(k, parity);
  auto it = d->graphs.find(key);
  if (it == d->graphs.end()) {
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const int rc = dist_enqueue(d, k, parity);
    const cudaError_t ce = cudaStreamEndCapture(c->stream, &graph);
    if (rc) return rc;
    if (ce != cudaSuccess) return fail(WD_ERR_CUDA, std::string("capture: ") + cudaGetErrorString(ce));
    cudaGraphExec_t exec;
    const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(WD_ERR_CUDA, std::string("graph: ") + cudaGetErrorString(e));
    it = d->graphs.emplace(key, exec).first;
  }
  CK(cudaGraphLaunch(it->second, c->stream));
  d->enq += k;
  return WD_OK;
}

int wd_dist_read_status(wd_dist* d, wd_status* out) {
  if (!d) return fail(WD_ERR_INVALID, "null argument");
  return wd_read_status(d->c, out);
}

// The caller's slab holds the latest state afterwards.  Step t (1-based)
// writes the second buffer when t is odd and frozen steps write nothing, so
// the parity of the completed-step count says where the state lives -- not
// the number of steps enqueued (steps past a stop are no-ops).
int wd_dist_finish(wd_dist* d) {
  if (!d || !d->phi) return fail(WD_ERR_INVALID, "context not bound");
  wd_ctx* c = d->c;
  if (!d->fused) return wd_finish(c);
  wd_status s;
  if (int rc = wd_read_status(c, &s)) return rc;
  const double* src = (s.state != WD_STATE_DIVERGED && (s.iters & 1)) ? c->phiY : d->A;
  CK(cudaMemcpyAsync(d->phi, src + (long long)d->G * d->plane, (size_t)d->Nl * sizeof(double),
                     cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return WD_OK;
}

// One filter sweep of the fused path's kernels on an arbitrary (n0, n1, n2)
// array (operator-level parity of the scan / checkpointed sweeps).
int wd_fused_filter(wd_ctx* c, int axis, const double* in, double* out, int n0, int n1, int n2,
                    int periodic, const double* A) {
  if (!c || !c->fused.active || !c->sd.use_filter || axis < 0 || axis > 2)
    return fail(WD_ERR_INVALID, "bad arguments");
  const int nn[3] = {n0, n1, n2};
  const int n = nn[axis];
  auto key = std::make_pair(n, periodic ? 1 : 0);
  auto it = c->dfilt.find(key);
  if (it == c->dfilt.end()) {
    HostFactor F;
    int rc = filter_factor(c->sd.alpha_f, n, periodic, F);
    if (rc) return rc;
    for (double sw : F.swap)
      if (sw != 0.0) return fail(WD_ERR_INVALID, "filter factor with interchanges");
    std::vector<double> packed, sc;
    factor_pack(F, packed);
    int m = 0;
    const size_t nf = packed.size();
    if (c->sd.arith == 1 && scan_pack(F, sc, m)) packed.insert(packed.end(), sc.begin(), sc.end());
    double* dev = nullptr;
    CK(cudaMalloc(&dev, packed.size() * sizeof(double)));
    CK(upload_sync(dev, packed.data(), packed.size() * sizeof(double)));
    fused_filter_prepare(n);
    F.scan_m = m;
    F.scan_off = nf;
    it = c->dfilt.emplace(key, std::make_pair(F, dev)).first;
  }
  const TriDev T = factor_view(it->second.first, it->second.second);
  ScanDev SD;
  if (it->second.first.scan_m) {
    SD.n = n;
    SD.m = it->second.first.scan_m;
    SD.tab = it->second.second + it->second.first.scan_off;
    SD.denom = it->second.first.cyclic ? it->second.first.denom : 1.0;
  }
  fused_filter_any(c->fused, axis, in, out, n0, n1, n2, periodic, T, A, c->st, c->stream,
                   SD.n ? &SD : nullptr);
  CK(cudaGetLastError());
  return WD_OK;
}

// Marching-squares segments of a 2-D field (levelset.py:214-318): per cell
// (n0 - 1)(n1 - 1): count, 4 edge ids, 4 points (wd_metrics.cuh).
int wd_iso_segments(const double* field, const double* coords, int n0, int n1, double level,
                    int* count, long long* ids, double* pts, void* stream) {
  if (!field || !coords || !count || !ids || !pts || n0 < 2 || n1 < 2)
    return fail(WD_ERR_INVALID, "bad arguments");
  const long long cells = (long long)(n0 - 1) * (n1 - 1);
  k_iso_segments<<<nblocks(cells, kThreads), kThreads, 0, (cudaStream_t)stream>>>(
      field, coords, coords + (long long)n0 * n1, n0, n1, level, count, ids, pts);
  CK(cudaGetLastError());
  return WD_OK;
}

// running maxima of the status word (max|delta| bits, max|phi| bits, non-finite flag)
int wd_status_maxima(wd_ctx* c, long long* dev3) {
  if (!c || !dev3) return fail(WD_ERR_INVALID, "bad arguments");
  k_stats_out<<<1, 1, 0, c->stream>>>(c->st, dev3);
  CK(cudaGetLastError());
  return WD_OK;
}

void* wd_dist_stream(wd_dist* d) { return d ? (void*)d->c->stream : nullptr; }

wd_ctx* wd_dist_context(wd_dist* d) { return d ? d->c : nullptr; }

int wd_dist_info(wd_dist* d, int* out8) {
  if (!d || !out8) return fail(WD_ERR_INVALID, "null argument");
  out8[0] = d->nl;
  out8[1] = d->G;
  out8[2] = d->fused;
  out8[3] = d->filter0;
  out8[4] = d->overlap;
  out8[5] = (d->comm->capturable() && !getenv("WD_DIST_NO_GRAPH")) | (d->p2p << 1);
  out8[6] = d->P;
  out8[7] = d->rank;
  return WD_OK;
}

}  // extern "C"
