/*
 * walldist_b200.h -- C ABI of the B200-native pseudo-time wall-distance
 * solver (libwd_b200.so).
 *
 * The reference (walldist, pure Python/numpy) has no native ABI; these entry
 * points are what its solver would bind through ctypes to replace the hot
 * path (INTEGRATION.md shows the binding).  Each function cites the
 * reference interface it replaces.  All pointers named *_dev are CUDA device
 * pointers owned by the caller; every call is asynchronous on the given
 * context's stream unless stated otherwise.  A context runs on its OWN
 * non-blocking stream (wd_get_stream); the `stream` argument of wd_create is
 * reserved.  Results of wd_steps are valid for other streams only after
 * wd_finish / wd_read_status (both synchronise the context stream) or after
 * waiting on an event recorded on wd_get_stream().  Fields are fp64, C-order (n0, n1[, n2]),
 * axis 0 slowest (reference grid.py:5-11).  Metrics are (d, d, N) with
 * metrics[l][m] = d xi_l / d x_m (grid.py:9, 32).
 *
 * Return values: WD_OK or a WD_ERR_* code; wd_last_error() gives the text.
 * The Python layer maps the codes to the reference exception classes
 * (errors.py:8-44).
 */
#ifndef WALLDIST_B200_H
#define WALLDIST_B200_H

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (-> reference errors.py) -------------------------- */
#define WD_OK 0
#define WD_ERR_INVALID 1          /* ValueError                          */
#define WD_ERR_LINE_TOO_SHORT 2   /* LineTooShortError  errors.py:20     */
#define WD_ERR_ZERO_PIVOT 3       /* ZeroPivotError     errors.py:24     */
#define WD_ERR_SINGULAR_METRIC 4  /* SingularMetricError errors.py:16    */
#define WD_ERR_NEGATIVE_RADICAND 5 /* NegativeRadicandError errors.py:44 */
#define WD_ERR_DIVERGED 6         /* DivergenceError    errors.py:28     */
#define WD_ERR_CUDA 7             /* CUDA runtime failure                */
#define WD_ERR_DIM_TOO_SMALL 8    /* DimensionTooSmallError errors.py:8  */

/* ---- schemes (operators.py:24-36; E6 is an EXTENSION) --------------- */
#define WD_UW 0
#define WD_E2 1
#define WD_E4 2
#define WD_E6 3
#define WD_C4 4
#define WD_C6 5

/* ---- formulations (formulations.py:36) ------------------------------ */
#define WD_EIKONAL 0
#define WD_HJ 1
#define WD_HJ_LAD 2
#define WD_HJ_CURVATURE 3
#define WD_POISSON 4

/* ---- face kinds (solver.py:27-29; PERIODIC is an EXTENSION) --------- */
#define WD_FACE_NONE 0
#define WD_FACE_WALL 1
#define WD_FACE_FARFIELD 2
#define WD_FACE_PERIODIC 3

/* ---- solve states (device status word) ------------------------------ */
#define WD_STATE_RUNNING 0
#define WD_STATE_CONVERGED 1   /* change <= tol   solver.py:270-272      */
#define WD_STATE_DIVERGED 2    /* DivergenceError solver.py:214-217      */
#define WD_STATE_MAXITERS 3    /* converged=False solver.py:249          */

typedef struct wd_grid_desc {
  int ndim;                  /* 2 or 3                                    */
  int dims[3];               /* (n0, n1, n2); n2 ignored when ndim == 2   */
  int face[6];               /* WD_FACE_* for imin, imax, jmin, jmax, kmin, kmax */
  int uniform;               /* 1: diagonal constant metrics (build_cartesian) */
  double inv_spacing[3];     /* uniform only: d xi_l / d x_l              */
  const double* metrics_dev; /* (d, d, N) or NULL when uniform            */
  const unsigned char* solid_mask_dev; /* (N) or NULL (solver.py:42)      */
  double ref_length;         /* grid.ref_length                           */
} wd_grid_desc;

typedef struct wd_solver_desc {
  int scheme;                /* WD_UW..WD_C6   (SolveConfig.scheme)       */
  int kind;                  /* WD_EIKONAL..   (FormulationConfig.kind)   */
  double epsilon;            /* FormulationConfig.epsilon                 */
  double lad_c;              /* FormulationConfig.lad_c                   */
  double eps0;               /* resolved eps0 (1e-12/Lref when None)      */
  int use_filter;            /* SolveConfig.uses_filter()                 */
  double alpha_f;            /* FilterConfig.alpha_f                      */
  double cfl;                /* SolveConfig.cfl                           */
  double tol;                /* SolveConfig.tol                           */
  int max_iters;             /* SolveConfig.max_iters                     */
  int arith;                 /* EXTENSION: 0 exact (bit-identical to the
                                reference), 1 fast (FMA + composite
                                Laplacian stencil; round-off differences) */
} wd_solver_desc;

typedef struct wd_status {
  int state;                 /* WD_STATE_*                                */
  int iters;                 /* completed pseudo-steps                    */
  int max_iters;
  int diverged_iter;         /* 1-based iteration that raised, else 0     */
} wd_status;

typedef struct wd_ctx wd_ctx;

/* ---- library ---------------------------------------------------------- */
int wd_version(void);
const char* wd_last_error(void);
int wd_device_count(void);

/* ---- solver context (replaces solver.py:221-286 solve_steady) ---------
 * wd_create validates the configuration (SolveConfig.__post_init__
 * solver.py:125-129, FormulationConfig formulations.py:54-63, FilterConfig
 * operators.py:263-266, line lengths operators.py:106) and precomputes the
 * field-independent tridiagonal factors and per-node metric sums.        */
int wd_create(const wd_grid_desc* grid, const wd_solver_desc* solver, void* stream,
              wd_ctx** out);
/* Contexts whose descriptors carry no caller-owned device pointers (uniform
 * grid, no solid mask) are parked on wd_destroy (at most two per process)
 * and handed back by wd_create for an equal descriptor, so repeated one-shot
 * solves do not pay the factorisation, allocations and graph instantiation
 * again (WD_NO_CTX_POOL disables it).  Not thread-safe per context; the
 * pool itself is.                                                          */
int wd_destroy(wd_ctx* ctx);
/* Bind the caller's state field (in/out), the device history buffer
 * (max_iters doubles, SolveReport.residual_history) and reset the status.
 * Applies the boundary conditions to phi (solver.py:235-236).             */
int wd_bind(wd_ctx* ctx, double* phi_dev, double* history_dev);
/* Enqueue k pseudo-steps (solver.py:249-272).  Steps after a stop
 * (converged / diverged / max_iters) are no-ops, so the state freezes at
 * the reference's stopping iteration.  Uses a CUDA graph per k.          */
int wd_steps(wd_ctx* ctx, int k);
/* Copy the device status to *out (synchronises the stream).              */
int wd_read_status(wd_ctx* ctx, wd_status* out);
/* Async copy of the status word into caller memory (pinned host OK).     */
int wd_status_async(wd_ctx* ctx, wd_status* out_host_pinned);
/* Make the bound phi hold the latest state (after an odd stop).          */
int wd_finish(wd_ctx* ctx);
/* The context's CUDA stream (for event timing by the caller).            */
void* wd_get_stream(wd_ctx* ctx);
/* 1 when a fused (specialised) pseudo-step kernel path is in use.        */
int wd_fused_active(wd_ctx* ctx);
/* Average device time (CUDA events on the context stream) of one kernel of
 * the fused step, run `reps` times on the bound state: kid 1..4 RK stages,
 * 5..7 filter sweeps, 8 change reduction.  Clobbers the workspace; for
 * benchmarking only.                                                     */
int wd_time_kernel(wd_ctx* ctx, int kid, int reps, double* avg_ms);
/* Algorithmic fp64 words per node that kernel `kid` (as above) of the fused
 * step moves (reads + writes of whole fields, halos excluded); 0 when the
 * context has no fused path.  The fast stage kernels run a low-storage RK4
 * (stage words 3 / 5 / 4 / 5 instead of 4 / 6 / 6 / 5).                   */
int wd_kernel_words(wd_ctx* ctx, int kid);

/* ---- operator-level entry points (parity + drop-in operators) -------- */
/* RK4 step solver.py:183-218 (phi_out = BC(filter(RK4(phi_in))))         */
int wd_rk4_step(wd_ctx* ctx, const double* phi_dev, const double* dt_dev, double* out_dev,
                int* diverged_host);
/* tendency formulations.py:244-252                                       */
int wd_tendency(wd_ctx* ctx, const double* phi_dev, double* k_dev);
/* local_timestep solver.py:160-180                                       */
int wd_local_timestep(wd_ctx* ctx, const double* phi_dev, double* dt_dev);
/* apply_boundary_conditions solver.py:87-110 (in place)                 */
int wd_apply_bc(wd_ctx* ctx, double* phi_dev);
/* poisson_postprocess formulations.py:255-270 (+ BC, solver.py:284-285)  */
int wd_poisson_post(wd_ctx* ctx, const double* pp_dev, double* phi_dev);
/* the same map with the boundary conditions optional: apply_bc = 0 is the
 * reference's _l2_vs_exact sampling (solver.py:289-293), which post-maps
 * without re-applying the BCs                                            */
int wd_poisson_map(wd_ctx* ctx, const double* pp_dev, double* phi_dev, int apply_bc);

/* central_derivative operators.py:94-148 (E6/periodic: EXTENSION).
 * offset = coordinate jump per period (coordinate differencing only).    */
int wd_derivative(const double* in_dev, double* out_dev, int ndim, const int* dims, int axis,
                  int scheme, int periodic, double offset, void* stream);
/* fourth_derivative operators.py:236-250                                 */
int wd_fourth_derivative(const double* in_dev, double* out_dev, int ndim, const int* dims,
                         int axis, int periodic, void* stream);
/* apply_filter operators.py:305-352 (pinned may be NULL)                 */
int wd_filter(const double* in_dev, double* out_dev, const unsigned char* pinned_dev, int ndim,
              const int* dims, int axis, double alpha_f, int periodic, void* stream);
/* solve_tridiagonal operators.py:53-78 (LAPACK dgtsv order); host
 * diagonals (n), device rhs (n, nrhs) solved in place.                   */
int wd_solve_tridiagonal(const double* lower, const double* diag, const double* upper,
                         double* rhs_dev, int n, int nrhs, void* stream);
/* compute_metrics grid.py:180-217; coords (d, N) -> metrics (d, d, N),
 * jacobian (N).  periods: (d, d) host array, periods[l*d+m] = jump of x_m
 * across the wrap of periodic axis l (NULL = none).                      */
int wd_compute_metrics(const double* coords_dev, double* metrics_dev, double* jac_dev, int ndim,
                       const int* dims, int scheme, const int* periodic, const double* periods,
                       void* stream);
/* max |a - b| over mask == 0 nodes (mask may be NULL) -> *out_host       */
int wd_linf_delta(const double* a_dev, const double* b_dev, const unsigned char* mask_dev,
                  long long n, double* out_host, void* stream);

/* ---- validation (reference metrics.py) ---------------- */
/* metrics.py:20-34 sampled_wall_distance: out[i] = min_m |p_i - w_m|,
 * points (n, d) and wall samples (m, d) row-major, d <= 3; bit-identical
 * to the reference's numpy evaluation.                                   */
int wd_sampled_wall_distance(const double* points_dev, long long n, const double* wall_dev,
                             long long m, int d, double* out_dev, void* stream);
/* metrics.py:54-66 l2_norm: sqrt(sum (1/J) (phi - exact)^2); jac_dev NULL
 * -> the constant jac_const.  Deterministic reduction -> *out_host.       */
int wd_l2_norm(const double* phi_dev, const double* exact_dev, const double* jac_dev,
               double jac_const, long long n, double* out_host, void* stream);
/* metrics.py:121-124 gradient_magnitude: |grad phi| = sqrt(sum_m U_m^2)
 * with the context's (central) scheme and metrics.                       */
int wd_gradient_magnitude(wd_ctx* ctx, const double* phi_dev, double* out_dev);
/* levelset.py:169-202 levelset_step: one RK4 step of
 * d phi_s / dt = source - F |grad phi_s| with zero-gradient (far-field)
 * faces; the context is created with every face far-field.               */
int wd_levelset_step(wd_ctx* ctx, const double* phi_dev, double* out_dev, double F, double dt,
                     double source);

/* levelset.py:214-318 extract_isolines, the per-cell part: marching-squares
 * segments of a 2-D (n0, n1) field at `level`, coords (2, n0 n1).  Per cell
 * c = i (n1 - 1) + j: count[c] in 0..2 segments; ids[4 c + 2 s + e] the cell
 * edge of endpoint e of segment s (2 * node + 0: edge towards i + 1, + 1:
 * towards j + 1); pts[8 c + 4 s + 2 e ..] its interpolated (x, y).  The host
 * chains segments through shared edge ids.                                */
int wd_iso_segments(const double* field_dev, const double* coords_dev, int n0, int n1,
                    double level, int* count_dev, long long* ids_dev, double* pts_dev,
                    void* stream);

/* One implicit-filter sweep (operators.py:305-352) of the fused path's
 * kernels along `axis` of an arbitrary (n0, n1, n2) array; with A_dev the
 * sweep also accumulates max|out - A|, max|out| and the non-finite flag into
 * the status word, readable with wd_status_maxima (int64 x 3: the two maxima
 * as order-preserving bit patterns).  Operator-level parity entry points. */
int wd_fused_filter(wd_ctx* ctx, int axis, const double* in_dev, double* out_dev, int n0, int n1,
                    int n2, int periodic, const double* A_dev);
int wd_status_maxima(wd_ctx* ctx, long long* dev3);

/* ---- multi-GPU: slab decomposition along axis 0 (EXTENSION) --
 * One process per GPU.  The reference has no distributed path; these entry
 * points put its solve loop (solver.py:221-286) on P ranks that each own the
 * planes [rank n0/P, (rank+1) n0/P) of the PERIODIC axis 0.  Explicit
 * stencils exchange ghost planes (NCCL send/recv over NVLink) per RK stage;
 * compact derivatives, the filter and the other line operators ALONG axis 0
 * run on pencils between two all_to_all transposes (operators.py:130-148,
 * 305-352 see whole lines), or -- fast arithmetic on the fused path -- as a
 * partitioned solve with one all_gather of per-line carries; the stop test
 * (solver.py:253-272) all_reduces (max) three words per step.  Results:
 * bit-identical to one GPU with transposes, round-off level with the
 * partitioned filter.                                                      */
typedef struct wd_comm wd_comm;
typedef struct wd_dist wd_dist;
#define WD_NCCL_ID_BYTES 128
#define WD_DECOMP_SLAB0 0        /* contiguous slabs of axis 0              */
#define WD_FILTER0_AUTO (-1)     /* partitioned if arith = fast, else transpose */
#define WD_FILTER0_PARTITIONED 0
#define WD_FILTER0_TRANSPOSE 1
/* rank 0: a fresh NCCL unique id (128 bytes) to hand to every rank        */
int wd_comm_unique_id(void* id_out);
/* wd_comm_init(nccl_id, rank, nranks, decomposition).  Call
 * with the rank's device current; collective over the ranks.  nranks == 1
 * needs no id and no NCCL.                                                 */
int wd_comm_init(const void* nccl_id, int rank, int nranks, int decomposition, wd_comm** out);
/* The same four collectives through host callbacks (another transport, or P
 * logical ranks in one process, for tests): each gets device pointers and
 * the stream the operation must be ordered on, returns 0 on success.  Not
 * CUDA-graph capturable.                                                   */
typedef struct wd_comm_callbacks {
  void* user;
  /* ghost planes of a (nl + 2G) x plane slab: [nl, nl+G) -> right rank's
   * [0, G), [G, 2G) -> left rank's [nl+G, nl+2G)                           */
  int (*halo)(void* user, double* slab_dev, long long plane, int nl, int G, void* stream);
  /* all[q * count ..] <- rank q's mine[0 .. count)                         */
  int (*allgather)(void* user, const double* mine_dev, double* all_dev, long long count,
                   void* stream);
  /* recv[q * count ..] <- rank q's send[my_rank * count ..]                */
  int (*alltoall)(void* user, const double* send_dev, double* recv_dev, long long count,
                  void* stream);
  /* element-wise max of n int64 words over the ranks, in place             */
  int (*allreduce_max)(void* user, long long* buf_dev, int n, void* stream);
} wd_comm_callbacks;
int wd_comm_init_callbacks(const wd_comm_callbacks* cb, int rank, int nranks, wd_comm** out);
/* One rank of an nranks-way decomposition run ALONE (benchmarking): its slab
 * wraps onto itself, collectives are device copies of the real volume.     */
int wd_comm_init_solo(int rank, int nranks, wd_comm** out);
/* all[q * count ..] <- rank q's mine[0 .. count) (collecting the slabs of
 * a result)                                                                */
int wd_comm_allgather(wd_comm* comm, const double* mine_dev, double* all_dev, long long count,
                      void* stream);
int wd_comm_destroy(wd_comm* comm);
/* Decomposed solver context.  `grid` describes the GLOBAL grid (dims, faces,
 * spacing); metrics_dev / solid_mask_dev point at this rank's slab
 * ((d, d, nl n1 n2) and (nl n1 n2)).  filter0: WD_FILTER0_*; overlap: run
 * interior planes while ghost planes are in flight (fused path, NCCL).     */
int wd_dist_create(wd_comm* comm, const wd_grid_desc* grid, const wd_solver_desc* solver,
                   int filter0, int overlap, wd_dist** out);
int wd_dist_destroy(wd_dist* d);
/* phi_dev: this rank's (nl, n1[, n2]) slab (in/out); history as wd_bind    */
int wd_dist_bind(wd_dist* d, double* phi_dev, double* history_dev);
/* k pseudo-steps; with an NCCL communicator one CUDA graph per k holds the
 * kernels AND the collectives, frozen in-device at the stop               */
int wd_dist_steps(wd_dist* d, int k);
int wd_dist_read_status(wd_dist* d, wd_status* out);
/* the bound slab holds the latest state afterwards                         */
int wd_dist_finish(wd_dist* d);
void* wd_dist_stream(wd_dist* d);
/* the rank's local solver context (operator-level calls on the slab; the
 * axis-0 operators of a GENERIC-program context are collective)            */
wd_ctx* wd_dist_context(wd_dist* d);
/* out8 = {nl, G, fused, filter0, overlap, graph, nranks, rank}             */
int wd_dist_info(wd_dist* d, int* out8);

#ifdef __cplusplus
}
#endif

#endif /* WALLDIST_B200_H */
