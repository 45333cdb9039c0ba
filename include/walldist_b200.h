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

/* ---- slab decomposition (EXTENSION; paper_2111_09859_b200/dist.py) ----
 * The context is created for a rank's ghosted slab (nl + 2G, n1, n2) with
 * axis 0 non-periodic; the host exchanges ghost planes between stages and
 * transposes slab <-> pencil around the axis-0 filter (all_to_all), so the
 * per-node and per-line arithmetic equals the single-GPU path exactly.   */
/* stages update planes [i_lo, i_hi) only (the slab interior)             */
int wd_dist_configure(wd_ctx* ctx, int i_lo, int i_hi);
/* one RK stage (1..4): out = stage(p) with phi0 = A (all ghosted)        */
int wd_dist_stage(wd_ctx* ctx, int stage, const double* A_dev, const double* p_dev,
                  double* out_dev);
/* implicit-filter sweep along `axis` of an (n0, n1, n2) array; with A_dev
 * the sweep also accumulates max|out - A|, max|out| into the status     */
int wd_dist_filter(wd_ctx* ctx, int axis, const double* in_dev, double* out_dev, int n0, int n1,
                   int n2, int periodic, const double* A_dev);
/* slab (nl, n1, n2) <-> all_to_all buffer (P, nl, n1/P, n2)              */
int wd_dist_pack(const double* slab_dev, double* buf_dev, int nl, int n1, int n2, int P,
                 void* stream);
int wd_dist_unpack(const double* buf_dev, double* slab_dev, int nl, int n1, int n2, int P,
                   void* stream);
/* status maxima -> dev3 (int64 x3) for all_reduce(max); then finalize    */
/* Partitioned axis-0 filter (fast arithmetic; wd_dist_filter0.cuh): the
 * rank's rows [rank nl, (rank+1) nl) of the n0-long periodic lines, three
 * phases around two all_gathers of per-line carries.  in: ghosted slab
 * (nl + 2G, n1, n2), G >= 5 ghosts filled; out: interior (nl, n1, n2).
 * phase 1 writes mine[2][n1 n2] (Y_blk, h.rhs); phase 2 reads xa =
 * gathered phase-1 slots [P][2][n1 n2], writes out (x') and mine[n1 n2]
 * (X_blk); phase 3 reads xa and xb = gathered phase-2 slots [P][n1 n2].   */
int wd_dist_filter0(wd_ctx* ctx, int phase, const double* in_dev, double* out_dev, int n0,
                    int n1, int n2, int G, int P, int rank, const double* xa_dev,
                    const double* xb_dev, double* mine_dev);
int wd_dist_stats(wd_ctx* ctx, long long* dev3);
int wd_dist_finalize(wd_ctx* ctx, const long long* dev3);

#ifdef __cplusplus
}
#endif

#endif /* WALLDIST_B200_H */
