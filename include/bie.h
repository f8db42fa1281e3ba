/*
 * bie.h -- C ABI of libbie.so, the B200 (sm_100a) hot path of the
 * boundary-integral GMRES method of arxiv 1609.04484 (2D Stokes flow in
 * porous media), scoped per SURVEY.md s8:
 *   completed double-layer (DLP) matvec  -> bie_dlp_apply
 *   block-diagonal (BD) preconditioner   -> bie_blockdiag_factor / _apply
 *   left-preconditioned full GMRES       -> bie_gmres_solve
 *
 * Citations: P:l.N = PAPER.md line N (arxiv 1609.04484 LaTeX body); readings
 * C1..C26 are listed in DESIGN.md s3.
 *
 * Conventions for every call:
 *  - Returns BIE_OK (0) or a negative BIE_E* code; bie_last_error() returns a
 *    thread-local message describing the last failure on the calling thread.
 *  - "device" pointers are CUDA device (or managed) memory owned by the caller
 *    (e.g. torch.Tensor.data_ptr()); "host" pointers are ordinary host memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Calls documented "async" only enqueue work on that stream.
 *  - All floating point is IEEE FP64.  Vectors of unknowns are interleaved
 *    (sigma_x, sigma_y) per node, 2N doubles per vector, in dof order:
 *    pore 1 nodes, ..., pore M nodes, then the outer wall Gamma_0
 *    (P:l.734-736: "the first 2x128x22 dofs" are the pores).  A batch of
 *    nvec vectors is [nvec][2N], vector-major.
 *  - One geometry handle owns one workspace: calls that use the same
 *    geometry (or a blockdiag built from it) must be serialised on one stream.
 */
#ifndef BIE_H
#define BIE_H

#ifdef __cplusplus
extern "C" {
#endif

#define BIE_OK 0
#define BIE_EINVAL (-1)     /* bad argument, null handle, wrong handle kind */
#define BIE_EGEOM (-2)      /* invalid geometry (pore radius <= 0, ...) */
#define BIE_ESINGULAR (-3)  /* a BD block has a zero pivot (S:l.386: fail loudly) */
#define BIE_ECUDA (-4)      /* CUDA launch/runtime error */
#define BIE_ENOMEM (-5)     /* device or host allocation failed */
#define BIE_ECHECK (-6)     /* checked build: corrupted allocation canary or failed device bounds check */

/* bie_dlp_apply flags */
#define BIE_FULL 0u    /* -1/2 I + D + self term + N0 + pore completion (reading C5/C6) */
#define BIE_D_ONLY 1u  /* PV trapezoid DLP sum + self term only (Gauss-identity pins) */
#define BIE_ONE_SIDED 2u /* force the one-sided all-pairs kernel even where the symmetric
                            (pair-reusing) kernel applies (A/B measurement; same result to rounding) */

#define BIE_MAX_NVEC 16

#if defined(__GNUC__)
#define BIE_API __attribute__((visibility("default")))
#else
#define BIE_API
#endif

typedef struct bie_geometry_s *bie_geometry_t;
typedef struct bie_blockdiag_s *bie_blockdiag_t;

/*
 * bie_geometry_create -- A1: derive the node table on the
 * device and allocate the matvec workspace.
 *   P:l.191-204 (Gamma_0 = mollified rectangle, pores = circles),
 *   P:l.296-309 (collocation at N = M N_int + N_ext points),
 *   P:l.318-319, P:l.354 (w_j = arclength element x trapezoid weight).
 * Inputs (host):
 *   outer_xy, outer_dxy, outer_ddxy : [n_outer][2] samples x(t_j), x'(t_j),
 *       x''(t_j) of the outer wall at t_j = j*outer_period/n_outer, CCW.
 *   pore_c : [n_pores][2] centres, pore_r : [n_pores] radii (> 0).
 *   nodes_per_pore : N_int; pore node j at theta_j = 2 pi j/N_int (C12).
 * Derived per node: w = |x'| T/n (C7); t = x'/|x'|; n = out of the fluid
 * domain (C2): (t_y,-t_x) on Gamma_0, -(cos,sin) on pores; kappa_n =
 * x''.n/|x'|^2.  The handle owns all device data; destroy frees it.
 * Errors: BIE_EINVAL (null pointer, n_outer or nodes_per_pore < 16 or odd
 * (S:l.55-57), n_pores < 0, outer_period <= 0), BIE_EGEOM (radius <= 0,
 * non-finite input, overlapping pores, a pore crossing or outside the outer
 * wall -- S:l.36), BIE_ENOMEM, BIE_ECUDA.  Synchronous.
 */
BIE_API int bie_geometry_create(const double *outer_xy, const double *outer_dxy, const double *outer_ddxy,
                        int n_outer, double outer_period, const double *pore_c, const double *pore_r,
                        int n_pores, int nodes_per_pore, bie_geometry_t *out);
BIE_API int bie_geometry_destroy(bie_geometry_t g);
/* N = number of nodes (2N unknowns), M = number of pores. */
BIE_API int bie_geometry_info(bie_geometry_t g, int *N, int *M);
/* Copy node positions to host: pos_host [N][2]. Synchronous. */
BIE_API int bie_geometry_nodes(bie_geometry_t g, double *pos_host);
/*
 * bie_geometry_node_table -- copy the whole A1 node table to host buffers:
 * pos, nrm, tan [N][2], w [N], kappa [N] (kappa_n = x''.n/|x'|^2).  The table
 * is uniquely defined by the inputs (reading C27: correctly rounded pore
 * template, one fixed sequence of IEEE operations per quantity, no FMA
 * contraction), so any implementation of the same formulas reproduces it bit
 * for bit.  Errors: BIE_EINVAL (bad handle / null), BIE_ECUDA.  Synchronous.
 */
BIE_API int bie_geometry_node_table(bie_geometry_t g, double *pos, double *nrm, double *tan, double *w,
                                    double *kappa);
/*
 * bie_pore_template -- host-only (no device needed): unit[j] = (cos, sin) of
 * theta_j = 2 pi j / n, j < n, each CORRECTLY ROUNDED to double (reading C27 of
 * DESIGN.md; exact octant reduction of j, double-double Taylor series, one
 * rounding).  Pore node j of pore (c, r) is x = c + r unit[j] (P:l.191-204,
 * C12).  unit: host [n][2].  Errors: BIE_EINVAL (null, n < 1).
 */
BIE_API int bie_pore_template(int n, double *unit);

/*
 * bie_dlp_apply -- A2-A5: out = A sigma for nvec densities (async on stream).
 *   y_i = -1/2 sigma_i                                        (jump, C3)
 *       + sum_{j != i} (w_j/pi)(r.n_j)(r.sigma_j) r / rho^4    (P:l.243-248, trapezoid P:l.310-319)
 *       + (w_i/2pi) kappa_n,i (t_i.sigma_i) t_i                (diagonal limit, C4)
 *       + [i in Gamma_0] nu n_i                                (N0 term, C5)
 *       + sum_k Stokeslet(x_i-c_k) lambda_k + r_k rotlet(x_i-c_k) mu_k   (completion, C5;
 *         forms of P:l.944-948)
 *   r = x_i - x_j, rho = |r|; moments lambda_k, mu_k, nu as in DESIGN.md s2.
 * sigma, out : device [nvec][2N]; out must not alias sigma.
 * nvec in [1, BIE_MAX_NVEC].  flags: BIE_FULL or BIE_D_ONLY.
 * Errors: BIE_EINVAL (null, nvec out of range, out == sigma, bad flags),
 * BIE_ECUDA (launch error; asynchronous faults surface at the next sync).
 * Does not synchronise, except when the geometry's workspace is allocated or
 * grown (the first symmetric-path apply, or the first apply with a larger
 * nvec / row range), which allocates it synchronously.
 */
BIE_API int bie_dlp_apply(bie_geometry_t g, const double *sigma, double *out, int nvec, unsigned flags, void *stream);

/*
 * bie_dlp_apply_rows -- same operator restricted to target nodes
 * [row_begin, row_end) (row sharding).  sigma is the full
 * [nvec][2N] density; out is [nvec][2*(row_end-row_begin)].  Async.
 */
BIE_API int bie_dlp_apply_rows(bie_geometry_t g, const double *sigma, double *out, int nvec, unsigned flags,
                       int row_begin, int row_end, void *stream);

/*
 * bie_dlp_apply_host -- end-to-end variant: sigma_host / out_host are HOST
 * buffers [nvec][2N] (pinned for full speed, pageable accepted).  Copies
 * H2D, applies, copies D2H and synchronises the stream before returning.
 */
BIE_API int bie_dlp_apply_host(bie_geometry_t g, const double *sigma_host, double *out_host, int nvec, unsigned flags,
                       void *stream);

/*
 * bie_field_eval -- SURVEY s8(f) NEXT-2: off-surface velocity from a density,
 *   u(x) = sum_j (w_j/pi)(r.n_j)(r.sigma_j) r / rho^4                 (P:l.243-246 kernel,
 *        + sum_k Stokeslet(x-c_k) lambda_k + r_k rotlet(x-c_k) mu_k     trapezoid rule P:l.346-354,
 *   r = x - x_j                                                         completion C5)
 * i.e. the representation whose boundary limit bie_dlp_apply discretises (no
 * jump, no self term, no N0).  Spectrally accurate for d(x, Gamma) > sqrt(ds)
 * (P:l.356-358 footnote); no near-field correction (C18).
 * sigma : device [2N];  targets : device [ntgt][2];  out : device [ntgt][2].
 * Async on stream.  Errors: BIE_EINVAL (null, ntgt < 0, out aliasing sigma), BIE_ECUDA.
 */
BIE_API int bie_field_eval(bie_geometry_t g, const double *sigma, const double *targets, int ntgt, double *out,
                           void *stream);

/*
 * bie_blockdiag_factor -- A6: block-diagonal preconditioner, P:l.651-657
 * ("diagonal blocks corresponding to the self-interactions of the individual
 * pores and the outer boundary ... assembled, factorized, and inverted
 * exactly").  Block b = rows/cols of the completed operator on body b (pore
 * blocks include their own Stokeslet/rotlet columns; the Gamma_0 block
 * includes N0).  Each block is inverted explicitly by Gauss-Jordan
 * elimination with partial pivoting (row of max |.|).  The handle owns the
 * inverses (sum_b (2 n_b)^2 doubles of device memory).
 * Synchronises `stream` once to read the pivot status.  Blocks of order >= 4096
 * (the wall) are factored on `stream` plus one internal high-priority stream owned
 * by the geometry (fork/join by events; the call waits for that stream before it
 * returns), so `stream` must not be in capture mode.
 * Errors: BIE_ESINGULAR (message names the body), BIE_ENOMEM, BIE_ECUDA, BIE_EINVAL.
 */
BIE_API int bie_blockdiag_factor(bie_geometry_t g, bie_blockdiag_t *out, void *stream);
/* A7: out_b = B_b^{-1} in_b for every body, nvec vectors, device [nvec][2N]; async; in != out. */
BIE_API int bie_blockdiag_apply(bie_blockdiag_t bd, const double *in, double *out, int nvec, void *stream);
BIE_API int bie_blockdiag_destroy(bie_blockdiag_t bd);
/* Copy the explicit inverse of body b ([2n_b][2n_b] row-major) to host (test hook). Synchronous. */
BIE_API int bie_blockdiag_block_inverse(bie_blockdiag_t bd, int body, double *host, long long host_len);

/*
 * bie_gmres_solve -- A8/A9: left-preconditioned full GMRES (no restart),
 * x0 = 0, CGS2 orthogonalisation, Givens rotations (reading C13), tolerance on
 * the preconditioned relative residual estimate |g_{k+1}|/||P^{-1} f||
 * (P:l.596-601, P:l.661-663, P:l.678-681).  bd == NULL -> no preconditioner.
 *   f, x : device [2N] (x is written).
 *   hist_host : host [max_iter+1]; hist_host[0..*iters] = estimates (hist[0] = 1).
 *   iters, converged : host outputs (converged = 0 at the iteration cap, S:l.376;
 *     happy breakdown counts as converged, S:l.377).
 *   res_pc, res_true : host outputs ||P^{-1}(f-Ax)||/||P^{-1}f|| and ||f-Ax||/||f||
 *     (P:l.678-686), from one extra matvec at the end.
 * The Krylov basis lives in device memory: (max_iter+1)*2N doubles.
 * Synchronises once per iteration (8-byte D2H of the estimate).
 * Errors: BIE_EINVAL, BIE_ENOMEM (basis allocation), BIE_ECUDA.
 */
BIE_API int bie_gmres_solve(bie_geometry_t g, bie_blockdiag_t bd, const double *f, double *x, double tol, int max_iter,
                    double *hist_host, int *iters, double *res_pc, double *res_true, int *converged,
                    void *stream);
/*
 * bie_gmres_solve_host -- bie_gmres_solve with HOST buffers (the end-to-end
 * call): f_host [2N] is copied to a device staging buffer owned
 * by the geometry, solved on the device, and x_host [2N] receives the solution.
 * Pinned (cudaHostAlloc / torch pin_memory) buffers give async DMA copies on
 * `stream`; pageable buffers also work.  Same outputs, bars and errors as
 * bie_gmres_solve (+ BIE_EINVAL for f_host == x_host).  Synchronous: returns
 * after x_host is written.  Not re-entrant per geometry (shared staging).
 */
BIE_API int bie_gmres_solve_host(bie_geometry_t g, bie_blockdiag_t bd, const double *f_host, double *x_host,
                                 double tol, int max_iter, double *hist_host, int *iters, double *res_pc,
                                 double *res_true, int *converged, void *stream);

/*
 * bie_gmres_solve_batch -- SURVEY s8(f) NEXT-3: nrhs independent left-
 * preconditioned GMRES solves (same algorithm and stopping rule as
 * bie_gmres_solve, one Krylov basis per right-hand side) whose operator
 * applications are batched: every iteration applies A and P^{-1} to the
 * current basis vectors of all still-active systems in one nvec-wide call
 * (BIE_MAX_NVEC per chunk).  A system leaves the batch when it converges.
 *   F, X      : device [nrhs][2N].
 *   hist_host : host [nrhs][max_iter+1];  iters, converged : host [nrhs];
 *   res_pc, res_true : host [nrhs].
 * nrhs in [1, 64].  Device memory: nrhs (max_iter+1) 2N doubles for the bases.
 * Errors: as bie_gmres_solve.
 */
BIE_API int bie_gmres_solve_batch(bie_geometry_t g, bie_blockdiag_t bd, const double *F, double *X, int nrhs,
                                  double tol, int max_iter, double *hist_host, int *iters, double *res_pc,
                                  double *res_true, int *converged, void *stream);

/*
 * Row sharding: a rank owns the nodes of a
 * contiguous body range.  bie_blockdiag_factor_range factors only bodies
 * [body_begin, body_end) (pores 0..M-1, wall M); its bie_blockdiag_apply then
 * takes LOCAL vectors [nvec][2 (row_end - row_begin)] for the node range that
 * bie_blockdiag_rows reports.  Such a handle is rejected by bie_gmres_solve*.
 */
BIE_API int bie_blockdiag_factor_range(bie_geometry_t g, int body_begin, int body_end, bie_blockdiag_t *out,
                                       void *stream);
BIE_API int bie_blockdiag_rows(bie_blockdiag_t bd, int *row_begin, int *row_end);

/*
 * Sharded symmetric matvec, nvec = 1.  The all-pairs work of
 * the symmetric kernel is a triangular list of `units` (512-node block x
 * 32-node chunk after it) plus `blocks` in-block diagonal tiles
 * (bie_dlp_sym_info).  bie_dlp_pairs_partial computes the pair sums
 * sum_{j != i} (w_j/pi)(r.n_j)(r.sigma_j) r/rho^4 restricted to units
 * [unit_begin, unit_end) and diagonal blocks [block_begin, block_end) into a
 * FULL output out_full [2N] (both directions of every pair in the slice); the
 * ranks' vectors sum (e.g. NCCL reduce-scatter) to the complete pair sum.
 * bie_dlp_epilogue_rows then adds the local terms of the operator (jump, self,
 * N0, completion -- BIE_FULL; self only -- BIE_D_ONLY) for rows
 * [row_begin, row_end): out_rows = pairsum_rows + local terms, both [2 rows].
 * sigma is the full density [2N].  Async on stream.
 */
BIE_API int bie_dlp_sym_info(bie_geometry_t g, long long *units, int *blocks);
BIE_API int bie_dlp_pairs_partial(bie_geometry_t g, const double *sigma, double *out_full, long long unit_begin,
                                  long long unit_end, int block_begin, int block_end, void *stream);
BIE_API int bie_dlp_epilogue_rows(bie_geometry_t g, const double *sigma, const double *pairsum_rows,
                                  double *out_rows, int row_begin, int row_end, unsigned flags, void *stream);

/*
 * Krylov building blocks for a row-sharded GMRES (the kernels bie_gmres_solve
 * uses; a multi-rank driver adds only the collectives).  All device pointers,
 * async on stream; reading C13 conventions:
 *   dots     : out[j] = sum_e V[j*ldv + e] w[e], j < nv (local partial; fixed-order two-stage reduction)
 *   axpy     : y = beta y + alpha sum_j c[j] V[j*ldv + .]   (c on the device)
 *   scale    : y = x / s[0]                                  (s on the device, a norm)
 *   sqrt     : out[i] = sqrt(in[i]), i < n
 *   givens   : Hessenberg column k = h + h2 with H[k+1,k] = scal[2]; applies the previous
 *              rotations, forms rotation k, updates g; scal[0] = beta, scal[1] = ||P^-1 A v_k||,
 *              scal[2] = ||w|| after CGS2; writes scal[3] = |g[k+1]|/beta, scal[4] = breakdown flag.
 *              H is column-major with leading dimension ldh.
 *   trisolve : y = H[0:iters,0:iters]^{-1} g (upper triangular).
 */
BIE_API int bie_krylov_dots(const double *V, long long ldv, int nv, const double *w, long long n, double *out,
                            void *stream);
BIE_API int bie_krylov_axpy(const double *V, long long ldv, int nv, const double *c, double alpha, double beta,
                            double *y, long long n, void *stream);
BIE_API int bie_krylov_scale(const double *x, const double *s, double *y, long long n, void *stream);
BIE_API int bie_krylov_sqrt(const double *in, double *out, int n, void *stream);
BIE_API int bie_krylov_givens(double *H, int ldh, double *cs, double *sn, double *g, const double *h,
                              const double *h2, int k, double *scal, void *stream);
BIE_API int bie_krylov_trisolve(const double *H, int ldh, const double *g, double *y, int iters, void *stream);

BIE_API const char *bie_last_error(void);

/*
 * Measurement hooks (bench.py; not needed for computing).
 * bie_profile_begin: from now on every bie_dlp_apply* on g records CUDA events
 *   on its stream around its three phases (moments | all-pairs | epilogue).
 * bie_profile_end: synchronises those events, returns the summed durations in
 *   milliseconds and the number of applies recorded, and stops recording.
 * bie_launch_count: number of kernels this library has launched in the
 *   process so far (monotone counter; take differences).
 */
BIE_API int bie_profile_begin(bie_geometry_t g);
BIE_API int bie_profile_end(bie_geometry_t g, double *ms_moments, double *ms_pairs, double *ms_epilogue,
                            int *applies);
/*
 * bie_fp64_peak -- measurement hook: runs a DFMA-chain kernel (8 independent
 * chains per thread, 8 x 256-thread CTAs per SM) for `iters` iterations on
 * `stream` and returns the achieved FP64 rate (tflops, 2 flop per DFMA) and
 * its duration (ms, CUDA events).  The measured denominator of the all-pairs
 * roofline.  Errors: BIE_EINVAL, BIE_ECUDA.  Synchronous.
 */
BIE_API int bie_fp64_peak(int iters, double *tflops, double *ms, void *stream);
BIE_API long long bie_launch_count(void);

/*
 * bie_debug_check -- verification hook of the checked build
 * (lib/libbie_checked.so, compiled with -DBIE_CHECKED), the
 * stand-in for compute-sanitizer memcheck on a pool that does not allow it:
 * synchronises the device, verifies the 256-byte canaries on both sides of
 * every live library allocation (and of every allocation freed since the last
 * call) and reads the device-side bounds-check flags.  *checked_allocs = the
 * number of live allocations verified (-1 in the normal build, which checks
 * nothing and returns BIE_OK); *dcheck_line = source line of the first failed
 * device check (0 if none).  Errors: BIE_ECHECK (message names the
 * violation), BIE_EINVAL (null output), BIE_ECUDA.
 */
BIE_API int bie_debug_check(int *checked_allocs, int *dcheck_line);

/*
 * bie_blockdiag_factor_structured -- NEXT-4: the same BD
 * preconditioner as bie_blockdiag_factor with structured pore blocks.  For
 * equispaced circular pores of equal n_p the completed-DLP blocks differ only
 * by the Stokeslet's -log r_k term (pin V10):
 *   B_k = B_0 + c_k (1 1^T (x) I_2),  c_k = (log r_0 - log r_k) / (4 pi n_p),
 * so one exact inverse X = B_0^-1 plus a rank-2 Woodbury term per pore gives
 * every B_k^-1 (P:l.655-657 footnote: the pore blocks need not be factorised
 * one by one).  The wall block is inverted exactly as before.  Apply is one
 * GEMM over all pores plus the rank-2 corrections; block_inverse materialises
 * X - W M_k Z on the host.  Same handle semantics and errors as
 * bie_blockdiag_factor (BIE_ESINGULAR for a zero pivot or a singular 2x2
 * Woodbury capacitance, naming the body).
 */
BIE_API int bie_blockdiag_factor_structured(bie_geometry_t g, bie_blockdiag_t *out, void *stream);

/* ---------------------------------------------------------------------------
 * NEXT-1: the paper's own operator, the Stokes single-layer
 * potential with the sixth-order Kapur-Rokhlin correction (P:l.270-330):
 *   (A sigma)_i = sum_{j != i} W_ij G(x_i, x_j) sigma_j,
 *   G(x, y) = (1/4pi)(-log rho I + r r^T / rho^2),  r = x - y    (eq. stokesSLP, eq. dense)
 *   W_ij = w_j (1 + gamma_k) for j on i's own closed curve at periodic offset
 *   +-k, 1 <= k <= 6 ("weights modified at the six nodes to the left and right
 *   of the singularity", P:l.321-325); W_ij = w_j otherwise (readings C24-C26).
 * The same handles, layouts, stream semantics and error codes as the DLP calls.
 * ------------------------------------------------------------------------- */

/* gamma_1..gamma_6 of the Kapur-Rokhlin rule as this library computes them
 * (host, long double; reading C24).  gamma: host double[6].  BIE_EINVAL if null. */
BIE_API int bie_kr_weights(double *gamma);

/*
 * bie_slp_apply -- out = A_SLP sigma.  sigma, out: device [nvec][2N], out must
 * not alias sigma; nvec in [1, BIE_MAX_NVEC]; flags: 0 or BIE_ONE_SIDED
 * (BIE_D_ONLY is rejected).  Async, never synchronises.
 * Errors: BIE_EINVAL (null, nvec, aliasing, flags), BIE_ECUDA, BIE_ENOMEM.
 */
BIE_API int bie_slp_apply(bie_geometry_t g, const double *sigma, double *out, int nvec, unsigned flags, void *stream);

/* Same operator for target rows [row_begin, row_end): out is [nvec][2*(row_end-row_begin)]. */
BIE_API int bie_slp_apply_rows(bie_geometry_t g, const double *sigma, double *out, int nvec, int row_begin,
                               int row_end, void *stream);

/*
 * bie_slp_field_eval -- off-surface velocity u(x) = sum_j w_j G(x, x_j) sigma_j,
 * the trapezoid rule of P:l.346-354 (eq. stokesSLP_discretized), no correction
 * (accurate for d(x, Gamma) > sqrt(ds), P:l.356-358 footnote).
 * sigma: device [2N]; targets: device [ntgt][2]; out: device [ntgt][2]. Async.
 * Errors: BIE_EINVAL (null, ntgt < 0, out aliasing sigma), BIE_ECUDA.
 */
BIE_API int bie_slp_field_eval(bie_geometry_t g, const double *sigma, const double *targets, int ntgt, double *out,
                               void *stream);

/*
 * bie_blockdiag_factor_slp -- the BD preconditioner of the SLP system: exact
 * inverses of the per-body SLP blocks (P:l.651-657 footnote), same object and
 * apply as bie_blockdiag_factor.  The blocks are nearly singular (S n_b = 0,
 * reading C26) but invertible; a zero pivot still raises BIE_ESINGULAR.
 */
BIE_API int bie_blockdiag_factor_slp(bie_geometry_t g, bie_blockdiag_t *out, void *stream);

/*
 * bie_blockdiag_factor_structured_slp -- the same SLP BD preconditioner with
 * the pore blocks inverted through their structure (P:l.655-657 footnote:
 * "accelerated using the FFT").  On a pore of equispaced nodes x_j = c + r
 * (cos, sin)(2 pi j / n) the SLP block satisfies T_i^T B[i][j] T_j = b(j - i),
 * T_j the rotation by 2 pi j / n, so B = D C D^T with C block-circulant; its
 * exact inverse is block-circulant with first block row d(m) (one 2x2 complex
 * inverse per Fourier mode).  Stored per pore: d(m), 4 n doubles.  The wall is
 * inverted exactly as in bie_blockdiag_factor_slp.  Apply, block_inverse and
 * the GMRES calls behave as for bie_blockdiag_factor_slp.  Errors: BIE_EINVAL,
 * BIE_ECUDA, BIE_ESINGULAR (a singular Fourier block or a zero wall pivot).
 */
BIE_API int bie_blockdiag_factor_structured_slp(bie_geometry_t g, bie_blockdiag_t *out, void *stream);

/*
 * bie_gmres_solve_slp / bie_gmres_solve_batch_slp -- bie_gmres_solve and
 * bie_gmres_solve_batch on the SLP system A_SLP sigma = f (P:l.596-601,
 * 661-663).  bd must be NULL or come from bie_blockdiag_factor_slp on g
 * (BIE_EINVAL otherwise).
 */
BIE_API int bie_gmres_solve_slp(bie_geometry_t g, bie_blockdiag_t bd, const double *f, double *x, double tol,
                                int max_iter, double *hist_host, int *iters, double *res_pc, double *res_true,
                                int *converged, void *stream);
BIE_API int bie_gmres_solve_batch_slp(bie_geometry_t g, bie_blockdiag_t bd, const double *F, double *X, int nrhs,
                                      double tol, int max_iter, double *hist_host, int *iters, double *res_pc,
                                      double *res_true, int *converged, void *stream);

/*
 * Row-sharded SLP (NEXT-1 x NEXT-4): the single-layer counterparts of
 * bie_dlp_pairs_partial / bie_dlp_epilogue_rows / bie_blockdiag_factor_range
 * (same slicing, layouts and errors).  bie_slp_pairs_partial
 * writes the all-pairs sums sum_{j != i} w_j G(x_i, x_j) sigma_j of its slice
 * into a full-size vector; bie_slp_epilogue_rows adds the Kapur-Rokhlin
 * corrections of rows [row_begin, row_end) to the reduced pair sums.
 */
BIE_API int bie_slp_pairs_partial(bie_geometry_t g, const double *sigma, double *out_full, long long unit_begin,
                                  long long unit_end, int block_begin, int block_end, void *stream);
BIE_API int bie_slp_epilogue_rows(bie_geometry_t g, const double *sigma, const double *pairsum_rows,
                                  double *out_rows, int row_begin, int row_end, void *stream);
BIE_API int bie_blockdiag_factor_range_slp(bie_geometry_t g, int body_begin, int body_end, bie_blockdiag_t *out,
                                           void *stream);

#ifdef __cplusplus
}
#endif
#endif /* BIE_H */
