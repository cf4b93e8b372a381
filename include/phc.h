/* phc.h — C ABI of the B200 evaluator of a sparse polynomial system and its Jacobian
 * in complex double-double (DD) or quad-double (QD) arithmetic.
 *
 * What is computed (PAPER.md = Verschelde & Yoffe 2011, arXiv 1109.0545):
 *   Y = "the evaluated polynomials ... along with all partial derivatives as needed
 *   in the Jacobian matrix" (Alg. 2 discussion), i.e. for a point x in C^n
 *     F[i]    = f_i(x)        = sum_{t in T_i} c_t prod_j x_{i_{t,j}}^{a_{t,j}}
 *     J[i][v] = df_i/dx_v(x),
 *   by the paper's algorithmic-differentiation scheme for normalised monomials
 *   x_{i_1}^{a_1} ... x_{i_k}^{a_k}, i_1 < ... < i_k, a_j >= 1 (§6):
 *   Speelpenning prefix/suffix products (indices as DESIGN.md reading C1)
 *   over a shared per-point table of variable powers, then the coefficient product
 *   and the sums per polynomial / per Jacobian entry (Alg. 2 "Monomial_Evaluation",
 *   "Coefficient_Product").
 *
 * Number layout.  A complex number is 2*L doubles: L real limbs then L imaginary
 * limbs, limbs non-overlapping and decreasing in magnitude (L = 2: DD, L = 4: QD).
 *   x   : [n_var][2][L]
 *   F   : [n_eq][2][L]
 *   J   : [n_eq][n_var][2][L], row-major, J[i][v] = df_i/dx_v; structural zeros are exact 0.
 *   Batched arrays have a leading [n_points] dimension.
 * Device pointers must be 32-byte aligned (256-bit vector accesses).
 *
 * Errors.  Every int-returning function returns PHC_OK (0) or a negative code and
 * sets a thread-local message readable with phc_last_error().  Non-finite inputs x
 * are not checked on the hot path: NaN/Inf propagate into F and J.
 *
 * Ordering.  Device-pointer calls are asynchronous on the caller's stream
 * (cudaStream_t passed as void*; NULL = legacy default stream): they return once
 * the work is enqueued.  Kernel faults surface at the caller's next synchronisation.
 * A handle owns per-stream-agnostic scratch: do not run two eval calls of the same
 * handle concurrently on different streams (calls on one stream are fine).
 *
 * Determinism.  For a given system and point the results are bitwise reproducible:
 * every sum is taken in a fixed order, independent of the launch configuration and of
 * the device list or chunking of a batch call.  Two regimes exist per system (DESIGN.md
 * reading N2-2): calls whose total point count times the number of terms is at most
 * 148 * 32 take the latency path (one warp per term for DD, a segment of G lanes per
 * term for QD; phc_system_stats out[15..17]), larger calls the batch kernels; the regime
 * is chosen from the call's total point count, each regime is deterministic, and the two
 * agree within the DD/QD tolerance (not bitwise).
 *
 * Precision.  Results are within 1e-28 (DD) / 1e-60 (QD) of the exact values, normwise
 * (BASELINE.json north_star).  The QD kernels keep intermediate products and sums as
 * unnormalised level expansions and renormalise what they store (reading R4):
 * measured errors ~3e-62 on the largest config.
 */
#ifndef PHC_H
#define PHC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PHC_OK = 0,
  PHC_EINVAL = -1,       /* invalid argument or malformed system */
  PHC_ENOMEM = -2,       /* device or host allocation failed */
  PHC_ECUDA = -3,        /* a CUDA runtime call or kernel launch failed */
  PHC_EUNSUPPORTED = -4  /* valid but beyond the compiled limits (see below) */
};

/* Compiled limits: limbs in {2, 4}; factors per term k <= PHC_MAX_K; exponents <= PHC_MAX_EXP;
 * n_var <= PHC_MAX_VARS. */
#define PHC_MAX_K 64
#define PHC_MAX_EXP 255
#define PHC_MAX_VARS 65534

typedef struct phc_system phc_system; /* opaque; owned by the library */

/* Create a system handle on CUDA device `device` (the "home" device).
 *   n_eq, n_var >= 1;  limbs = 2 (complex DD) or 4 (complex QD).
 *   poly_ptr [n_eq+1]     CSR over terms: polynomial i owns terms poly_ptr[i] .. poly_ptr[i+1]-1;
 *                         poly_ptr[0] = 0, non-decreasing, poly_ptr[n_eq] = n_terms.
 *   term_ptr [n_terms+1]  CSR over factors: term t owns factors term_ptr[t] .. term_ptr[t+1]-1;
 *                         term_ptr[0] = 0, non-decreasing. k = 0 is a constant term.
 *   var_idx  [n_factors]  0-based variable of each factor, strictly increasing within a term
 *                         (normalised monomial).
 *   exponent [n_factors]  a_j >= 1.
 *   coeff    [n_terms][2][limbs]  c_t, finite limbs.
 * All array pointers are HOST pointers; they are deep-copied (the caller keeps ownership).
 * Duplicate terms within a polynomial are allowed and summed.
 * Returns PHC_EINVAL on malformed input, PHC_EUNSUPPORTED beyond the compiled limits. */
int phc_system_create(phc_system** out, int32_t n_eq, int32_t n_var, int32_t limbs, int64_t n_terms,
                      const int64_t* poly_ptr, const int64_t* term_ptr, const int32_t* var_idx,
                      const int32_t* exponent, const double* coeff, int32_t device);

/* Release the handle and every device buffer it owns (all devices). NULL is a no-op. */
void phc_system_destroy(phc_system* s);

/* One point on the home device.  x, f, jac: device pointers on the home device
 * (layouts above); f and jac are written in full and must not alias x. */
int phc_eval_jacobian(const phc_system* s, const double* x, double* f, double* jac, void* stream);

/* n_points points.  x [n_points][n_var][2][L], f [n_points][n_eq][2][L],
 * jac [n_points][n_eq][n_var][2][L]: device pointers on the home device.
 * devices[0..n_devices-1]: CUDA devices to shard the points over (contiguous, equal
 * ranges; repeats allowed, e.g. {0,0,0,0}, for testing the shard bookkeeping on one GPU);
 * devices = NULL or n_devices = 0 means {home}.  Inputs are scattered and outputs
 * gathered over NVLink peer copies; every device's work is ordered after the work
 * already enqueued on `stream`, and `stream` waits for the gather.  Results are
 * bitwise identical for every device list. */
int phc_eval_jacobian_batch(const phc_system* s, int64_t n_points, const double* x, double* f, double* jac,
                            const int32_t* devices, int32_t n_devices, void* stream);

/* Points [p_begin, p_end) of an n_points-point batch call -- the same Y (the polynomials and
 * all partial derivatives) as phc_eval_jacobian_batch -- evaluated on the handle's
 * home device and written into the FULL output arrays: x [n_points][n_var][2][L] (only rows
 * p_begin .. p_end-1 are read), f [n_points][n_eq][2][L], jac [n_points][n_eq][n_var][2][L]
 * (only those rows are written).  The evaluation regime is that of the whole n_points call,
 * so the rows are bitwise those phc_eval_jacobian_batch writes for all n_points: a batch
 * split over processes (one per GPU, BASELINE.json configs[3] "points sharded across
 * 1/2/4/8 GPUs") gives the unsharded result.  f and jac may be peer memory
 * of another device or process (phc_ipc_open): the kernels then store the rows straight into
 * that device's buffers over NVLink -- the final gather fused into the evaluation.  x must be
 * readable from the home device.  Asynchronous on `stream`; PHC_EINVAL unless
 * 0 <= p_begin <= p_end <= n_points. */
int phc_eval_jacobian_batch_range(const phc_system* s, int64_t n_points, int64_t p_begin, int64_t p_end,
                                  const double* x, double* f, double* jac, void* stream);

/* CUDA IPC for the multi-process gather (one process per GPU).  phc_ipc_get_handle describes
 * the device allocation containing dev_ptr: a PHC_IPC_HANDLE_BYTES-byte handle to send to
 * another process, and the byte offset of dev_ptr inside that allocation.  phc_ipc_open maps
 * the allocation on CUDA device `device` of the calling process (peer access enabled
 * lazily) and returns its base (add the offset); phc_ipc_close unmaps it.  The exporting
 * process owns the memory and must keep it alive until every importer closed it.
 * Open a handle once per importing process (CUDA maps an allocation once per context).
 * PHC_ECUDA when the runtime refuses (e.g. memory not from cudaMalloc). */
#define PHC_IPC_HANDLE_BYTES 64
int phc_ipc_get_handle(const void* dev_ptr, void* handle, int64_t* offset);
int phc_ipc_open(const void* handle, int32_t device, void** base);
int phc_ipc_close(void* base, int32_t device);

/* End-to-end convenience: x, f, jac are HOST pointers (pinned or pageable); copies in,
 * evaluates n_points points on the home device (or sharded as above) and copies out.
 * On one device the call is a pipeline over chunks of points: the output copies of chunk c
 * (J dominates the bytes) overlap the evaluation of chunk c+1 (pinned buffers needed for the
 * overlap); results are bitwise those of phc_eval_jacobian_batch.
 * Synchronous: returns after f and jac are written. */
int phc_eval_jacobian_batch_host(const phc_system* s, int64_t n_points, const double* x_host, double* f_host,
                                 double* jac_host, const int32_t* devices, int32_t n_devices);

/* NEXT-1: one Newton iteration of Alg. 2 per point,
 * for square systems (n_eq == n_var).  For each of the n_points points x_p:
 *   F, J := the evaluation above at x_p
 *   residual[p] := max_i |F_i| (binary64 from the leading limbs)  (reading N1)
 *   solve J dz = -F by Gaussian elimination with partial pivoting (largest |.| in the column,
 *     ties to the lowest row) and back substitution
 *   x_new[p] := x_p + dz
 *   status[p] := 0, or 1 when a pivot column is exactly zero (x_new[p] := x_p).
 * x, x_new [n_points][n][2][L], residual [n_points] (double), status [n_points] (int32):
 * device pointers on the home device; x_new may alias x.  Asynchronous on `stream`.
 * The elimination runs one warp per point (n <= 32 and few points), one CTA per point with
 * [J | -F] in shared memory, or -- matrices beyond shared memory -- one cooperative launch
 * over all SMs (<= 4 points) or two launches per column (more points); all of them make the
 * same pivot choices and operations per entry, so the step is bitwise the same in every
 * regime.  Uses cudaLaunchCooperativeKernel in the cooperative regime. */
int phc_newton_step_batch(const phc_system* s, int64_t n_points, const double* x, double* x_new, double* residual,
                          int32_t* status, void* stream);

/* ---------------------------------------------------------------------------------------
 * NEXT-2: common-support systems and the paper's two-stage evaluation
 * (Alg. 2: "V := Monomial_Evaluation", then "Y := Coefficient_Product", PAPER.md P:269-284,
 * P:329-333; Table 1's "system of 40 variables with a common support of 200 monomials",
 * P:355-358).  Every polynomial uses the same n_mono monomials:
 *     f_i(x) = sum_{j < n_mono} coeff[i][j] * x^{a_j}.
 *   mono_ptr [n_mono+1]  CSR over factors of monomial j (mono_ptr[0] = 0, non-decreasing)
 *   var_idx, exponent    as in phc_system_create (strictly increasing indices, a >= 1)
 *   coeff    [n_eq][n_mono][2][limbs]  dense coefficient matrix C (HOST pointer, copied)
 * The handle works with phc_eval_jacobian[_batch][_host] and phc_newton_step_batch (same
 * layouts and semantics).  Each monomial and its partials are evaluated once per point,
 * then [F | J] = C [V | D] (D: the partials, sparse).  phc_system_set_target attaches a
 * dense target matrix [n_eq][n_mono][2][limbs]; the homotopy calls then blend
 * C(t) = (1 - t) C + t C_target entry by entry inside the coefficient product. */
int phc_system_create_common(phc_system** out, int32_t n_eq, int32_t n_var, int32_t limbs, int64_t n_mono,
                             const int64_t* mono_ptr, const int32_t* var_idx, const int32_t* exponent,
                             const double* coeff, int32_t device);

/* ---------------------------------------------------------------------------------------
 * NEXT-3: homotopy coefficients.  PAPER.md §7 P:647-649 (Table 6,
 * P:651-668): the "new" evaluator handles the continuation parameter t through the
 * coefficients, the "old" one treats t "as just another variable".  With start
 * coefficients c_s (the system's own, given to phc_system_create) and target coefficients
 * c_f on the same support, the homotopy is (reading H1)
 *     h_i(x, t) = sum_{t' in T_i} ((1 - t) c_s + t c_f) x^{a_t'} .
 * --------------------------------------------------------------------------------------- */

/* Attach target coefficients coeff_target [n_terms][2][limbs] (HOST pointer, deep-copied,
 * same term order as coeff; for a common-support handle the dense [n_eq][n_mono][2][limbs]
 * matrix) and upload them to every device the handle uses.  Calling it
 * again replaces them (the home device is synchronised first).  PHC_EINVAL on NULL or
 * non-finite limbs.  The plain eval calls keep evaluating the start coefficients. */
int phc_system_set_target(phc_system* s, const double* coeff_target);

/* h(., t_p) and its Jacobian in x at n_points points, each with its own real t_p:
 * t [n_points][limbs] (DD/QD limbs of a real, device pointer on the home device); x, f,
 * jac, devices, stream as in phc_eval_jacobian_batch.  The blend c(t) is formed per term
 * inside the kernels (one complex-by-real product per coefficient, 2 per term).
 * PHC_EINVAL if no target is attached. */
int phc_eval_homotopy_batch(const phc_system* s, int64_t n_points, const double* x, const double* t, double* f,
                            double* jac, const int32_t* devices, int32_t n_devices, void* stream);

/* One Newton iteration on h(., t_p) = 0 per point (phc_newton_step_batch with the homotopy
 * coefficients at t [n_points][limbs], device pointer). */
int phc_newton_step_homotopy_batch(const phc_system* s, int64_t n_points, const double* x, const double* t,
                                   double* x_new, double* residual, int32_t* status, void* stream);

/* Alg. 2 complete: Newton's method to tolerance per point,
 *   i := 0; ||h|| := 1;  while ||h|| > tol and i < max_it:  ||h|| := max_k |h_k(z)| at z,
 *   solve J dz = -h, z := z + dz, i := i + 1;           fail := ||h|| >= tol
 * -- the residual tested is the one computed at the start of the iteration, so the update of
 * the iteration whose residual passes is applied (the paper's loop).  t: NULL for the system
 * itself, else [n_points][limbs] (DEVICE) for the homotopy h(., t) (phc_system_set_target).
 * Per point out (DEVICE): x_out [n_points][n][2][limbs] (may alias x), residual [n_points]
 * (the last one computed; 1.0 when max_it = 0), iterations [n_points] (int32), status
 * [n_points] (int32): 0 converged, 1 failed (residual >= tol when the loop ended, or not
 * finite), 2 singular Jacobian (x_out = the point at which it was met).  Every point runs the
 * same kernels as phc_newton_step_batch, so its iterates are bitwise those of calling that
 * function i times; finished points are frozen.  tol >= 0, max_it >= 0; synchronous. */
int phc_newton_solve_batch(const phc_system* s, int64_t n_points, const double* x, const double* t, double tol,
                           int32_t max_it, double* x_out, double* residual, int32_t* iterations, int32_t* status,
                           void* stream);

/* The "old" evaluator of Table 6: a handle for the (n_var + 1)-variable system
 * in which every term c x^a of the homotopy becomes c_s x^a - c_s t x^a + c_f t x^a with t
 * the variable n_var.  Evaluating it with phc_eval_jacobian[_batch] at (x, t) (t as a
 * complex coordinate with zero imaginary part) gives h, and a Jacobian of n_var + 1 columns
 * whose last column is dh/dt.  Same arguments and validation as phc_system_create plus
 * coeff_target. */
int phc_homotopy_old_create(phc_system** out, int32_t n_eq, int32_t n_var, int32_t limbs, int64_t n_terms,
                            const int64_t* poly_ptr, const int64_t* term_ptr, const int32_t* var_idx,
                            const int32_t* exponent, const double* coeff_start, const double* coeff_target,
                            int32_t device);

/* ---------------------------------------------------------------------------------------
 * NEXT-4: predictor and path tracker (Alg. 1, the
 * quadratic predictor of §5), many paths side by side on the home device.
 * --------------------------------------------------------------------------------------- */

/* Predictor (§5, "interpolate points ... by a parabola ... value of this parabola at the
 * point (t + current step size)").  For each path p and coordinate i independently, x_out[p][i]
 * = the value at t_new[p] of the polynomial of degree h - 1, h = min(n_hist[p], order + 1),
 * through (t_hist[p][s], x_hist[p][s][i]), s < h (slot 0 the newest point): order 0 = constant,
 * 1 = secant, 2 = quadratic (Newton divided differences).  All pointers are device pointers:
 *   n_hist [n_paths] int32 in 1..3;  t_hist [n_paths][3][limbs] real limbs (distinct t);
 *   x_hist [n_paths][3][n_var][2][limbs];  t_new [n_paths][limbs];  x_out [n_paths][n_var][2][limbs].
 * No system handle is needed.  Asynchronous on `stream`. */
int phc_predict_batch(int32_t limbs, int32_t n_var, int64_t n_paths, int32_t order, const int32_t* n_hist,
                      const double* t_hist, const double* x_hist, const double* t_new, double* x_out, void* stream);

/* Tracker controls (the paper states none; defaults in DESIGN.md reading T1 follow SPEC's
 * tracker / corrector decisions). */
typedef struct phc_track_params {
  double step_init;   /* lambda_0 */
  double step_min;    /* stop (fail) when lambda < step_min */
  double step_max;    /* lambda <= step_max <= 1 */
  double expand;      /* lambda := min(lambda * expand, step_max) after each accepted step (>= 1) */
  double contract;    /* lambda := lambda * contract after a rejected step (0 < contract < 1) */
  double tol;         /* corrector tolerance eps on max_i |h_i| (Alg. 2) */
  int32_t max_newton; /* Max_It of each corrector call (Alg. 2) */
  int32_t max_steps;  /* predictor-corrector steps per path before it is declared failed */
  int32_t end_newton; /* extra Newton iterations at t = 1 on the paths that arrived */
  int32_t predictor;  /* 0 constant, 1 secant, 2 quadratic (§5) */
} phc_track_params;

/* Track n_paths solution paths of the homotopy h (phc_system_set_target) from t = 0 to t = 1
 * (Alg. 1): per path, predict (t_try = min(t + lambda, 1), z_guess from the last accepted
 * points), correct with Newton on h(., t_try) (phc_newton_step_homotopy_batch), accept when
 * the residual reaches tol within max_newton iterations (history updated only on success),
 * otherwise step back; step-size control as in phc_track_params.  All active paths advance
 * together (one batched corrector call per Newton iteration); the step-size control runs on
 * the device and the host re-compacts the active paths every 8 steps (paths that stopped in
 * between are frozen, so the decisions are those of a check after every step).  The work runs
 * on a private stream ordered after `stream`, each window of 8 steps replayed as a CUDA graph
 * (captured per active-path count; plain launches where a capture is not possible).
 *   x          [n_paths][n_var][2][limbs] DEVICE pointer: start solutions in, end points out
 *              (the last accepted point of every path, refined by end_newton iterations for
 *              the paths that reached t = 1)
 *   status     [n_paths] HOST int32 out: 1 reached t = 1, 2 failed (step below step_min or
 *              max_steps exhausted)
 *   path_stats [n_paths][5] HOST double out or NULL: accepted steps, corrector calls,
 *              Newton iterations, min and mean accepted step size (Tables 2-3 columns)
 *   t_end      [n_paths][limbs] DEVICE out or NULL: t of the returned points
 * Synchronous (returns when every path has stopped).  PHC_EINVAL without a target or with
 * inconsistent parameters. */
int phc_track_paths(const phc_system* s, int64_t n_paths, double* x, const phc_track_params* params,
                    int32_t* status, double* path_stats, double* t_end, void* stream);

/* Static facts about the system, as built: counts used by the benchmark's model.
 * out[0] = n_terms, out[1] = n_factors, out[2] = max k, out[3] = max exponent D,
 * out[4] = nnz(J) (structurally nonzero entries), out[5] = complex multiplies per point
 * performed by the kernels, out[6] = complex additions per point performed by the kernels,
 * out[7] = kernel launches per eval call (single point), out[8] = executed FP64 flops per
 * point of the kernels' useful work (DADD = DMUL = 1, DFMA = 2; padding lanes/slots not
 * counted), out[9] = path (0 generic, 1 fused block), out[10] = block layout,
 * out[11] = slots per lane K, out[12] = executed FP64 flops per point on the latency path
 * (includes its redundant products; 0 if the system never takes it),
 * out[13] = the latency-path bound: calls with n_points * n_terms <= out[13] take it,
 * out[14] = 1 for a common-support handle, out[15] = the latency-path kernel (0 none,
 * 1 one warp per term, 2 segmented: G lanes per term), out[16] = its G (0 unless segmented),
 * out[17] = kernel launches per latency-path call. */
#define PHC_STATS_LEN 18
int phc_system_stats(const phc_system* s, int64_t out[PHC_STATS_LEN]);

/* FP64 pipe peak of `device` in TFLOP/s (2 flops per DFMA), measured with independent
 * DFMA chains over `ms_target` milliseconds; the SURVEY.md §8(d) denominator. */
int phc_fp64_peak(int32_t device, double ms_target, double* tflops);

/* Kernel timing for measurement (bench.py's roofline).  When enabled, every kernel the
 * handle launches on its HOME device is bracketed by CUDA events recorded on the stream
 * it is launched on.  phc_profile_read synchronises those events and returns, per kernel
 * class c (0 power table, 1 term/monomial stage, 2 reductions, 3 fused block kernel),
 * the summed milliseconds ms[c] and launch counts launches[c]; reset != 0 clears them. */
int phc_profile_enable(const phc_system* s, int enable);
int phc_profile_read(const phc_system* s, double ms[4], int64_t launches[4], int reset);

/* Self-test hook of the DD/QD arithmetic core (test infrastructure, not the evaluation path):
 * applies operation `op` elementwise to n operands on the device (all pointers device,
 * asynchronous on `stream`).  op 0 two_sum / 1 two_prod: a, b [n] doubles -> out [n][2];
 * 2 add / 3 mul / 4 div of reals: [n][limbs]; 5 complex mul / 6 complex add / 7 lazy complex
 * mul + renormalisation / 8 complex reciprocal (of a): [n][2][limbs]; 9 real times the
 * double b[i][0]; 10 complex reciprocal as the eliminations form it (one warp per operand,
 * the two long divisions on two lanes: must equal op 8 bitwise).  PHC_EINVAL for an
 * unknown op. */
int phc_arith_test(int32_t op, int32_t limbs, int64_t n, const double* a, const double* b, double* out, void* stream);

/* Thread-local message describing the last failure in this thread ("" if none). */
const char* phc_last_error(void);

/* Library version string. */
const char* phc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PHC_H */
