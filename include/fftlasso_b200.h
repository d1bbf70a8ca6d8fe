/*
 * libfftlasso_b200 -- C ABI of the B200-native matrix-free IPM hot path.
 *
 * Drop-in boundary for the reference package ``fftlasso`` (Python,
 * /root/reference/pkg/src/fftlasso).  Each entry point names the reference
 * function it replaces (file:line).  The reference has no native code, so
 * these are the functions a ctypes/cffi binding of the reference's hot path
 * would call (see INTEGRATION.md for the binding a maintainer would add).
 *
 * Conventions
 *  - All vectors are fp64 DEVICE pointers, grids row-major (C order), the
 *    layout of the reference (fourier.py:14-16).  n = product of dims.
 *  - Masks are device bitmasks: bit (v & 31) of word v >> 5 set <=> voxel v
 *    is missing (masking.py:22-51 keeps the same set as sorted int64 +
 *    bool).  ``obs_offsets[w]`` = number of observed voxels before word w.
 *  - Every call is ordered on ``stream`` (a cudaStream_t) and returns an
 *    fl_status.  Calls that return scalars to the host synchronise the
 *    stream.  The library never frees caller memory; a plan owns only its
 *    twiddle tables.  Per host thread the library keeps a small reduction
 *    scratch (partials + pinned result slots).
 *  - Status -> reference exception: FL_E_SHAPE -> UnsupportedShapeError,
 *    FL_E_VALUE -> ValueError, FL_E_INTERIOR -> InteriorViolationError,
 *    FL_E_BREAKDOWN -> NumericalBreakdownError, FL_E_STALLED -> StalledError
 *    (errors.py:4-25); FL_E_CUDA / FL_E_NOMEM -> RuntimeError / MemoryError.
 */
#ifndef FFTLASSO_B200_H
#define FFTLASSO_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FL_API __attribute__((visibility("default")))
#else
#define FL_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum fl_status {
  FL_OK = 0,
  FL_E_SHAPE = 1,
  FL_E_VALUE = 2,
  FL_E_INTERIOR = 3,
  FL_E_BREAKDOWN = 4,
  FL_E_STALLED = 5,
  FL_E_CUDA = 6,
  FL_E_NOMEM = 7
};

typedef struct fl_plan* fl_plan_t;
typedef void* fl_stream_t; /* cudaStream_t */

/* IPM iterate (ipm.py:85-97): eight device vectors of length n. */
typedef struct {
  double* beta;
  double* z;
  double* s1;
  double* s2;
  double* y1;
  double* y2;
  double* nu1;
  double* nu2;
} fl_state;

/* Exact-KKT and barrier residual norms at an iterate.
 * Replaces check_convergence (ipm.py:241-273) + _barrier_residual (ipm.py:276-282). */
typedef struct {
  double stationarity;    /* max|A^T(b - M beta) + y1 - y2|          ipm.py:244-254 */
  double dual_equality;   /* max|lam - y1 - y2|                       ipm.py:246,255 */
  double multiplier_gap;  /* max(max|y1-nu1|, max|y2-nu2|)            ipm.py:247-256 */
  double primal;          /* max(max|z+beta-s1|, max|z-beta-s2|)      ipm.py:249-257 */
  double complementarity; /* max(max s1 nu1, max s2 nu2)              ipm.py:258 */
  double min_product;     /* min(min s1 nu1, min s2 nu2)              ipm.py:262 */
  double dot_nu_s1;       /* nu1 . s1                                  ipm.py:105 */
  double dot_nu_s2;       /* nu2 . s2                                  ipm.py:105 */
  double barrier_residual;/* _barrier_residual at mu                   ipm.py:276-282 */
} fl_assess;

typedef struct {
  int64_t iterations;
  int32_t converged;
  int32_t _pad;
  double residual_norm;
  double norm0;
} fl_pcg_result;

/* ---- library / plan -------------------------------------------------- */
FL_API int fl_version(void);
FL_API const char* fl_last_error(void);
/* GridShape (fourier.py:52-77): 1..3 even dims >= 2.  Builds per-axis FFT
 * plans and twiddle tables on ``device``. */
FL_API int fl_plan_create(int ndim, const int64_t* dims, int device, fl_plan_t* out);
FL_API int fl_plan_destroy(fl_plan_t plan);
FL_API int64_t fl_plan_n(fl_plan_t plan);

/* Local plan of a slab-sharded grid: only the axes set in ``transform_axes``
 * (bit a = axis a) are planned/validated (even, >= 2); the others are batch
 * extents of any size >= 1 (slab heights d0/P, d1/P). */
FL_API int fl_plan_create_ex(int ndim, const int64_t* dims, int transform_axes, int device,
                             fl_plan_t* out);

/* ---- transforms (fourier.py) ----------------------------------------- */
/* synthesize (fourier.py:201-222): x = A beta.  ``beta`` may equal ``x``. */
FL_API int fl_synthesize(fl_plan_t plan, const double* beta, double* x, fl_stream_t stream);
/* analyze (fourier.py:225-235): beta = A^T x.  ``x`` may equal ``beta``. */
FL_API int fl_analyze(fl_plan_t plan, const double* x, double* beta, fl_stream_t stream);

/* One per-axis pass: _synthesize_axis (fourier.py:172-183, analysis = 0)
 * or _analyze_axis (fourier.py:186-198, analysis = 1) along ``axis``.
 * Building block of the slab-sharded transform; in may equal out.
 * analysis = 2 runs the tile-copy measurement kernel (same tiles and lanes as
 * the power-of-two pass, FFT removed) used to separate access-pattern cost
 * from FFT cost (tools/pass_copy_probe.py). */
FL_API int fl_axis_pass(fl_plan_t plan, int axis, int analysis, const double* in, double* out,
                        fl_stream_t stream);

/* ---- observation operators (masking.py) ------------------------------ */
/* The fused last-axis pass on its own: synthesis along the last (contiguous)
 * axis, Z x (b_hat == NULL: gram, masking.py:116-117) or Z (b_hat - x)
 * (residual), analysis along the same axis.  With ``nrm_host`` != NULL and
 * b_hat == NULL also returns ||Z x||^2 (synchronises).  This is the middle
 * step of the slab-sharded gram, run in the Y-slab layout. */
FL_API int fl_fused_mask_pass(fl_plan_t plan, const uint32_t* miss_bits, const double* b_hat,
                              const double* in, double* out, double* nrm_host, fl_stream_t stream);
/* Slab transposes of a (d0, d1, d2) grid over P ranks (d0 = P*a, d1 = P*b):
 *   X-slab of rank r: rows i0 in [r a, (r+1) a), local layout (a, d1, d2);
 *   Y-slab of rank r: i1 in [r b, (r+1) b), local layout (b, d2, d0) -- axis 0
 *   made contiguous so the fused mask pass runs on it.
 * pack_x:   X-slab -> send buffer of P blocks (a, b, d2), block s for rank s.
 * unpack_y: receive buffer of P blocks (a, b, d2) (block r from rank r) -> Y-slab.
 * pack_y / unpack_x: the inverse pair (Y-slab -> blocks -> X-slab). */
FL_API int fl_slab_pack_x(int64_t a, int64_t d1, int64_t d2, int nranks, const double* x_slab,
                          double* send, fl_stream_t stream);
FL_API int fl_slab_unpack_y(int64_t a, int64_t b, int64_t d2, int nranks, const double* recv,
                            double* y_slab, fl_stream_t stream);
FL_API int fl_slab_pack_y(int64_t a, int64_t b, int64_t d2, int nranks, const double* y_slab,
                          double* send, fl_stream_t stream);
FL_API int fl_slab_unpack_x(int64_t a, int64_t d1, int64_t d2, int nranks, const double* recv,
                            double* x_slab, fl_stream_t stream);

/* Mask bookkeeping: bits + per-word observed offsets from a byte mask
 * (masking.py:61-69 from_bool).  ``flags`` is a device uint8 array (1 =
 * missing); writes n_words = ceil(n/32) words and offsets; returns the
 * observed count through ``n_observed`` (synchronises). */
FL_API int fl_mask_build(int64_t n, const uint8_t* flags, uint32_t* miss_bits, int64_t* obs_offsets,
                  int64_t* n_observed, fl_stream_t stream);
/* On-device input generation: the Bragg-peak punch mask
 * of the C3-C5 recipes -- voxel missing when the summed squared periodic
 * distances to the nearest multiple of ``spacing`` along every axis are
 * <= radius^2 (bitwise equal to fl_mask_build of the host formula) -- built
 * straight into bits + observed offsets, no host flags.  Synchronises. */
FL_API int fl_mask_bragg(int ndim, const int64_t* dims, int64_t spacing, double radius, uint32_t* miss_bits,
                         int64_t* offsets, int64_t* n_observed, fl_stream_t stream);
/* On-device observation noise for the C4/C5 recipes (no
 * reference counterpart: the reference draws noise on the host,
 * synthetic.py:45-63).  In place on a local box of a grid:
 * x[k] = missing(k) ? 0 : x[k] + sigma * N(seed, g(k)), where k indexes the
 * box ext[0] x ext[1] x ext[2] (row-major; miss_bits indexed by k) and
 * g(k) = sum_a (l_a + off[a]) * stride[a] is the voxel's GLOBAL flat index,
 * so the full grid, X-slabs and Y-slabs get bitwise the same draws. */
FL_API int fl_noisy_embed(const int64_t* ext, const int64_t* off, const int64_t* stride, uint64_t seed,
                          double sigma, const uint32_t* miss_bits, double* x, fl_stream_t stream);
/* embed (masking.py:90-99): full = 0; full[observed] = obs. */
FL_API int fl_embed(int64_t n, const uint32_t* miss_bits, const int64_t* obs_offsets,
             const double* obs, double* full, fl_stream_t stream);
/* gather half of observe (masking.py:81-87): obs = full[observed]. */
FL_API int fl_gather_observed(int64_t n, const uint32_t* miss_bits, const int64_t* obs_offsets,
                       const double* full, double* obs, fl_stream_t stream);
/* gram (masking.py:107-118): out = A^T Z A beta (Z zeroes missing samples). */
FL_API int fl_gram(fl_plan_t plan, const uint32_t* miss_bits, const double* beta, double* out,
            fl_stream_t stream);
/* observe_adjoint(b - observe(beta)) on the full grid (masking.py:102-104 with
 * ipm.py:244-245 / newton_system.py:136-137): out = A^T Z (b_hat - A beta),
 * b_hat = embed(b).  ``beta`` may be NULL (treated as 0 -> A^T b_hat). */
FL_API int fl_residual_adjoint(fl_plan_t plan, const uint32_t* miss_bits, const double* b_hat,
                        const double* beta, double* out, fl_stream_t stream);

/* ---- condensed KKT algebra (newton_system.py) ------------------------- */
/* barrier_diagonals (newton_system.py:72-91).  sigma1/sigma2 always
 * written; lambda1/lambda2/dvec/bvec optional (NULL to skip).  Returns
 * FL_E_INTERIOR if any input is <= 0 or non-finite (synchronises). */
FL_API int fl_barrier_diagonals(int64_t n, const double* s1, const double* s2, const double* nu1,
                         const double* nu2, double* sigma1, double* sigma2, double* lambda1,
                         double* lambda2, double* dvec, double* bvec, fl_stream_t stream);
/* apply_kkt (newton_system.py:148-152) from (sigma1, sigma2); one fused
 * gram + epilogue.  If ``pkp_host`` != NULL also returns d . K d
 * (synchronises). */
FL_API int fl_kkt_apply(fl_plan_t plan, const uint32_t* miss_bits, const double* sigma1,
                 const double* sigma2, const double* d_beta, const double* d_z, double* top,
                 double* bottom, double* pkp_host, fl_stream_t stream);
/* fl_kkt_apply with a cudaEvent after every HBM pass; writes the per-pass
 * device times (ms) to ``pass_ms`` (host, up to 2*ndim entries) and the
 * number of passes to ``npasses``: order A (fl_kkt_order 0) 2*ndim-1
 * transform passes + the elementwise KKT epilogue; order B (1) 2*ndim-1
 * transform passes, the epilogue fused into the last.  Measurement hook for
 * bench.py. */
/* Operator order of fl_kkt_apply for this plan: 0 = axis-0 synthesis first,
 * fused mask pass on the contiguous axis, separate KKT epilogue; 1 = the
 * contiguous axis first and last (fused mask pass on axis 0, epilogue fused
 * into the final contiguous analysis; 3D grids with axes 0 and 2 of 512). */
FL_API int fl_kkt_order(fl_plan_t plan);
FL_API int fl_kkt_apply_profiled(fl_plan_t plan, const uint32_t* miss_bits, const double* sigma1,
                                 const double* sigma2, const double* d_beta, const double* d_z,
                                 double* top, double* bottom, double* pass_ms, int* npasses,
                                 fl_stream_t stream);
/* KKT epilogue alone on a gram output g (in place -> top):
 * top = (g + L1 d_beta) + L2 d_z, bottom = L2 d_beta + L1 d_z
 * (newton_system.py:150-151); optional LOCAL d.Kd to the host (synchronises).
 * Used by the slab-sharded matvec after the sharded gram. */
FL_API int fl_kkt_epilogue(int64_t n, double* g_top, const double* d_beta, const double* d_z,
                           const double* sigma1, const double* sigma2, double* bottom,
                           double* pkp_host, fl_stream_t stream);
/* apply_precond_inverse (newton_system.py:155-159). */
FL_API int fl_precond_apply(int64_t n, const double* sigma1, const double* sigma2, const double* r_beta,
                     const double* r_c, double* top, double* bottom, fl_stream_t stream);
/* newton_rhs (newton_system.py:113-145) given g = A^T Z (b_hat - A beta)
 * (fl_residual_adjoint).  r1..r6 are optional outputs (NULL to skip). */
FL_API int fl_newton_rhs(int64_t n, const fl_state* st, const double* g, const double* sigma1,
                  const double* sigma2, double lam, double mu, double* r1, double* r2,
                  double* r3, double* r4, double* r5, double* r6, double* r_beta, double* r_c,
                  fl_stream_t stream);
/* recover_eliminated (newton_system.py:184-196): d_s1, d_s2, d_y1, d_y2 in
 * the condensed sign convention from the condensed solution and r3..r6. */
FL_API int fl_recover_eliminated(int64_t n, const double* sigma1, const double* sigma2,
                                 const double* r3, const double* r4, const double* r5,
                                 const double* r6, const double* d_beta, const double* d_z,
                                 double* d_s1, double* d_s2, double* d_y1, double* d_y2,
                                 fl_stream_t stream);

/* ---- PCG (pcg.py) ------------------------------------------------------ */
/* Device work doubles needed by fl_pcg_kkt for a plan of size n. */
FL_API int64_t fl_pcg_work_doubles(int64_t n);
/* PCG loop of fl_pcg_kkt / fl_ipm_newton_pcg / fl_ipm_newton_step, process
 * wide: 3 (default) = one CUDA graph per solve whose WHILE node loops on the
 * device; 2 = host loop over the same kernels (one sync per iteration).  Both
 * give bitwise the same iterates (tested); no reference counterpart. */
FL_API int fl_set_pcg_loop(int mode);
/* pcg_solve (pcg.py:57-127) on the condensed KKT system K x = rhs
 * (ipm.py:318-327), device resident: fused gram+epilogue matvec, fused
 * update/preconditioner/dot pass, one host sync per iteration.
 * rhs, x: 2n vectors [beta-block; z-block].  ``history`` (nullable) receives
 * up to ``max_history`` residual norms.  Returns FL_E_BREAKDOWN on NaN or
 * non-positive curvature (message in fl_last_error); non-convergence is
 * reported through res->converged. */
FL_API int fl_pcg_kkt(fl_plan_t plan, const uint32_t* miss_bits, const double* sigma1,
               const double* sigma2, const double* rhs, double* x, double* work,
               double abs_tol, double rel_tol, int64_t max_iters, fl_pcg_result* res,
               double* history, int64_t max_history, fl_stream_t stream);

/* Step-wise PCG kernels of fl_pcg_kkt (v2) for callers that combine the
 * scalars across ranks themselves (slab-sharded solve).  All return LOCAL
 * partial sums to the host (synchronise):
 *   init:    x = 0, r = rhs, p = P^{-1} r;  out[0] = r.p, out[1] = p.(K-G)p
 *   update:  with K p formed from g = G p_beta: x += alpha p, r -= alpha K p;
 *            out[0] = r.P^{-1}r
 *   pupdate: p = P^{-1} r + beta p;  out[0] = p.(K-G)p */
FL_API int fl_pcg_step_init(int64_t n, const double* sigma1, const double* sigma2, const double* rhs,
                            double* x, double* r, double* p, double* out, fl_stream_t stream);
FL_API int fl_pcg_step_update(int64_t n, const double* sigma1, const double* sigma2, double alpha,
                              double* x, double* r, const double* p, const double* g, double* out,
                              fl_stream_t stream);
FL_API int fl_pcg_step_pupdate(int64_t n, const double* sigma1, const double* sigma2, const double* r,
                               double beta, double* p, double* out, fl_stream_t stream);
/* Device-scalar forms for the sharded loop (no host synchronisation): the
 * local partial is written to device memory (out_dev), alpha is read from
 * device memory; fl_pcg_step_alpha forms curv = red2[0] + red2[1] and
 * alpha = rho / curv (pcg.py:103-110, the host's operation order) into
 * out_dev[0..1]; fl_fused_mask_pass_dev is fl_fused_mask_pass (gram form)
 * with ||Z A beta||^2 written to device memory. */
FL_API int fl_pcg_step_update_dev(int64_t n, const double* sigma1, const double* sigma2, const double* alpha_dev,
                                  double* x, double* r, const double* p, const double* g, double* out_dev,
                                  fl_stream_t stream);
FL_API int fl_pcg_step_pupdate_dev(int64_t n, const double* sigma1, const double* sigma2, const double* r,
                                   double beta, double* p, double* out_dev, fl_stream_t stream);
FL_API int fl_pcg_step_alpha(const double* red2, const double* rho_dev, double* out_dev, fl_stream_t stream);
FL_API int fl_fused_mask_pass_dev(fl_plan_t plan, const uint32_t* miss_bits, const double* in, double* out,
                                  double* nrm_dev, fl_stream_t stream);
/* Objective pieces on a full (or slab) grid given x = A beta:
 * out[0] = sum over observed (b_hat - x)^2, out[1] = sum |beta| (beta may be
 * NULL -> 0).  ipm.py:209-211. */
FL_API int fl_objective_terms(int64_t n, const uint32_t* miss_bits, const double* b_hat,
                              const double* x, int64_t n_beta, const double* beta, double* out,
                              fl_stream_t stream);

/* ---- IPM outer step (ipm.py) ------------------------------------------ */
/* initial_state (ipm.py:214-238): beta=0, z=s=1, y=nu=0.5*lam. */
FL_API int fl_ipm_init(int64_t n, const fl_state* st, double lam, fl_stream_t stream);
/* check_convergence + _barrier_residual norms (synchronises). */
FL_API int fl_ipm_assess(int64_t n, const fl_state* st, const double* g, double lam, double mu,
                  fl_assess* out, fl_stream_t stream);
/* Back-substitution, slack sign flip and d_nu (ipm.py:334-338) fused with
 * the four fraction-to-boundary ratio minima (ipm.py:355-376).  ``ratios``
 * (host, 4) = min over dv<0 of v/(-dv) for (s1, s2, nu1, nu2), +inf when no
 * component shrinks.  Synchronises. */
FL_API int fl_ipm_ratios(int64_t n, const fl_state* st, const double* sigma1, const double* sigma2,
                  double mu, const double* d_beta, const double* d_z, double* ratios,
                  fl_stream_t stream);
/* Full 8-block direction (NewtonDirection, ipm.py:285-352), for callers that
 * need it materialised.  Outputs may alias nothing. */
FL_API int fl_ipm_direction(int64_t n, const fl_state* st, const double* sigma1, const double* sigma2,
                     double mu, const double* d_beta, const double* d_z, double* d_s1,
                     double* d_s2, double* d_y1, double* d_y2, double* d_nu1, double* d_nu2,
                     fl_stream_t stream);
/* State update with primal/dual step lengths (ipm.py:382-393), directions
 * recomputed in registers.  Returns FL_E_STALLED if the new iterate is not
 * strictly interior (assert_interior, ipm.py:107-110).  Synchronises. */
FL_API int fl_ipm_update(int64_t n, const fl_state* st, const double* sigma1, const double* sigma2,
                  double mu, const double* d_beta, const double* d_z, double alpha_p,
                  double alpha_d, fl_stream_t stream);
/* Apply explicit directions (used when a caller supplies its own
 * NewtonDirection): v += alpha * dv; interior check as above. */
FL_API int fl_ipm_update_explicit(int64_t n, const fl_state* st, const fl_state* dir, double alpha_p,
                           double alpha_d, fl_stream_t stream);
/* lasso_objective (ipm.py:209-211) on the full grid (synchronises). */
FL_API int fl_lasso_objective(fl_plan_t plan, const uint32_t* miss_bits, const double* b_hat,
                       const double* beta, double lam, double* work, double* out,
                       fl_stream_t stream);

/* ---- vector primitives for the generic pcg_solve plug-in (pcg.py) ------ */
FL_API int fl_dot(int64_t n, const double* a, const double* b, double* out, fl_stream_t stream);
FL_API int fl_max_abs(int64_t n, const double* a, double* out, fl_stream_t stream);
FL_API int fl_min(int64_t n, const double* a, double* out, fl_stream_t stream);
/* fraction_to_boundary core (ipm.py:355-361): min over dv<0 of v/(-dv),
 * +inf when no component shrinks (synchronises). */
FL_API int fl_ftb_ratio(int64_t n, const double* v, const double* dv, double* out,
                        fl_stream_t stream);
/* y = y + alpha * x   (NumPy ``y += alpha * x``) */
FL_API int fl_axpy(int64_t n, double alpha, const double* x, double* y, fl_stream_t stream);
/* y = x + beta * y    (NumPy ``p = z + beta * p``) */
FL_API int fl_xpby(int64_t n, const double* x, double beta, double* y, fl_stream_t stream);

/* ---- slab exchange over peer memory (sharded transform) ------
 * One kernel per direction instead of pack -> all-to-all -> unpack: each
 * element of the local slab is stored once, transposed, straight into the
 * owning rank's slab.  ``y_slabs`` / ``x_slabs`` hold ``nranks`` device
 * pointers (peer allocations opened with fl_ipc_open; this rank's own buffer
 * at index ``rank``).  The caller orders the exchange with a cross-rank
 * barrier on the stream afterwards (e.g. a one-element all-reduce). */
FL_API int fl_slab_x_to_y_peers(int64_t a, int64_t d1, int64_t d2, int nranks, int rank, const double* x_slab,
                                double* const* y_slabs, fl_stream_t stream);
FL_API int fl_slab_y_to_x_peers(int64_t a, int64_t b, int64_t d2, int nranks, int rank, const double* y_slab,
                                double* const* x_slabs, fl_stream_t stream);
/* The X->Y exchange of planes [i0_begin, i0_begin + i0_count) of this rank's
 * slab (``x_planes`` points at plane i0_begin): lets the exchange of one
 * chunk of planes run while the next chunk is still being transformed. */
FL_API int fl_slab_x_to_y_peers_planes(int64_t a, int64_t d1, int64_t d2, int nranks, int rank,
                                       int64_t i0_begin, int64_t i0_count, const double* x_planes,
                                       double* const* y_slabs, fl_stream_t stream);
/* cudaMalloc + cudaIpcGetMemHandle (64-byte handle), the peer side's open /
 * close, and the matching free. */
FL_API int fl_ipc_alloc(int64_t bytes, void** ptr, unsigned char* handle64);
FL_API int fl_ipc_open(const unsigned char* handle64, void** ptr);
FL_API int fl_ipc_close(void* ptr);
FL_API int fl_dev_free(void* ptr);

/* ---- fused Newton step front half (ipm.py:303-332) ---------------------
 * One pass computes the barrier diagonals sigma = nu/s with the interior
 * check (newton_system.py:72-91 -> FL_E_INTERIOR), the condensed RHS
 * (newton_system.py:113-145, never stored) and the PCG start, then runs the
 * condensed PCG (pcg.py:57-127) to x = (d_beta, d_z).  Bitwise equal to
 * fl_barrier_diagonals + fl_newton_rhs + fl_pcg_kkt; ``sigma1``/``sigma2`` are
 * written for the back-substitution.  ``work`` as for fl_pcg_kkt. */
FL_API int fl_ipm_newton_pcg(fl_plan_t plan, const uint32_t* miss_bits, const fl_state* st, const double* g,
                             double lam, double mu, double* sigma1, double* sigma2, double* x, double* work,
                             double abs_tol, double rel_tol, int64_t max_iters, fl_pcg_result* res,
                             fl_stream_t stream);

/* One IPM step (ipm.py:364-394, the fused form of newton_direction +
 * fraction_to_boundary + the state update) with no host sync after the PCG
 * start: fl_ipm_newton_pcg, then the ratio minima, the step lengths
 * alpha = min(1, tau * ratio) on the device, the state update (skipped when
 * the PCG did not converge or alpha < 1e-12) and the interior flag.  The
 * verdict lands in pinned ``host_out`` (13 doubles: ratio minima[4], alpha_p,
 * alpha_d, skipped, interior flag, PCG status 1 converged / 2 cap /
 * 3 curvature / 4 r'P^{-1}r breakdown, PCG iterations, residual norm,
 * offending value, initial norm) after the caller's next stream sync.  The
 * same kernels in the same order as fl_ipm_newton_pcg + fl_ipm_ratios +
 * fl_ipm_update, so the iterates are bitwise those of that path. */
FL_API int fl_ipm_newton_step(fl_plan_t plan, const uint32_t* miss_bits, const fl_state* st, const double* g,
                              double lam, double mu, double tau, double* sigma1, double* sigma2, double* x,
                              double* work, double abs_tol, double rel_tol, int64_t max_iters, double* host_out,
                              fl_stream_t stream);

/* ---- diagnostics (diagnostics.py) -------------------------------------- */
/* out = sign(x) * max(|x| - t, 0) elementwise, NumPy conventions
 * (soft_threshold, diagnostics.py:325-328); in place allowed. */
FL_API int fl_soft_threshold(int64_t n, const double* x, double t, double* out, fl_stream_t stream);
/* One ISTA iteration after the gram (ista_solve, diagnostics.py:352-357):
 * next = soft(beta - (gram_beta - xi), lam); *step = max|next - beta| (host
 * scalar, synchronises). */
FL_API int fl_ista_step(int64_t n, const double* beta, const double* gram_beta, const double* xi,
                        double lam, double* next, double* step, fl_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* FFTLASSO_B200_H */
