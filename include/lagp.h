/*
 * lagp.h — C ABI of the B200 (sm_100a) implementation of the greedy ALC
 * local-design hot path of Gramacy, Niemi & Weiss, "Massively parallel
 * approximate Gaussian process regression" (arXiv 1310.5182).
 *
 * Citations: "P:n" = PAPER.md line n; "S:n" = SPEC.md line n; "Rk" = reading k
 * of DESIGN.md §3 (where the paper is silent or ambiguous).
 *
 * Conventions for every entry point
 *  - All array arguments are DEVICE pointers (cudaMalloc'd / torch CUDA
 *    tensors), row-major, FP64 unless noted; indices are 0-based int32.
 *    laGP_alc_batch_host is the one exception (HOST pointers, see below).
 *  - The caller owns every input and output buffer. The library owns only a
 *    per-call workspace, allocated stream-ordered from the library's own memory
 *    pool (one cudaMemPool per device, created on first use; the device's default
 *    pool is not touched) and freed back to that pool before return. The pool
 *    keeps up to 4 GiB of freed workspace mapped so that repeated calls do not
 *    re-map it; lagp_release_workspace() returns it to the driver. Other global
 *    state: the pool handles and the thread-local error string (lagp_last_error).
 *  - Work is enqueued on `cuda_stream` (a cudaStream_t; NULL = legacy default
 *    stream) and the call synchronises that stream before returning, so a
 *    status can report per-location outcomes. Reentrant on distinct streams.
 *  - Status: LAGP_EINVAL = a precondition failed; nothing was launched and the
 *    outputs are untouched; lagp_last_error() names the argument. Numerical
 *    trouble is per location (flags), never a call failure.
 */
#ifndef LAGP_H
#define LAGP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LAGP_ABI_VERSION 4
#define LAGP_SCORES_JMAX 768 /* laGP_alc_scores: largest j (Fig 4 goes to 512) */
#define LAGP_NMAX 128  /* largest local design size n of the greedy path (laGP_alc_scores: LAGP_SCORES_JMAX) */
#define LAGP_PMAX 16   /* largest input dimension p */
#define LAGP_NPRIME_MAX 65536 /* largest candidate pool N' (laGP_alc_batch; laGP_nn_pool's
                                 sorted output N' <= 8192) */
#define LAGP_NPRIME_MAX_INC 8192 /* largest N' of the incremental form (LAGP_ALC_INCREMENTAL) */

typedef enum {
    LAGP_OK = 0,      /* every location reached size n                                   */
    LAGP_PARTIAL = 1, /* ran; >= 1 location flagged EXHAUSTED or NONFINITE               */
    LAGP_EINVAL = 2,  /* bad argument: nothing launched, outputs untouched               */
    LAGP_ECUDA = 3,   /* a CUDA runtime error (message in lagp_last_error)               */
    LAGP_ENOMEM = 4   /* workspace allocation failed                                     */
} lagp_status;

/* Per-location flag bits (flags_out). */
enum {
    LAGP_FLAG_NEAR_TIE = 1u << 0,  /* some step had top-2 relative gap < 1e-12 (or all Delta == 0)   */
    LAGP_FLAG_SENTINEL = 1u << 1,  /* some candidate had m^{-1} = s_c <= 1e-12 and was excluded */
    LAGP_FLAG_EXHAUSTED = 1u << 2, /* no valid candidate before size n; idx tail = -1          */
    LAGP_FLAG_NONFINITE = 1u << 3, /* a non-finite score or prediction                                */
    /* row f2 (local MLE, laGP_mle / laGP_local_fit) */
    LAGP_FLAG_MLE_BOUND = 1u << 4, /* theta-hat ended on theta_min or theta_max                      */
    LAGP_FLAG_MLE_MAXIT = 1u << 5, /* the Newton iteration limit (64) was reached                    */
    LAGP_FLAG_MLE_FAIL = 1u << 6   /* l(theta) not finite at the start: theta-hat = incoming theta   */
};

/* Which formulation the ALC step uses (both select the same x_{j+1} in exact
 * arithmetic):
 *  LAGP_ALC_EXPLICIT    — the paper's: explicit K_j^{-1} kept per location and
 *                         s_c = 1 + eta - k_c^T K_j^{-1} k_c per candidate per
 *                         step (Eq (5)-(6), Fig 3 step 3), O(j^2) per candidate.
 *                         For n <= 64 the j×j × j×T products run on the FP64
 *                         tensor path (mma.sync m8n8k4 f64, SASS DMMA); for
 *                         larger n on a register-blocked DFMA micro-kernel.
 *  LAGP_ALC_INCREMENTAL — SURVEY §8f row f1: per-candidate Schur-complement
 *                         downdates, O(j) per candidate per step.
 *  LAGP_ALC_EXPLICIT_DFMA — the explicit form forced onto the DFMA micro-kernel
 *                         for every n (the comparison arm for the DMMA choice).
 *  LAGP_ALC_AUTO        — LAGP_ALC_INCREMENTAL wherever this build's incremental
 *                         kernels take the shape (N' <= LAGP_NPRIME_MAX_INC), else
 *                         LAGP_ALC_EXPLICIT; what laGP_alc_batch uses. The
 *                         resolved form is reported in lagp_timing.alc_form. */
typedef enum {
    LAGP_ALC_EXPLICIT = 0,
    LAGP_ALC_INCREMENTAL = 1,
    LAGP_ALC_EXPLICIT_DFMA = 2,
    LAGP_ALC_AUTO = 3
} lagp_alc_form;

/* Phase timings (milliseconds, CUDA events on cuda_stream) filled when the
 * optional `timing` argument is non-NULL. */
typedef struct {
    float nn_ms;      /* a1: NN pool kernel(s)                              */
    float alc_ms;     /* a2+a3+a4 (+a5 when fused): local-design kernel(s)  */
    float predict_ms; /* a5 when run as a separate kernel (else 0)          */
    float total_ms;   /* whole call on the device                           */
    int32_t launches; /* number of kernel launches this call issued          */
    int32_t nn_fallbacks; /* locations whose NN pool needed the exact radix-select fallback */
    int32_t alc_form; /* the formulation that ran (lagp_alc_form; LAGP_ALC_AUTO resolved) */
    int32_t reserved; /* (alignment; 0) */
    /* NN work of the call (ABI 4): (row, query) pairs the prefilter evaluated, pairs of
     * the threshold sample, exact FP64 keys computed (filter survivors) */
    int64_t nn_filter_pairs;
    int64_t nn_sample_pairs;
    int64_t nn_exact_keys;
} lagp_timing;

/*
 * laGP_alc_batch — Fig 1 steps 2 and 5 for every row of XX, with a
 * fixed global theta (Fig 1 step 1; the local MLE of steps 3-4 is
 * laGP_mle / laGP_local_fit below).
 * For each predictive location x = XX[i]:
 *   (a1) pool = the N' nearest rows of X by the key (d^2, row index), with d^2
 *        accumulated by fma in the order k = 0..p-1 (R8);
 *        X_{n0}(x) = its first n0 rows (Fig 1 step 2(a));
 *   (a2) K_{n0} = C(X_{n0}) + g I with C_ab = exp(-||x_a - x_b||^2 / d);
 *   (a3) for j = n0..n-1: x_{j+1} = argmax over pool \ X_j of the reduction in
 *        variance Delta = v_j(x) - v_{j+1}(x) of Eq (5)-(6), ties to
 *        the lowest global row index (R7); candidates with s_c <= 1e-12 excluded;
 *   (a4) partitioned-inverse update of K_j^{-1};
 *   (a5) mean, s2 (Eq (1)-(2) with N -> n) from a fresh factorisation
 *        of K_n; var = s2 n/(n-2), NaN if n <= 2.
 * The formulation is LAGP_ALC_AUTO: the incremental form (the
 * same argmax in exact arithmetic, on per-candidate Cholesky-factor state, with
 * the factor of K_n built column by column for a5) where N' <= LAGP_NPRIME_MAX_INC,
 * otherwise the explicit-K^{-1} form of the paper (a4 as written, fresh Cholesky
 * in a5). laGP_alc_batch_ex selects a form explicitly.
 *
 * Arguments
 *   X [N×p], Z [N]          design and responses (zero-mean GP, Z used raw, R14)
 *   XX [M×p]                predictive locations (this shard); M may be 0
 *   d  (theta > 0, finite)  lengthscale;  g (eta >= 0, finite) nugget
 *   1 <= n0 <= n <= Nprime <= N,  n <= LAGP_NMAX,  1 <= p <= LAGP_PMAX,
 *   Nprime <= LAGP_NPRIME_MAX (<= 8192 for LAGP_ALC_INCREMENTAL)
 *   idx_out  [M×n] int32    first n0 = NN order, then greedy order; -1 tail if exhausted
 *   mean_out [M], s2_out [M]
 *   var_out  [M]   nullable
 *   flags_out[M]   nullable (uint32 LAGP_FLAG_* bits)
 *   gap_out  [M×(n-n0)] nullable: top-2 relative gap (D1-max(D2,0))/D1 per step (NaN after exhaustion)
 * Exhausted location: stops at its current size j, predicts from D_j with
 * df = j (s2 divides by j, var = s2 j/(j-2)).
 * Returns LAGP_OK, LAGP_PARTIAL, LAGP_EINVAL, LAGP_ECUDA or LAGP_ENOMEM.
 */
lagp_status laGP_alc_batch(const double *X, int64_t N, int32_t p, const double *Z,
                           const double *XX, int64_t M, double d, double g,
                           int32_t n0, int32_t n, int32_t Nprime,
                           int32_t *idx_out, double *mean_out, double *s2_out,
                           double *var_out, uint32_t *flags_out, double *gap_out,
                           void *cuda_stream);

/* Same as laGP_alc_batch with an explicit ALC formulation and optional phase
 * timings (timing may be NULL). */
lagp_status laGP_alc_batch_ex(const double *X, int64_t N, int32_t p, const double *Z,
                              const double *XX, int64_t M, double d, double g,
                              int32_t n0, int32_t n, int32_t Nprime,
                              int32_t *idx_out, double *mean_out, double *s2_out,
                              double *var_out, uint32_t *flags_out, double *gap_out,
                              int32_t alc_form, lagp_timing *timing, void *cuda_stream);

/* End-to-end variant on HOST buffers: copies X, Z, XX host->device, runs
 * laGP_alc_batch_ex on the device, copies the outputs back (all arguments are
 * host pointers with the layouts above; nullable ones may be NULL). The copies
 * are part of the call (the bench's e2e leg). Pinned host memory is faster. */
lagp_status laGP_alc_batch_host(const double *X, int64_t N, int32_t p, const double *Z,
                                const double *XX, int64_t M, double d, double g,
                                int32_t n0, int32_t n, int32_t Nprime,
                                int32_t *idx_out, double *mean_out, double *s2_out,
                                double *var_out, uint32_t *flags_out, double *gap_out,
                                int32_t alc_form, void *cuda_stream);

/*
 * laGP_nn_pool — row a1 alone: for each of the M rows of
 * XX the Nprime nearest rows of X, sorted ascending by (d^2, row index) with d^2
 * accumulated by fma in order k = 0..p-1 (bit-exact against the oracle).
 *   pool_out [M×Nprime] int32;  d2_out [M×Nprime] nullable.
 * Constraints: 1 <= Nprime <= N, Nprime <= 8192 (sorted output), 1 <= p <= LAGP_PMAX.
 */
lagp_status laGP_nn_pool(const double *X, int64_t N, int32_t p, const double *XX, int64_t M,
                         int32_t Nprime, int32_t *pool_out, double *d2_out, void *cuda_stream);

/*
 * laGP_alc_scores — row a3 alone, the batched Fig 2 I/O: for B
 * independent locations, local design X_j [B×j×p], explicit K_j^{-1} [B×j×j]
 * (symmetric), nc candidates cands [B×nc×p] with global row ids cand_idx
 * [B×nc], reference point x [B×p]:
 *   delta_out [B×nc] nullable: Delta = (kappa - h^T K^{-1} k_c)^2 / s_c with
 *             s_c = 1 + g - k_c^T K^{-1} k_c (Eq (5)-(6)); -inf where s_c <= 1e-12;
 *   best_out  [B] int32: position (0..nc-1) of the argmax, ties to the lowest
 *             cand_idx (R7); -1 if every candidate is excluded;
 *   gap_out   [B] nullable: top-2 relative gap.
 * Constraints: 1 <= j <= LAGP_SCORES_JMAX, nc >= 1, 1 <= p <= LAGP_PMAX.
 * Also the paper's Fig 4 experiment (one location,
 * N' = 60,000 candidates, n = 16..512): beyond small batches the scores run as
 * a dense FP64 tensor-core contraction U = K^{-1}[k_c1..k_cT] over 32-candidate
 * tiles (alc_scores_gemm.cu), q_c = sum_a k_c[a] U[a][c]; the library owns a
 * stream-ordered workspace of B·(j + 4·ceil(nc/32)) doubles for the call.
 */
lagp_status laGP_alc_scores(int32_t B, int32_t j, int32_t p, int32_t nc, const double *Xj,
                            const double *Kinv, const double *cands, const int32_t *cand_idx,
                            const double *x, double d, double g, double *delta_out,
                            int32_t *best_out, double *gap_out, void *cuda_stream);

/*
 * laGP_pinv_update — row a4 alone (Eq (6)): for B
 * independent matrices, K_{j+1}^{-1} [B×(j+1)×(j+1)] from K_j^{-1} [B×j×j],
 * k = k_j(x_new) [B×j] and kdiag = K(x_new,x_new) + g (scalar, 1 + g for the
 * isotropic Gaussian): u = K^{-1}k, s = kdiag - k^T u,
 *   K_{j+1}^{-1} = [[K^{-1} + u u^T / s, -u/s], [-u^T/s, 1/s]].
 * Constraints: 1 <= j < LAGP_NMAX.
 */
lagp_status laGP_pinv_update(int32_t B, int32_t j, const double *Kinv, const double *k,
                             double kdiag, double *Kinv_out, void *cuda_stream);

/*
 * laGP_predict — row a5 alone (Eq (1)-(2), N -> n): for B local
 * designs Xn [B×n×p] with responses Yn [B×n] and reference points x [B×p]:
 * fresh Cholesky of K_n = C(X_n) + g I; mean = h^T K^{-1} Y, psi = Y^T K^{-1} Y,
 * s2 = psi (1 + g - h^T K^{-1} h) / n, var = s2 n/(n-2) (NaN if n <= 2).
 * var_out nullable. Constraints: 1 <= n <= LAGP_NMAX.
 */
lagp_status laGP_predict(int32_t B, int32_t n, int32_t p, const double *Xn, const double *Yn,
                         const double *x, double d, double g, double *mean_out, double *s2_out,
                         double *var_out, void *cuda_stream);

/*
 * laGP_exp_nonpos — the correlation kernel's exponential alone: y[i] = exp(x[i])
 * for x[i] <= 0 as the incremental local-design kernels evaluate it inside
 * K(x, x') = exp(-||x - x'||^2 / theta) (Gaussian correlation): a
 * 16-entry table of 2^(k/16) and a degree-7 polynomial, ~1 ulp; exp(x) = 0 for
 * x < -708; NaN in, NaN out. x, y device arrays of n doubles (may alias).
 * Positive inputs are outside the contract (the kernels never form them).
 * Constraints: n >= 0.
 */
lagp_status laGP_exp_nonpos(const double *x, double *y, int64_t n, void *cuda_stream);

/*
 * laGP_alc_batch_theta — laGP_alc_batch_ex with a per-location lengthscale
 * theta [M] (device, each finite and > 0; not checked on the device): location
 * i uses theta[i] in every correlation of a2-a5 (Fig 1 step 2 with theta_x,
 * P:362-371; the NN pool a1 does not depend on theta). d is still validated and
 * otherwise unused.
 */
lagp_status laGP_alc_batch_theta(const double *X, int64_t N, int32_t p, const double *Z,
                                 const double *XX, int64_t M, const double *theta, double d, double g,
                                 int32_t n0, int32_t n, int32_t Nprime,
                                 int32_t *idx_out, double *mean_out, double *s2_out,
                                 double *var_out, uint32_t *flags_out, double *gap_out,
                                 int32_t alc_form, lagp_timing *timing, void *cuda_stream);

/*
 * laGP_alc_batch_sep — SURVEY §8f row f3: laGP_alc_batch_ex under the separable
 * Gaussian correlation K(x, x') = exp(-sum_k (x_k - x'_k)^2 / theta_k) + g [x = x']
 * ("a separable version via a vectorized theta parameter"). The NN
 * pool (a1) orders rows by the same weighted distance ("relative to
 * the chosen correlation function"). Evaluated as the isotropic path with d = 1
 * on inputs rescaled by s_k = 1/sqrt(theta_k) (reading R23): x~_k = x_k * s_k,
 * s_k formed on the host with IEEE sqrt and division, x~ by one correctly
 * rounded product per entry (a stream-ordered workspace copy of X and XX).
 *   theta: HOST array of p lengthscales, each finite and > 0 (else LAGP_EINVAL).
 * Other arguments, outputs, flags and status as laGP_alc_batch_ex; timing->launches
 * includes the two rescaling launches.
 */
lagp_status laGP_alc_batch_sep(const double *X, int64_t N, int32_t p, const double *Z,
                               const double *XX, int64_t M, const double *theta, double g,
                               int32_t n0, int32_t n, int32_t Nprime,
                               int32_t *idx_out, double *mean_out, double *s2_out,
                               double *var_out, uint32_t *flags_out, double *gap_out,
                               int32_t alc_form, lagp_timing *timing, void *cuda_stream);

/*
 * laGP_mle — SURVEY §8f row f2, Fig 1 step 3: for each location i,
 * the local MLE theta-hat_n(x_i) of the concentrated likelihood Eq (3)
 * on D_n(x_i) = (X[idx[i,:]], Z[idx[i,:]]) (the valid prefix of the
 * row when it has a -1 tail), then the prediction of Fig 1 step 5 (Eq (1)-(2),
 * P:171-187) at x_i = XX[i] with theta-hat on the same design.
 *   Search (readings R20-R21): safeguarded Newton on tau = log(theta) with the
 *   analytic first and second derivatives, inside [theta_min, theta_max], started
 *   at theta_in[i] (or theta0 when theta_in is NULL) clamped into the bounds;
 *   Newton steps capped at |1| in tau; long or non-Newton steps halved until l
 *   does not decrease; stops at a bound the gradient points out of, when
 *   |step| <= 1e-10 max(1, |tau|), or after 64 iterations.
 * Arguments
 *   X [N×p], Z [N], XX [M×p]; idx [M×n] int32 local designs (e.g. laGP_alc_batch's idx_out)
 *   theta_in [M] nullable; theta0 > 0 (used when theta_in is NULL)
 *   0 < theta_min <= theta_max finite;  g (eta >= 0) nugget;  1 <= n <= LAGP_NMAX
 *   theta_out [M]; loglik_out [M] nullable (l at theta-hat); iters_out [M] int32 nullable
 *   flags_out [M] nullable: LAGP_FLAG_MLE_* (and NONFINITE) bits are OR-ed in
 *   mean_out [M], s2_out [M], var_out [M] (nullable): prediction at theta-hat
 * A location whose l is not finite at its start keeps the incoming theta
 * (LAGP_FLAG_MLE_FAIL) and predicts with it.
 */
lagp_status laGP_mle(const double *X, int64_t N, int32_t p, const double *Z, const double *XX, int64_t M,
                     const int32_t *idx, int32_t n, const double *theta_in, double theta0,
                     double theta_min, double theta_max, double g,
                     double *theta_out, double *loglik_out, int32_t *iters_out, uint32_t *flags_out,
                     double *mean_out, double *s2_out, double *var_out, void *cuda_stream);

/*
 * laGP_local_fit — the multi-stage scheme of Fig 1 (the "two-stage
 * scheme" of P:351-355): theta_x = theta0 (step 1); then `stages` times: the
 * local design X_n(x, theta_x) (step 2, as laGP_alc_batch_theta) and
 * theta_x = theta-hat_n(x) | D_n(x, theta_x) (step 3, as laGP_mle started at
 * theta_x); finally the prediction with theta_x on the last D_n(x) (step 5).
 * The NN pool (a1) is computed once per location.
 *   1 <= stages <= 16;  theta_out [stages×M]: theta_x after each stage
 *   idx_out [M×n]: the last stage's design;  mean/s2/var: step 5
 *   flags_out [M] nullable: the last design's flags | the last MLE's flags
 *   timing nullable: nn_ms = a1, alc_ms = all designs, predict_ms = all MLE+predict
 * Other arguments and constraints as laGP_alc_batch_ex and laGP_mle.
 */
lagp_status laGP_local_fit(const double *X, int64_t N, int32_t p, const double *Z,
                           const double *XX, int64_t M, double theta0, double theta_min, double theta_max,
                           double g, int32_t n0, int32_t n, int32_t Nprime, int32_t stages, int32_t alc_form,
                           int32_t *idx_out, double *theta_out, double *mean_out, double *s2_out,
                           double *var_out, uint32_t *flags_out, lagp_timing *timing, void *cuda_stream);

/* Return the current device's cached workspace memory (the library's pool) to
 * the driver; synchronises the device. LAGP_OK or LAGP_ECUDA. */
lagp_status lagp_release_workspace(void);

/* Thread-local message for the last non-OK status of this thread. */
const char *lagp_last_error(void);
/* LAGP_ABI_VERSION of the loaded library. */
int lagp_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LAGP_H */
