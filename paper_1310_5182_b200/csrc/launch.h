// launch.h — host-side launchers of the sm_100a kernels (one definition of the
// argument structs, shared by the kernel TUs and abi.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lagp {

// nn.cu (row a1)
// sorted = true: the whole pool ascending by (d^2, index) (laGP_nn_pool); false:
// pool[0..n0) ascending, the rest of the N' nearest in any order (laGP_alc_batch).
// Mmax: the largest chunk of query locations a call with this workspace passes (M <= Mmax).
cudaError_t launch_nn(const double *X, int64_t N, int p, const double *XX, int64_t M, int64_t Mmax, int Nprime, int n0,
                      bool sorted, int32_t *pool, double *d2, void *ws, int grid, int *fb, cudaStream_t st, bool prepared,
                      int *launches);
size_t nn_ws_bytes(int grid, int64_t N, int p, int Nprime, bool sorted, int64_t Mmax);
// NN work counters in an NN workspace: [0] prefilter pairs, [1] sample pairs, [2] exact keys
unsigned long long *nn_pair_counters(void *ws);
int nn_grid(int64_t M, int num_sms, int Nprime);

// fused local-design kernels (rows a2-a5)
struct AlcArgs {
    const double *X;
    int64_t N;
    int p;
    const double *Z;
    const double *XX;
    int64_t M;
    double eta, rtheta;
    const double *theta_vec;  // [M] per-location theta (multi-stage scheme), nullptr = 1/rtheta everywhere
    int n0, n, Nprime, ld;
    int Npad;             // Nprime rounded up to a multiple of 4 (16-byte rows)
    int64_t cache_stride; // doubles per CTA cache slab (n*Npad + tile overrun pad)
    const int32_t *pool;  // [M][Nprime], first n0 = NN order
    int32_t *idx_out;
    double *mean, *s2, *var;
    uint32_t *flags;
    double *gap_out;
    // per-CTA slabs in global memory
    double *cache;          // [grid][cache_stride]: rows a of K(X_j[a], x_c), row stride Npad
    double *coords;         // [grid][p][Npad] pool coordinates (SoA)
    int *n_partial;         // count of EXHAUSTED/NONFINITE locations
};
cudaError_t launch_alc_explicit(const AlcArgs &a, int grid, cudaStream_t st);
int alc_explicit_blocks_per_sm(int ld, int n, int p, int Npad);
cudaError_t launch_alc_explicit_dmma(const AlcArgs &a, int grid, cudaStream_t st);

// alc_incremental.cu (row f1): where the per-candidate w_c entries live
struct IncPlan {
    bool ok;
    int cpt;             // candidates per thread (1024 threads)
    int R;               // entries in registers
    int S;               // entries in shared memory
    int global_entries;  // entries in the per-CTA HBM slab (A.cache)
    int wsz;             // doubles of the shared w region (>= S*Npad, >= predict scratch)
    size_t smem;         // dynamic shared memory bytes
    bool v2;             // alc_incremental_v2.cu (N' <= 1024, p in {1,2,3,4,8})
    int64_t cache_doubles;  // per-CTA slab doubles (v2)
    int tfirst;             // v2 mode: bit 0 shared-memory entries before the tensor-memory ones, bit 1 no stagger
    int threads;            // v2: threads per CTA
    bool stream;            // alc_incremental_stream.cu (state in HBM, N' <= 65536)
};
IncPlan inc_plan(int n, int p, int Nprime, int Npad, size_t smem_optin);
// alc_incremental_v2.cu: one barrier per step, 512 threads, 1-2 candidates per thread
bool inc_v2_plan(int n, int p, int Nprime, size_t smem_optin, IncPlan &pl);
cudaError_t launch_alc_incremental_v2(const AlcArgs &a, const IncPlan &pl, int grid, cudaStream_t st);
cudaError_t launch_alc_incremental(const AlcArgs &a, const IncPlan &pl, int grid, cudaStream_t st);
// alc_incremental_stream.cu: per-candidate state in an HBM slab (cache_doubles per CTA), 2 CTAs/SM
bool inc_stream_plan(int n, int p, int Nprime, IncPlan &pl);
cudaError_t launch_alc_incremental_stream(const AlcArgs &a, int grid, cudaStream_t st);
int alc_explicit_dmma_blocks_per_sm(int n, int p, int Npad);

// mle.cu (row f2): local MLE of theta on given designs + prediction at theta-hat
struct MleArgs {
    const double *X;
    int p;
    const double *Z;
    const double *XX;
    const int32_t *idx;     // [M][n] local designs (-1 tail = exhausted)
    int64_t M;
    int n;
    const double *theta_in; // [M] starting theta, nullptr = theta0
    double theta0, lo, hi, eta;
    double *theta_out;      // [M]
    double *loglik_out;     // [M] nullable
    int32_t *iters_out;     // [M] nullable
    uint32_t *flags_out;    // [M] nullable, OR-ed
    double *mean, *s2, *var;  // [M] (var nullable): prediction at theta-hat
    double *ws;             // per-CTA matrices when they do not fit in shared memory
    int use_smem;
    int *n_partial;         // nullable: count of locations flagged NONFINITE
};
size_t mle_smem_bytes(int n, int p);
size_t mle_ws_bytes(int grid, int n, int p, bool use_smem);
int mle_blocks_per_sm(int n, int p, bool use_smem);
cudaError_t launch_mle(const MleArgs &a, int grid, cudaStream_t st);

// diag.cu (rows a3, a4, a5 alone)
cudaError_t launch_alc_scores(int B, int j, int p, int nc, const double *Xj, const double *Kinv, const double *cands,
                              const int32_t *cand_idx, const double *x, double rtheta, double eta, double *delta,
                              int32_t *best, double *gap, cudaStream_t st);
// alc_scores_gemm.cu (row f4): a3 alone as a dense FP64 DMMA contraction, j <= LAGP_SCORES_JMAX
size_t alc_scores_gemm_smem(int j, int p);
size_t alc_scores_gemm_ws_bytes(int B, int j, int nc);
cudaError_t launch_alc_scores_gemm(int B, int j, int p, int nc, const double *Xj, const double *Kinv,
                                   const double *cands, const int32_t *cand_idx, const double *x, double rtheta,
                                   double eta, double *delta, int32_t *best, double *gap, void *ws, cudaStream_t st,
                                   int *launches);
cudaError_t launch_pinv_update(int B, int j, const double *Kinv, const double *k, double kdiag, double *Kout,
                               cudaStream_t st);
cudaError_t launch_exp_nonpos(const double *x, double *y, int64_t n, cudaStream_t st);
struct SepScale {
    double s[16];  // 1/sqrt(theta_k), k < p <= LAGP_PMAX
};
cudaError_t launch_sep_scale(const double *x, int64_t rows, int p, const SepScale &s, double *out, cudaStream_t st);
cudaError_t launch_predict(int B, int n, int p, const double *Xn, const double *Yn, const double *x, double rtheta,
                           double eta, double *mean, double *s2, double *var, cudaStream_t st);

}  // namespace lagp
