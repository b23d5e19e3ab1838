// diag.cu — single-row kernels behind the diagnostic entry points
// laGP_alc_scores (a3), laGP_pinv_update (a4) and laGP_predict (a5). They let
// each row be parity-tested alone against the oracle; the product path runs the
// same algebra fused in alc_explicit.cu / alc_incremental.cu.
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "launch.h"

namespace lagp {

constexpr int DIAG_THREADS = 256;

// the table exponential of the incremental kernels, elementwise (laGP_exp_nonpos)
__global__ void exp_nonpos_kernel(const double *__restrict__ x, double *__restrict__ y, int64_t n) {
    __shared__ double tab[16];
    if (threadIdx.x < 16) tab[threadIdx.x] = c_exp2_16[threadIdx.x];
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = exp_nonpos_tab(x[i], tab);
}

// row f3: x~[i][k] = x[i][k] * s[k] (s_k = 1/sqrt(theta_k), formed on the host),
// the rescaling that turns the separable correlation into the isotropic one
__global__ void sep_scale_kernel(const double *__restrict__ x, int64_t rows, int p, SepScale s,
                                 double *__restrict__ out) {
    const int64_t total = rows * p;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = __dmul_rn(x[e], s.s[e % p]);
}

cudaError_t launch_sep_scale(const double *x, int64_t rows, int p, const SepScale &s, double *out, cudaStream_t st) {
    const int64_t total = rows * p;
    if (total <= 0) return cudaSuccess;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    sep_scale_kernel<<<(int)blocks, 256, 0, st>>>(x, rows, p, s, out);
    return cudaGetLastError();
}

cudaError_t launch_exp_nonpos(const double *x, double *y, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    exp_nonpos_kernel<<<(int)blocks, 256, 0, st>>>(x, y, n);
    return cudaGetLastError();
}

// a3 alone (Fig 2 I/O): one CTA per location, one warp per candidate.
//   w = K^{-1} h (h = k_j(x)), s_c = 1 + g - k_c^T K^{-1} k_c, cov_c = kappa_c - w^T k_c,
//   Delta_c = cov_c^2 / s_c (Eq (5)-(6) closed form, R1); -inf if s_c <= 1e-12.
__global__ void __launch_bounds__(DIAG_THREADS)
alc_scores_kernel(int j, int p, int nc, const double *__restrict__ Xj, const double *__restrict__ Kinv,
                  const double *__restrict__ cands, const int32_t *__restrict__ cand_idx,
                  const double *__restrict__ xref, double rtheta, double eta, double *__restrict__ delta_out,
                  int32_t *__restrict__ best_out, double *__restrict__ gap_out) {
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    double *K = sm;                  // j*j
    double *xs = K + (size_t)j * j;  // j*p
    double *h = xs + (size_t)j * p;  // j
    double *w = h + j;               // j
    double *kw = w + j;              // 8 warps × j
    double *red = kw + 8 * j;        // 160
    __shared__ double xq[LAGP_PMAX];
    const double *Kb = Kinv + (size_t)b * j * j;
    for (int e = tid; e < j * j; e += blockDim.x) K[e] = Kb[e];
    for (int e = tid; e < j * p; e += blockDim.x) xs[e] = Xj[(size_t)b * j * p + e];
    if (tid < p) xq[tid] = xref[(size_t)b * p + tid];
    __syncthreads();
    for (int a = tid; a < j; a += blockDim.x) h[a] = corr_from_d2(sqdist_fma(xs + a * p, xq, p), rtheta);
    __syncthreads();
    block_matvec(K, j, j, h, w);
    Top2 best;
    best.init();
    double *kc = kw + wid * j;
    for (int c = wid; c < nc; c += blockDim.x >> 5) {
        const double *xc = cands + ((size_t)b * nc + c) * p;
        for (int a = lane; a < j; a += 32) kc[a] = corr_from_d2(sqdist_fma(xs + a * p, xc, p), rtheta);
        __syncwarp();
        double q = 0.0, cv = 0.0;
        for (int a = lane; a < j; a += 32) {
            double acc = 0.0;
            for (int t = 0; t < j; t++) acc = fma(K[a * j + t], kc[t], acc);
            q = fma(kc[a], acc, q);
            cv = fma(w[a], kc[a], cv);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            q += __shfl_xor_sync(0xffffffffu, q, off);
            cv += __shfl_xor_sync(0xffffffffu, cv, off);
        }
        const double s = 1.0 + eta - q;
        double dl = -INFINITY;
        if (s > kSMin) {
            double kap = corr_from_d2(sqdist_fma(xc, xq, p), rtheta);
            double cov = kap - cv;
            dl = cov * cov / s;
        }
        if (lane == 0) {
            if (delta_out) delta_out[(size_t)b * nc + c] = dl;
            if (dl > -INFINITY) best.push(dl, cand_idx[(size_t)b * nc + c], c);
        }
        __syncwarp();
    }
    best = block_top2(best, red);
    if (tid == 0) {
        best_out[b] = best.pos;
        if (gap_out) gap_out[b] = (best.pos >= 0) ? top2_gap(best.d1, best.d2) : __longlong_as_double(0x7ff8000000000000LL);
    }
}

// a4 alone: K_{j+1}^{-1} from K_j^{-1}, one CTA per matrix.
__global__ void __launch_bounds__(DIAG_THREADS)
pinv_update_kernel(int j, const double *__restrict__ Kinv, const double *__restrict__ k, double kdiag,
                   double *__restrict__ Kout) {
    extern __shared__ __align__(16) double sm[];
    const int J = j + 1, b = blockIdx.x, tid = threadIdx.x;
    double *K = sm;            // J*J (ld = J)
    double *kv = K + J * J;    // J
    double *u = kv + J;        // J
    double *red = u + J;       // 160
    for (int e = tid; e < J * J; e += blockDim.x) {
        int a = e / J, c = e - a * J;
        K[e] = (a < j && c < j) ? Kinv[(size_t)b * j * j + a * j + c] : 0.0;
    }
    for (int a = tid; a < j; a += blockDim.x) kv[a] = k[(size_t)b * j + a];
    __syncthreads();
    pinv_append(K, J, j, kv, kdiag, u, red);
    for (int e = tid; e < J * J; e += blockDim.x) Kout[(size_t)b * J * J + e] = K[e];
}

// a5 alone: predict from a given local design, one CTA per location.
__global__ void __launch_bounds__(DIAG_THREADS)
predict_kernel(int n, int p, const double *__restrict__ Xn, const double *__restrict__ Yn,
               const double *__restrict__ xref, double rtheta, double eta, double *__restrict__ mean,
               double *__restrict__ s2, double *__restrict__ var) {
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.x, tid = threadIdx.x;
    double *A = sm;                 // n*n
    double *xs = A + (size_t)n * n; // n*p
    double *y = xs + (size_t)n * p; // n
    double *h = y + n;              // n
    double *y1 = h + n;             // n
    double *y2 = y1 + n;            // n
    double *red = y2 + n;           // 160
    __shared__ double xq[LAGP_PMAX];
    for (int e = tid; e < n * p; e += blockDim.x) xs[e] = Xn[(size_t)b * n * p + e];
    for (int a = tid; a < n; a += blockDim.x) y[a] = Yn[(size_t)b * n + a];
    if (tid < p) xq[tid] = xref[(size_t)b * p + tid];
    __syncthreads();
    for (int a = tid; a < n; a += blockDim.x) h[a] = corr_from_d2(sqdist_fma(xs + a * p, xq, p), rtheta);
    __syncthreads();
    double mu, sc, vr;
    block_predict(A, n, n, p, xs, y, h, rtheta, eta, y1, y2, red, &mu, &sc, &vr);
    if (tid == 0) {
        mean[b] = mu;
        s2[b] = sc;
        if (var) var[b] = vr;
    }
}

cudaError_t launch_alc_scores(int B, int j, int p, int nc, const double *Xj, const double *Kinv, const double *cands,
                              const int32_t *cand_idx, const double *x, double rtheta, double eta, double *delta,
                              int32_t *best, double *gap, cudaStream_t st) {
    size_t smem = ((size_t)j * j + (size_t)j * p + 2 * (size_t)j + 8 * (size_t)j + 160) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(alc_scores_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    alc_scores_kernel<<<B, DIAG_THREADS, smem, st>>>(j, p, nc, Xj, Kinv, cands, cand_idx, x, rtheta, eta, delta, best,
                                                    gap);
    return cudaGetLastError();
}

cudaError_t launch_pinv_update(int B, int j, const double *Kinv, const double *k, double kdiag, double *Kout,
                               cudaStream_t st) {
    const int J = j + 1;
    size_t smem = ((size_t)J * J + 2 * (size_t)J + 160) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(pinv_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    pinv_update_kernel<<<B, DIAG_THREADS, smem, st>>>(j, Kinv, k, kdiag, Kout);
    return cudaGetLastError();
}

cudaError_t launch_predict(int B, int n, int p, const double *Xn, const double *Yn, const double *x, double rtheta,
                           double eta, double *mean, double *s2, double *var, cudaStream_t st) {
    size_t smem = ((size_t)n * n + (size_t)n * p + 4 * (size_t)n + 160) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(predict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    predict_kernel<<<B, DIAG_THREADS, smem, st>>>(n, p, Xn, Yn, x, rtheta, eta, mean, s2, var);
    return cudaGetLastError();
}

}  // namespace lagp
