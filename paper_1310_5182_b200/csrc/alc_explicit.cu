// alc_explicit.cu — rows a2 + a3 + a4 + a5 fused, paper formulation
// (LAGP_ALC_EXPLICIT): one CTA owns one predictive location x at a time
// (persistent grid: CTA b handles x = b, b + grid, ...) and runs the whole
// Fig 1 step 2 j-loop plus the step-5 prediction with the local GP
// state resident in shared memory — no host round trip and no per-step launch
// (the paper issued one launch plus PCIe copies per (x, j)).
//
// Per step j (Eq (5)-(6); Fig 3 steps 2-8):
//   s_c   = 1 + eta - k_c^T K_j^{-1} k_c        (m_j^{-1}(x_c), Fig 3 steps 3-5)
//   cov_c = kappa_c - w^T k_c, w = K_j^{-1} h   (h = k_j(x); numerator of Eq (5)
//                                                 in closed form, reading R1)
//   Delta_c = cov_c^2 / s_c ; argmax with ties to the lowest global row (R7).
// The quadratic form is evaluated tile by tile as the small dense product
// V = K_j^{-1} [k_c1 ... k_cT] with a 4×4 register-blocked FP64 FMA micro-kernel
// (K_j^{-1} read row-wise thanks to symmetry, the k_c tile column-contiguous:
// both conflict-free, broadcast-heavy shared-memory reads — the B200 analogue of
// Fig 3's "work column-wise with K^{-1}" coalescing note).
// k_c is cached: one new row K(x_{j-1}, x_c) per step is appended to a per-CTA
// slab in HBM (row-major over candidates), instead of recomputing j
// exponentials per candidate per step as Fig 3 step 2 does.
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "launch.h"

namespace lagp {

constexpr int ALC_THREADS = 256;


// shared-memory carve-up (doubles): Kinv ld*ld | tile TILE | Xj n*p | h ld | w ld | ks ld | us ld | y ld | red 160
__host__ __device__ inline int alc_tile_elems(int ld) { return ld <= 64 ? 4096 : ld * 64; }
__host__ __device__ inline size_t alc_smem_doubles(int ld, int n, int p) {
    return (size_t)ld * ld + alc_tile_elems(ld) + (size_t)n * p + 5 * (size_t)ld + 160;
}

// new cache row a: cache[a][c] = K(Xj[a], x_c) for every pool position c
__device__ __forceinline__ void cache_row(double *cache_a, const double *xa, const double *coords, int Nprime,
                                          int p, double rtheta) {
    for (int c = threadIdx.x; c < Nprime; c += blockDim.x)
        cache_a[c] = corr_from_d2(sqdist_fma_strided(xa, coords + c, Nprime, p), rtheta);
}

__global__ void __launch_bounds__(ALC_THREADS)
alc_explicit_kernel(AlcArgs A) {
    extern __shared__ __align__(16) double sm[];
    const int ld = A.ld, n = A.n, p = A.p, Np = A.Nprime;
    double *Kinv = sm;
    double *tile = Kinv + ld * ld;
    double *Xj = tile + alc_tile_elems(ld);
    double *h = Xj + n * p;
    double *w = h + ld;
    double *ks = w + ld;
    double *us = ks + ld;
    double *yv = us + ld;
    double *red = yv + ld;  // 160 doubles of reduction scratch
    __shared__ double xq[LAGP_PMAX];
    __shared__ uint32_t fl_s;

    const int tid = threadIdx.x;
    double *cache = A.cache + (size_t)blockIdx.x * n * Np;
    double *coords = A.coords + (size_t)blockIdx.x * p * Np;
    double *kap = A.kap + (size_t)blockIdx.x * Np;
    unsigned char *chosen = A.chosen + (size_t)blockIdx.x * Np;
    const double rth = A.rtheta, eta = A.eta;
    const int G = n - A.n0;

    for (int64_t xi = blockIdx.x; xi < A.M; xi += gridDim.x) {
        const int32_t *pool = A.pool + xi * (int64_t)Np;
        int32_t *idx = A.idx_out + xi * (int64_t)n;
        if (tid < p) xq[tid] = A.XX[xi * p + tid];
        if (tid == 0) fl_s = 0;
        for (int e = tid; e < ld * ld; e += blockDim.x) Kinv[e] = 0.0;
        __syncthreads();
        // ---- gather the pool (SoA coords), kappa_c, chosen mask
        for (int c = tid; c < Np; c += blockDim.x) {
            const double *xr = A.X + (int64_t)pool[c] * p;
            for (int k = 0; k < p; k++) coords[k * Np + c] = xr[k];
            kap[c] = corr_from_d2(sqdist_fma(xr, xq, p), rth);
            chosen[c] = (c < A.n0) ? 1 : 0;
        }
        for (int t = tid; t < n; t += blockDim.x) idx[t] = (t < A.n0) ? pool[t] : -1;
        if (A.gap_out)
            for (int t = tid; t < G; t += blockDim.x) A.gap_out[xi * G + t] = __longlong_as_double(0x7ff8000000000000LL);
        for (int e = tid; e < A.n0 * p; e += blockDim.x) Xj[e] = A.X[(int64_t)pool[e / p] * p + (e % p)];
        __syncthreads();

        // ---- a2: K_{n0}^{-1} by successive partitioned-inverse appends of the
        // NN-ordered initial design (same algebra as a4), h, w, cache rows
        for (int t = 0; t < A.n0; t++) {
            if (tid < t) ks[tid] = corr_from_d2(sqdist_fma(Xj + tid * p, Xj + t * p, p), rth);
            __syncthreads();
            if (t == 0) {
                if (tid == 0) Kinv[0] = 1.0 / (1.0 + eta);
                __syncthreads();
            } else {
                double s = pinv_append(Kinv, ld, t, ks, 1.0 + eta, us, red);
                if (!(s > 0.0) && tid == 0) fl_s |= LAGP_FLAG_NONFINITE;
            }
            if (tid == 0) h[t] = corr_from_d2(sqdist_fma(Xj + t * p, xq, p), rth);
            cache_row(cache + (size_t)t * Np, Xj + t * p, coords, Np, p, rth);
            __syncthreads();
        }
        block_matvec(Kinv, ld, A.n0, h, w);
        __threadfence_block();
        __syncthreads();

        // ---- greedy ALC loop (Fig 1 step 2(b)), j = current design size
        int j = A.n0;
        for (; j < n; j++) {
            const int nab = (j + 3) >> 2;                       // a-blocks of 4 rows
            const int AB = nab <= 1 ? 1 : nab <= 2 ? 2 : nab <= 4 ? 4 : nab <= 8 ? 8 : 16;
            const int CB = ALC_THREADS / AB;                     // c-blocks of 4 candidates
            const int T = 4 * CB;                                // candidates per tile
            const int jpad = 4 * nab;
            const int ab = tid % AB, cb = tid / AB;
            Top2 best;
            best.init();
            bool sentinel = false, nonfinite = false;
            for (int t0 = 0; t0 < Np; t0 += T) {
                // stage the k_c tile [jpad][T] (zero padded) from the cache slab
                for (int e = tid; e < jpad * T; e += blockDim.x) {
                    int a = e / T, c = e - a * T;
                    int pc = t0 + c;
                    tile[e] = (a < j && pc < Np) ? cache[(size_t)a * Np + pc] : 0.0;
                }
                __syncthreads();
                double ps[4] = {0.0, 0.0, 0.0, 0.0}, pcv[4] = {0.0, 0.0, 0.0, 0.0};
                for (int ag = ab; ag < nab; ag += AB) {
                    double acc[4][4];
#pragma unroll
                    for (int r = 0; r < 4; r++)
#pragma unroll
                        for (int c = 0; c < 4; c++) acc[r][c] = 0.0;
                    const double *kcol = Kinv + 4 * ag;
                    const double *tcol = tile + 4 * cb;
#pragma unroll 2
                    for (int b = 0; b < j; b++) {
                        const double2 k01 = *reinterpret_cast<const double2 *>(kcol + b * ld);
                        const double2 k23 = *reinterpret_cast<const double2 *>(kcol + b * ld + 2);
                        const double2 t01 = *reinterpret_cast<const double2 *>(tcol + b * T);
                        const double2 t23 = *reinterpret_cast<const double2 *>(tcol + b * T + 2);
                        const double kr[4] = {k01.x, k01.y, k23.x, k23.y};
                        const double tc[4] = {t01.x, t01.y, t23.x, t23.y};
#pragma unroll
                        for (int r = 0; r < 4; r++)
#pragma unroll
                            for (int c = 0; c < 4; c++) acc[r][c] = fma(kr[r], tc[c], acc[r][c]);
                    }
#pragma unroll
                    for (int r = 0; r < 4; r++) {
                        const int a = 4 * ag + r;
                        const double2 t01 = *reinterpret_cast<const double2 *>(tcol + a * T);
                        const double2 t23 = *reinterpret_cast<const double2 *>(tcol + a * T + 2);
                        const double tc[4] = {t01.x, t01.y, t23.x, t23.y};
                        const double wa = (a < j) ? w[a] : 0.0;
#pragma unroll
                        for (int c = 0; c < 4; c++) {
                            ps[c] = fma(tc[c], acc[r][c], ps[c]);
                            pcv[c] = fma(wa, tc[c], pcv[c]);
                        }
                    }
                }
                // reduce over the AB lanes that share this c-block (aligned lane groups)
                for (int off = AB >> 1; off > 0; off >>= 1) {
#pragma unroll
                    for (int c = 0; c < 4; c++) {
                        ps[c] += __shfl_xor_sync(0xffffffffu, ps[c], off);
                        pcv[c] += __shfl_xor_sync(0xffffffffu, pcv[c], off);
                    }
                }
                if (ab == 0) {
#pragma unroll
                    for (int c = 0; c < 4; c++) {
                        const int pc = t0 + 4 * cb + c;
                        if (pc < Np && !chosen[pc]) {
                            const double s = 1.0 + eta - ps[c];
                            if (!(s > kSMin)) {
                                sentinel = true;
                            } else {
                                const double cv = kap[pc] - pcv[c];
                                const double dl = cv * cv / s;
                                if (isfinite(dl)) best.push(dl, pool[pc], pc);
                                else nonfinite = true;
                            }
                        }
                    }
                }
                __syncthreads();
            }
            if (sentinel) atomicOr(&fl_s, (uint32_t)LAGP_FLAG_SENTINEL);
            if (nonfinite) atomicOr(&fl_s, (uint32_t)LAGP_FLAG_NONFINITE);
            best = block_top2(best, red);
            if (best.pos < 0) {  // every remaining candidate excluded
                if (tid == 0) fl_s |= LAGP_FLAG_EXHAUSTED;
                __syncthreads();
                break;
            }
            const double gap = top2_gap(best.d1, best.d2);
            if (tid == 0) {
                if (!(best.d1 > 0.0) || gap < kTieGap) fl_s |= LAGP_FLAG_NEAR_TIE;
                if (A.gap_out) A.gap_out[xi * G + (j - A.n0)] = gap;
                idx[j] = best.i1;
                chosen[best.pos] = 1;
            }
            // ---- a4: append x* = pool[best.pos]; k_* is its cached column
            for (int a = tid; a < j; a += blockDim.x) ks[a] = cache[(size_t)a * Np + best.pos];
            for (int k = tid; k < p; k += blockDim.x) Xj[j * p + k] = coords[k * Np + best.pos];
            if (tid == 0) h[j] = kap[best.pos];
            __syncthreads();
            double s = pinv_append(Kinv, ld, j, ks, 1.0 + eta, us, red);
            if (!(s > 0.0) && tid == 0) fl_s |= LAGP_FLAG_NONFINITE;
            block_matvec(Kinv, ld, j + 1, h, w);
            if (j + 1 < n) cache_row(cache + (size_t)j * Np, Xj + j * p, coords, Np, p, rth);
            __threadfence_block();
            __syncthreads();
        }

        // ---- a5: predict on D_j (j = n unless exhausted), fresh Cholesky
        for (int t = tid; t < j; t += blockDim.x) yv[t] = A.Z[idx[t]];
        __syncthreads();
        double mu, sc, vr;
        bool ok = block_predict(Kinv, ld, j, p, Xj, yv, h, rth, eta, us, ks, red, &mu, &sc, &vr);
        if (tid == 0) {
            uint32_t f = fl_s;
            if (!ok || !isfinite(mu) || !isfinite(sc)) f |= LAGP_FLAG_NONFINITE;
            A.mean[xi] = mu;
            A.s2[xi] = sc;
            if (A.var) A.var[xi] = vr;
            if (A.flags) A.flags[xi] = f;
            if (f & (LAGP_FLAG_EXHAUSTED | LAGP_FLAG_NONFINITE)) atomicAdd(A.n_partial, 1);
        }
        __syncthreads();
    }
}

size_t alc_explicit_smem_bytes(int ld, int n, int p) { return alc_smem_doubles(ld, n, p) * sizeof(double); }

cudaError_t launch_alc_explicit(const AlcArgs &a, int grid, cudaStream_t st) {
    size_t smem = alc_explicit_smem_bytes(a.ld, a.n, a.p);
    cudaError_t e = cudaFuncSetAttribute(alc_explicit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    alc_explicit_kernel<<<grid, ALC_THREADS, smem, st>>>(a);
    return cudaGetLastError();
}

int alc_explicit_blocks_per_sm(int ld, int n, int p) {
    int nb = 0;
    size_t smem = alc_explicit_smem_bytes(ld, n, p);
    cudaFuncSetAttribute(alc_explicit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, alc_explicit_kernel, ALC_THREADS, smem) != cudaSuccess)
        nb = 1;
    return nb > 0 ? nb : 1;
}

}  // namespace lagp
