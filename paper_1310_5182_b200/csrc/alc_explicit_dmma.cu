// alc_explicit_dmma.cu — the explicit-K_j^{-1} local-design kernel (rows
// a2 + a3 + a4 + a5 fused, LAGP_ALC_EXPLICIT) with the quadratic form on the
// FP64 tensor path: mma.sync.aligned.m8n8k4.row.col.f64 (SASS DMMA.8x8x4).
// Used for n <= 64; alc_explicit.cu (register-blocked DFMA) covers larger n.
//
// Per step j, for a tile of T = 64 pool candidates (Eq (5)-(6)):
//   V = K_j^{-1} [k_c1 .. k_cT]          (jpad8 × T, DMMA; each warp owns 8 columns)
//   q_c   = sum_a k_c[a] V[a][c]         (= k_c^T K_j^{-1} k_c, Fig 3 steps 3-4)
//   cov_c = kappa_c - sum_a w[a] k_c[a]  (w = K_j^{-1} h; numerator of Eq (5), R1)
//   Delta_c = cov_c^2 / (1 + eta - q_c) ; argmax, ties to the lowest global row (R7)
// Fragment layouts (PTX ISA, mma.m8n8k4 .f64): A a0 = A[g][k], B b0 = B[k][g],
// C {c0,c1} = C[g][2k], C[g][2k+1] with g = lane>>2, k = lane&3.
// Shared-memory strides are chosen so every fragment load is conflict-free:
// K^{-1} row stride KL ≡ 4 (mod 16) doubles, k_c tile row stride 68 ≡ 4 (mod 16).
#include <cuda_runtime.h>
#include <stdlib.h>

#include "block_ops.cuh"
#include "launch.h"

namespace lagp {

// NWD warps per CTA (8: two CTAs per SM; 16: one CTA per SM, so that the per-CTA k_c
// caches of all resident CTAs — 148 x n x N' doubles — stay inside L2); each warp owns 8
// candidate columns of a tile of DM_T = 8 NWD candidates.
// Tile row stride DM_T + 4 (doubles). 64-bit shared loads are served per half-warp, so
// the B fragment tile[4s+k][c0+g] (k, g < 4 within a half-warp) is conflict-free iff
// TL ≡ 4 (mod 16); the same rule gives KL ≡ 4 (mod 16) for the A fragment.
__host__ __device__ constexpr int dm_tl(int nwd) { return 8 * nwd + 4; }

__host__ __device__ inline int dm_kl(int n) {
    int kl = (n + 3) & ~3;
    while ((kl & 15) != 4) kl += 4;
    return kl;
}
__host__ __device__ inline int dm_kr(int n) { return (n + 7) & ~7; }
__host__ __device__ inline int dm_vl(int n) { return dm_kr(n) > dm_kl(n) ? dm_kr(n) : dm_kl(n); }
// smem (doubles): K kr*kl | tiles 2*kr*TL | Xj r4(n*p) | h,w,ks,us,yv 5*vl | red 160
__host__ __device__ inline size_t dm_smem_bytes(int n, int p, int Npad, int nwd) {
    const int kl = dm_kl(n), kr = dm_kr(n);
    (void)Npad;  // kappa_c / chosen live in the CTA's global slab: smem does not grow with N'
    return ((size_t)kr * kl + 2 * (size_t)kr * dm_tl(nwd) + (size_t)((n * p + 3) & ~3) + 5 * (size_t)dm_vl(n) + 160) *
           sizeof(double);
}

__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

// The per-CTA k_c caches (n x N' doubles each) are the kernel's working set in L2;
// their loads and stores carry an evict_last policy so that the streaming inputs (pool
// indices, the rows of X) are evicted first.
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void cp_async16_dm(void *smem, const void *gmem, uint64_t pol) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "l"(pol));
}
__device__ __forceinline__ void st_keep(double *p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// out[a] = sum_b K[a][b] v[b] (row-major, stride kl); warp per row, lanes over b.
__device__ __forceinline__ void rm_matvec(const double *K, int kl, int rows, int cols, const double *v, double *out) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int a = wid; a < rows; a += nw) {
        double acc = 0.0;
        for (int b = lane; b < cols; b += 32) acc = fma(K[a * kl + b], v[b], acc);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) out[a] = acc;
    }
    __syncthreads();
}

// a4 (Eq (6)) on row-major K^{-1}: u = K^{-1}k, s = kdiag - k^T u,
// K_{j+1}^{-1} = [[K^{-1} + u u^T (1/s), -u/s], [-u^T/s, 1/s]] — bitwise symmetric.
__device__ __forceinline__ double rm_append(double *K, int kl, int j, const double *k, double kdiag, double *u,
                                            double *red) {
    rm_matvec(K, kl, j, j, k, u);
    double part = 0.0;
    for (int a = threadIdx.x; a < j; a += blockDim.x) part = fma(k[a], u[a], part);
    const double s = kdiag - block_sum(part, red);
    const double rs = 1.0 / s;
    for (int e = threadIdx.x; e < j * j; e += blockDim.x) {
        const int a = e / j, b = e - a * j;
        K[a * kl + b] += (u[a] * u[b]) * rs;
    }
    for (int a = threadIdx.x; a < j; a += blockDim.x) {
        const double v = -(u[a] * rs);
        K[a * kl + j] = v;
        K[j * kl + a] = v;
    }
    if (threadIdx.x == 0) K[j * kl + j] = rs;
    __syncthreads();
    return s;
}

template <int NWD>
__global__ void __launch_bounds__(32 * NWD, 16 / NWD)
alc_explicit_dmma_kernel(AlcArgs A) {
    constexpr int DM_T = 8 * NWD, DM_TL = dm_tl(NWD);
    extern __shared__ __align__(16) double sm[];
    const int n = A.n, p = A.p, Np = A.Nprime, Npad = A.Npad;
    const int kl = dm_kl(n), kr = dm_kr(n);
    double *K = sm;
    double *tbuf = K + kr * kl;
    const int tsz = kr * DM_TL;
    double *Xj = tbuf + 2 * tsz;
    double *h = Xj + ((n * p + 3) & ~3);
    const int vl = dm_vl(n);  // vector length covers both K rows (kr) and columns (kl)
    double *w = h + vl;
    double *ks = w + vl;
    double *us = ks + vl;
    double *yv = us + vl;
    double *red = yv + vl;
    __shared__ double xq[LAGP_PMAX];
    __shared__ uint32_t fl_s;

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int g = lane >> 2, kq = lane & 3;
    double *cache = A.cache + (size_t)blockIdx.x * A.cache_stride;
    double *coords = A.coords + (size_t)blockIdx.x * (p + 2) * Npad;  // [p][Npad] coords | kap | chosen
    double *kap = coords + (size_t)p * Npad;
    unsigned char *chosen = reinterpret_cast<unsigned char *>(kap + Npad);
    const double eta = A.eta;
    const int G = n - A.n0;
    const uint64_t pol = l2_evict_last();

    for (int64_t xi = blockIdx.x; xi < A.M; xi += gridDim.x) {
        const double rth = A.theta_vec ? 1.0 / A.theta_vec[xi] : A.rtheta;  // per-location theta (Fig 1 step 4)
        const int32_t *pool = A.pool + xi * (int64_t)Np;
        int32_t *idx = A.idx_out + xi * (int64_t)n;
        if (tid < p) xq[tid] = A.XX[xi * p + tid];
        if (tid == 0) fl_s = 0;
        for (int e = tid; e < kr * kl; e += blockDim.x) K[e] = 0.0;
        for (int e = tid; e < vl; e += blockDim.x) w[e] = 0.0;
        __syncthreads();
        // ---- gather the pool (SoA coords in the slab), kappa_c, chosen mask
        for (int c = tid; c < Np; c += blockDim.x) {
            const double *xr = A.X + (int64_t)pool[c] * p;
            for (int k = 0; k < p; k++) coords[k * Npad + c] = xr[k];
            kap[c] = corr_from_d2(sqdist_fma(xr, xq, p), rth);
            chosen[c] = (c < A.n0) ? 1 : 0;
        }
        for (int t = tid; t < n; t += blockDim.x) idx[t] = (t < A.n0) ? pool[t] : -1;
        if (A.gap_out)
            for (int t = tid; t < G; t += blockDim.x) A.gap_out[xi * G + t] = __longlong_as_double(0x7ff8000000000000LL);
        for (int e = tid; e < A.n0 * p; e += blockDim.x) Xj[e] = A.X[(int64_t)pool[e / p] * p + (e % p)];
        __syncthreads();

        // ---- a2: K_{n0}^{-1} by partitioned-inverse appends of the NN-ordered X_{n0}
        for (int t = 0; t < A.n0; t++) {
            if (tid < t) ks[tid] = corr_from_d2(sqdist_fma(Xj + tid * p, Xj + t * p, p), rth);
            if (tid == 0) h[t] = corr_from_d2(sqdist_fma(Xj + t * p, xq, p), rth);
            __syncthreads();
            if (t == 0) {
                if (tid == 0) K[0] = 1.0 / (1.0 + eta);
            } else {
                double s = rm_append(K, kl, t, ks, 1.0 + eta, us, red);
                if (!(s > 0.0) && tid == 0) fl_s |= LAGP_FLAG_NONFINITE;
            }
            for (int c = tid; c < Np; c += blockDim.x)
                st_keep(cache + (size_t)t * Npad + c, corr_from_d2(sqdist_fma_strided(Xj + t * p, coords + c, Npad, p), rth),
                        pol);
            __syncthreads();
        }
        rm_matvec(K, kl, A.n0, A.n0, h, w);

        // ---- greedy ALC loop (Fig 1 step 2(b)), j = current design size
        int j = A.n0;
        for (; j < n; j++) {
            const int nks = (j + 3) >> 2;  // k-steps of 4
            const int nrb = (j + 7) >> 3;  // row blocks of 8
            const int ntiles = (Np + DM_T - 1) / DM_T;
            for (int e = tid; e < (8 * nrb - j) * DM_TL; e += blockDim.x) {
                tbuf[j * DM_TL + e] = 0.0;
                tbuf[tsz + j * DM_TL + e] = 0.0;
            }
            auto load_tile = [&](int t, double *dst) {
                const int t0 = t * DM_T;
                for (int e = tid; e < j * (DM_T / 2); e += blockDim.x) {
                    const int a = e / (DM_T / 2), c2 = e % (DM_T / 2);
                    cp_async16_dm(dst + a * DM_TL + 2 * c2, cache + (size_t)a * Npad + t0 + 2 * c2, pol);
                }
                asm volatile("cp.async.commit_group;\n" ::);
            };
            load_tile(0, tbuf);
            Top2 best;
            best.init();
            bool sentinel = false, nonfinite = false;
            for (int t = 0; t < ntiles; t++) {
                const double *tile = tbuf + (t & 1) * tsz;
                if (t + 1 < ntiles) {
                    load_tile(t + 1, tbuf + ((t + 1) & 1) * tsz);
                    asm volatile("cp.async.wait_group 1;\n" ::);
                } else {
                    asm volatile("cp.async.wait_group 0;\n" ::);
                }
                __syncthreads();
                const int c0 = wid * 8;
                double q0 = 0.0, q1 = 0.0, v0 = 0.0, v1 = 0.0;
                for (int rb = 0; rb < nrb; rb += 2) {
                    const bool two = (rb + 1) < nrb;  // warp-uniform
                    double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
                    const double *Ka = K + (8 * rb + g) * kl + kq;
                    const double *Tb = tile + kq * DM_TL + c0 + g;
                    if (two) {
#pragma unroll 4
                        for (int s4 = 0; s4 < nks; s4++) {
                            const double b = Tb[4 * s4 * DM_TL];
                            dmma884(a00, a01, Ka[4 * s4], b);
                            dmma884(a10, a11, Ka[8 * kl + 4 * s4], b);
                        }
                    } else {
#pragma unroll 4
                        for (int s4 = 0; s4 < nks; s4++) dmma884(a00, a01, Ka[4 * s4], Tb[4 * s4 * DM_TL]);
                    }
                    {
                        const int row = 8 * rb + g;
                        const double2 tv = *reinterpret_cast<const double2 *>(tile + row * DM_TL + c0 + 2 * kq);
                        const double wv = w[row];
                        q0 = fma(tv.x, a00, q0);
                        q1 = fma(tv.y, a01, q1);
                        v0 = fma(wv, tv.x, v0);
                        v1 = fma(wv, tv.y, v1);
                    }
                    if (two) {
                        const int row = 8 * rb + 8 + g;
                        const double2 tv = *reinterpret_cast<const double2 *>(tile + row * DM_TL + c0 + 2 * kq);
                        const double wv = w[row];
                        q0 = fma(tv.x, a10, q0);
                        q1 = fma(tv.y, a11, q1);
                        v0 = fma(wv, tv.x, v0);
                        v1 = fma(wv, tv.y, v1);
                    }
                }
                // sum over the 8 row lanes g (lane bits 2..4)
#pragma unroll
                for (int off = 4; off < 32; off <<= 1) {
                    q0 += __shfl_xor_sync(0xffffffffu, q0, off);
                    q1 += __shfl_xor_sync(0xffffffffu, q1, off);
                    v0 += __shfl_xor_sync(0xffffffffu, v0, off);
                    v1 += __shfl_xor_sync(0xffffffffu, v1, off);
                }
                if (g == 0) {
                    const int t0 = t * DM_T;
#pragma unroll
                    for (int i = 0; i < 2; i++) {
                        const int pc = t0 + c0 + 2 * kq + i;
                        if (pc < Np && !chosen[pc]) {
                            const double s = 1.0 + eta - (i ? q1 : q0);
                            if (!(s > kSMin)) {
                                sentinel = true;
                            } else {
                                const double cv = kap[pc] - (i ? v1 : v0);
                                const double dl = cv * cv / s;
                                if (!isfinite(dl)) nonfinite = true;
                                else if (dl >= best.d1) best.push(dl, pool[pc], pc);
                                else if (dl > best.d2) best.d2 = dl;
                            }
                        }
                    }
                }
                __syncthreads();  // buffer (t & 1) is reloaded at iteration t + 1
            }
            if (sentinel) atomicOr(&fl_s, (uint32_t)LAGP_FLAG_SENTINEL);
            if (nonfinite) atomicOr(&fl_s, (uint32_t)LAGP_FLAG_NONFINITE);
            best = block_top2(best, red);
            if (best.pos < 0) {
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
                h[j] = kap[best.pos];
            }
            // ---- a4: append x* (its k_* is the cached column)
            for (int a = tid; a < j; a += blockDim.x) ks[a] = cache[(size_t)a * Npad + best.pos];
            for (int k = tid; k < p; k += blockDim.x) Xj[j * p + k] = coords[k * Npad + best.pos];
            __syncthreads();
            double s = rm_append(K, kl, j, ks, 1.0 + eta, us, red);
            if (!(s > 0.0) && tid == 0) fl_s |= LAGP_FLAG_NONFINITE;
            rm_matvec(K, kl, j + 1, j + 1, h, w);
            if (j + 1 < n)
                for (int c = tid; c < Np; c += blockDim.x)
                    st_keep(cache + (size_t)j * Npad + c,
                            corr_from_d2(sqdist_fma_strided(Xj + j * p, coords + c, Npad, p), rth), pol);
            __syncthreads();
        }

        // ---- a5: predict on D_j, fresh Cholesky in the K buffer (row-major, ld = kl)
        for (int t = tid; t < j; t += blockDim.x) yv[t] = A.Z[idx[t]];
        __syncthreads();
        double mu, sc, vr;
        bool ok = block_predict(K, kl, j, p, Xj, yv, h, rth, eta, us, ks, red, &mu, &sc, &vr);
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

// LAGP_DM_WARPS=16 (A/B): one 16-warp CTA per SM instead of two 8-warp CTAs
static int dm_warps() {
    const char *ev = getenv("LAGP_DM_WARPS");
    return (ev && ev[0] == '1') ? 16 : 8;
}

template <int NWD>
static cudaError_t dm_launch_t(const AlcArgs &a, int grid, cudaStream_t st) {
    size_t smem = dm_smem_bytes(a.n, a.p, a.Npad, NWD);
    cudaError_t e =
        cudaFuncSetAttribute(alc_explicit_dmma_kernel<NWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    alc_explicit_dmma_kernel<NWD><<<grid, 32 * NWD, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_alc_explicit_dmma(const AlcArgs &a, int grid, cudaStream_t st) {
    return dm_warps() == 8 ? dm_launch_t<8>(a, grid, st) : dm_launch_t<16>(a, grid, st);
}

template <int NWD>
static int dm_bps_t(int n, int p, int Npad) {
    int nb = 0;
    size_t smem = dm_smem_bytes(n, p, Npad, NWD);
    if (cudaFuncSetAttribute(alc_explicit_dmma_kernel<NWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess) {
        cudaGetLastError();  // do not leave a sticky error for the next launch check
        return 0;
    }
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, alc_explicit_dmma_kernel<NWD>, 32 * NWD, smem) !=
        cudaSuccess) {
        cudaGetLastError();
        nb = 0;
    }
    return nb;
}

int alc_explicit_dmma_blocks_per_sm(int n, int p, int Npad) {
    return dm_warps() == 8 ? dm_bps_t<8>(n, p, Npad) : dm_bps_t<16>(n, p, Npad);
}

}  // namespace lagp
