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
// V = K_j^{-1} [k_c1 ... k_cT] with a 4×4 register-blocked FP64 FMA micro-kernel.
// K_j^{-1} lives in a "planar" layout (two planes of double2 holding rows
// (4q, 4q+1) and (4q+2, 4q+3) of column b next to each other) so that the 4-row
// operand of each thread is two conflict-free LDS.128 — the B200 analogue of
// Fig 3's "work column-wise with K^{-1}" coalescing note.
// k_c is cached: one new row K(x_{j-1}, x_c) per step is appended to a per-CTA
// slab in HBM (row-major over candidates, L2-resident in practice) and tiles are
// streamed into shared memory with cp.async, double-buffered against the FMAs,
// instead of recomputing j exponentials per candidate per step (Fig 3 step 2).
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "launch.h"

namespace lagp {

constexpr int ALC_THREADS = 256;
// doubles per k_c tile buffer: jpad × (T + 2) <= 4·AB × 4·256/AB + 2·128 (row stride
// padded by 16 B so the epilogue's 4-row-strided reads do not all hit one bank)
constexpr int ALC_TILE = 4096 + 256;

// w = K^{-1} h is stored "planar" like K^{-1}: (w[4q], w[4q+1]) in plane 0 and
// (w[4q+2], w[4q+3]) in plane 1, so a thread's 4 entries are 2 conflict-free LDS.128.
__device__ __forceinline__ int wpi(int a, int ld) { return ((a >> 1) & 1) * (ld >> 1) + ((a >> 2) << 1) + (a & 1); }

// K^{-1} element (a, b) in the planar layout (ld = 4·NAB).
__device__ __forceinline__ int kp(int a, int b, int ld) {
    return ((a >> 1) & 1) * (ld * ld / 2) + ((b * (ld >> 2) + (a >> 2)) << 1) + (a & 1);
}

// smem carve-up (doubles): Kp ld*ld | tile 2*ALC_TILE | Xj n*p | h,w,ks,us,yv 5*ld | red 160.
// kappa_c and the chosen mask live in the per-CTA global slab after the pool
// coordinates (read once per candidate per step in the epilogue), so the
// shared-memory footprint does not grow with N' (n = 128 needs 128 KB for K^{-1}).
__host__ __device__ inline size_t alc_smem_bytes(int ld, int n, int p, int Npad) {
    (void)Npad;
    return ((size_t)ld * ld + 2 * ALC_TILE + (size_t)((n * p + 3) & ~3) + 5 * (size_t)ld + 160) * sizeof(double);
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// out[a] = sum_b K[a][b] v[b] for a < rows, b < cols; one warp per row, lanes
// over b reading column a (= row a: K^{-1} is kept exactly symmetric), which is
// contiguous in the planar layout. Deterministic shuffle tree.
__device__ __forceinline__ void kp_matvec(const double *Kp, int ld, int rows, int cols, const double *v,
                                          double *out, bool planar_out = false) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int a = wid; a < rows; a += nw) {
        double acc = 0.0;
        for (int b = lane; b < cols; b += 32) acc = fma(Kp[kp(b, a, ld)], v[b], acc);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) out[planar_out ? wpi(a, ld) : a] = acc;
    }
    __syncthreads();
}

// a4 on the planar K^{-1}: K_{j+1}^{-1} = [[K^{-1} + u u^T / s, -u/s], [-u^T/s, 1/s]],
// u = K^{-1} k, s = kdiag - k^T u. (u_a u_b) * (1/s) is bitwise symmetric.
__device__ __forceinline__ double kp_append(double *Kp, int ld, int j, const double *k, double kdiag, double *u,
                                            double *red) {
    kp_matvec(Kp, ld, j, j, k, u);
    double part = 0.0;
    for (int a = threadIdx.x; a < j; a += blockDim.x) part = fma(k[a], u[a], part);
    const double s = kdiag - block_sum(part, red);
    const double rs = 1.0 / s;
    for (int e = threadIdx.x; e < j * j; e += blockDim.x) {
        const int b = e / j, a = e - b * j;  // consecutive threads walk a: conflict-free
        Kp[kp(a, b, ld)] += (u[a] * u[b]) * rs;
    }
    for (int a = threadIdx.x; a < j; a += blockDim.x) {
        const double v = -(u[a] * rs);
        Kp[kp(a, j, ld)] = v;
        Kp[kp(j, a, ld)] = v;
    }
    if (threadIdx.x == 0) Kp[kp(j, j, ld)] = rs;
    __syncthreads();
    return s;
}

// new cache row a: cache[a][c] = K(Xj[a], x_c) for every pool position c
__device__ __forceinline__ void cache_row(double *cache_a, const double *xa, const double *coords, int Npad, int Np,
                                          int p, double rtheta) {
    for (int c = threadIdx.x; c < Np; c += blockDim.x)
        cache_a[c] = corr_from_d2(sqdist_fma_strided(xa, coords + c, Npad, p), rtheta);
}

__global__ void __launch_bounds__(ALC_THREADS, 2)
alc_explicit_kernel(AlcArgs A) {
    extern __shared__ __align__(16) double sm[];
    const int ld = A.ld, n = A.n, p = A.p, Np = A.Nprime, Npad = A.Npad;
    double *Kp = sm;
    double *tbuf = Kp + ld * ld;
    double *Xj = tbuf + 2 * ALC_TILE;
    double *h = Xj + ((n * p + 3) & ~3);  // keep 32-byte alignment of what follows
    double *w = h + ld;
    double *ks = w + ld;
    double *us = ks + ld;
    double *yv = us + ld;
    double *red = yv + ld;  // 160 doubles of reduction scratch
    __shared__ double xq[LAGP_PMAX];
    __shared__ uint32_t fl_s;

    const int tid = threadIdx.x;
    double *cache = A.cache + (size_t)blockIdx.x * A.cache_stride;
    double *coords = A.coords + (size_t)blockIdx.x * (p + 2) * Npad;  // [p][Npad] coords | kap | chosen
    double *kap = coords + (size_t)p * Npad;
    unsigned char *chosen = reinterpret_cast<unsigned char *>(kap + Npad);
    const double eta = A.eta;
    const int G = n - A.n0;

    for (int64_t xi = blockIdx.x; xi < A.M; xi += gridDim.x) {
        const double rth = A.theta_vec ? 1.0 / A.theta_vec[xi] : A.rtheta;  // per-location theta (Fig 1 step 4)
        const int32_t *pool = A.pool + xi * (int64_t)Np;
        int32_t *idx = A.idx_out + xi * (int64_t)n;
        if (tid < p) xq[tid] = A.XX[xi * p + tid];
        if (tid == 0) fl_s = 0;
        for (int e = tid; e < ld * ld; e += blockDim.x) Kp[e] = 0.0;
        __syncthreads();
        // ---- gather the pool (SoA coords), kappa_c and the chosen mask into the CTA's slab
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

        // ---- a2: K_{n0}^{-1} by successive partitioned-inverse appends of the
        // NN-ordered initial design (the a4 algebra), h, w and the cache rows
        for (int t = 0; t < A.n0; t++) {
            if (tid < t) ks[tid] = corr_from_d2(sqdist_fma(Xj + tid * p, Xj + t * p, p), rth);
            if (tid == 0) h[t] = corr_from_d2(sqdist_fma(Xj + t * p, xq, p), rth);
            __syncthreads();
            if (t == 0) {
                if (tid == 0) Kp[kp(0, 0, ld)] = 1.0 / (1.0 + eta);
            } else {
                double s = kp_append(Kp, ld, t, ks, 1.0 + eta, us, red);
                if (!(s > 0.0) && tid == 0) fl_s |= LAGP_FLAG_NONFINITE;
            }
            cache_row(cache + (size_t)t * Npad, Xj + t * p, coords, Npad, Np, p, rth);
            __syncthreads();
        }
        for (int e = tid; e < ld; e += blockDim.x) w[e] = 0.0;
        __syncthreads();
        kp_matvec(Kp, ld, A.n0, A.n0, h, w, true);

        // ---- greedy ALC loop (Fig 1 step 2(b)), j = current design size
        int j = A.n0;
        for (; j < n; j++) {
            const int nab = (j + 3) >> 2;  // 4-row blocks of K^{-1}
            const int AB = nab <= 1 ? 1 : nab <= 2 ? 2 : nab <= 4 ? 4 : nab <= 8 ? 8 : nab <= 16 ? 16 : 32;
            const int CB = ALC_THREADS / AB;  // 4-candidate blocks per tile
            const int T = 4 * CB;             // candidates per tile
            const int jpad = 4 * nab;
            const int ab = tid % AB, cb = tid / AB;
            const int ntiles = (Np + T - 1) / T;
            const int chunks = T >> 1;  // 16-byte chunks per tile row
            // zero the padding rows [j, jpad) of both tile buffers (never loaded)
            for (int e = tid; e < (jpad - j) * T; e += blockDim.x) {
                tbuf[j * T + e] = 0.0;
                tbuf[ALC_TILE + j * T + e] = 0.0;
            }
            auto load_tile = [&](int t, double *dst) {
                const int t0 = t * T;
                const int lg = 31 - __clz(chunks);  // chunks = T/2 is a power of two
                for (int e = tid; e < j * chunks; e += blockDim.x) {
                    const int a = e >> lg, c2 = e & (chunks - 1);
                    cp_async16(dst + a * T + 2 * c2, cache + (size_t)a * Npad + t0 + 2 * c2);
                }
                cp_async_commit();
            };
            load_tile(0, tbuf);
            Top2 best;
            best.init();
            bool sentinel = false, nonfinite = false;
            for (int t = 0; t < ntiles; t++) {
                double *tile = tbuf + (t & 1) * ALC_TILE;
                if (t + 1 < ntiles) {
                    load_tile(t + 1, tbuf + ((t + 1) & 1) * ALC_TILE);
                    cp_async_wait<1>();
                } else {
                    cp_async_wait<0>();
                }
                __syncthreads();
                const int t0 = t * T;
                double ps[4] = {0.0, 0.0, 0.0, 0.0}, pcv[4] = {0.0, 0.0, 0.0, 0.0};
                if (ab < nab) {
                    const int ag = ab;
                    double acc[4][4];
#pragma unroll
                    for (int r = 0; r < 4; r++)
#pragma unroll
                        for (int c = 0; c < 4; c++) acc[r][c] = 0.0;
                    const double2 *P0 = reinterpret_cast<const double2 *>(Kp) + ag;
                    const double2 *P1 = reinterpret_cast<const double2 *>(Kp + ld * ld / 2) + ag;
                    const double *tcol = tile + 4 * cb;
                    const int nq = ld >> 2;
                    // own[r][c] = tile[4ag+r][4cb+c], captured in the loop when the
                    // row block is this thread's (re-reading it afterwards is a
                    // 16-way bank conflict: 16 lanes, rows 4 apart, same column).
                    double own[4][4];
                    // rows b in [j, jpad) contribute 0: K^{-1} is zero there and the
                    // tile's padding rows are zeroed, so the loop runs whole 4-blocks.
                    for (int bb = 0; bb < nab; bb++) {
#pragma unroll
                        for (int r4 = 0; r4 < 4; r4++) {
                            const int b = 4 * bb + r4;
                            const double2 k01 = P0[b * nq];
                            const double2 k23 = P1[b * nq];
                            const double2 t01 = *reinterpret_cast<const double2 *>(tcol + b * T);
                            const double2 t23 = *reinterpret_cast<const double2 *>(tcol + b * T + 2);
                            const double kr[4] = {k01.x, k01.y, k23.x, k23.y};
                            const double tc[4] = {t01.x, t01.y, t23.x, t23.y};
#pragma unroll
                            for (int r = 0; r < 4; r++)
#pragma unroll
                                for (int c = 0; c < 4; c++) acc[r][c] = fma(kr[r], tc[c], acc[r][c]);
                            if (bb == ag) {
#pragma unroll
                                for (int c = 0; c < 4; c++) own[r4][c] = tc[c];
                            }
                        }
                    }
                    const double2 w01 = reinterpret_cast<const double2 *>(w)[ag];
                    const double2 w23 = reinterpret_cast<const double2 *>(w + (ld >> 1))[ag];
                    const double wr[4] = {w01.x, w01.y, w23.x, w23.y};
#pragma unroll
                    for (int r = 0; r < 4; r++) {
#pragma unroll
                        for (int c = 0; c < 4; c++) {
                            ps[c] = fma(own[r][c], acc[r][c], ps[c]);
                            pcv[c] = fma(wr[r], own[r][c], pcv[c]);
                        }
                    }
                }
                // reduce over the AB lanes sharing this c-block (aligned lane groups)
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
                                if (!isfinite(dl)) nonfinite = true;
                                else if (dl >= best.d1) best.push(dl, pool[pc], pc);
                                else if (dl > best.d2) best.d2 = dl;
                            }
                        }
                    }
                }
                __syncthreads();  // tile buffer (t & 1) is reloaded at iteration t + 1
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
                h[j] = kap[best.pos];
            }
            // ---- a4: append x* = pool[best.pos]; k_* is its cached column
            for (int a = tid; a < j; a += blockDim.x) ks[a] = cache[(size_t)a * Npad + best.pos];
            for (int k = tid; k < p; k += blockDim.x) Xj[j * p + k] = coords[k * Npad + best.pos];
            __syncthreads();
            double s = kp_append(Kp, ld, j, ks, 1.0 + eta, us, red);
            if (!(s > 0.0) && tid == 0) fl_s |= LAGP_FLAG_NONFINITE;
            kp_matvec(Kp, ld, j + 1, j + 1, h, w, true);
            if (j + 1 < n) cache_row(cache + (size_t)j * Npad, Xj + j * p, coords, Npad, Np, p, rth);
            __syncthreads();
        }

        // ---- a5: predict on D_j (j = n unless exhausted), fresh Cholesky in the Kp buffer
        for (int t = tid; t < j; t += blockDim.x) yv[t] = A.Z[idx[t]];
        __syncthreads();
        double mu, sc, vr;
        bool ok = block_predict(Kp, ld, j, p, Xj, yv, h, rth, eta, us, ks, red, &mu, &sc, &vr);
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

size_t alc_explicit_smem(int ld, int n, int p, int Npad) { return alc_smem_bytes(ld, n, p, Npad); }

cudaError_t launch_alc_explicit(const AlcArgs &a, int grid, cudaStream_t st) {
    size_t smem = alc_smem_bytes(a.ld, a.n, a.p, a.Npad);
    cudaError_t e = cudaFuncSetAttribute(alc_explicit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    alc_explicit_kernel<<<grid, ALC_THREADS, smem, st>>>(a);
    return cudaGetLastError();
}

int alc_explicit_blocks_per_sm(int ld, int n, int p, int Npad) {
    int nb = 0;
    size_t smem = alc_smem_bytes(ld, n, p, Npad);
    if (cudaFuncSetAttribute(alc_explicit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();  // do not leave a sticky error for the next launch check
        return 0;
    }
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, alc_explicit_kernel, ALC_THREADS, smem) != cudaSuccess) {
        cudaGetLastError();
        nb = 0;
    }
    return nb;
}

}  // namespace lagp
