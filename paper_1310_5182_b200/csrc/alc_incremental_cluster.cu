// alc_incremental_cluster.cu — LAGP_ALC_INCREMENTAL on a 2-CTA thread-block
// cluster per location (the same algebra as alc_incremental.cu).
//
// Why a cluster: the per-candidate state w_c = L_j^{-1} k_j(x_c) is read in full
// every step (e_c = K(x_c, x*) - w_*^T w_c). For N' = 1000, n = 50 that is 392 KB
// per location — more than one SM's shared memory, and a 1024-thread CTA caps a
// thread at 64 registers. Splitting the pool over the two SMs of a cluster (512
// candidates per SM, one per thread, 128 registers per thread) keeps the first
// R = 28-32 entries of every w_c in registers and the rest in shared memory: the
// dot product runs from the register file instead of the shared-memory port.
//
// Per step j (one cluster barrier):
//   1. each CTA: block argmax of Delta_c = cov_c^2/s_c (ties -> lowest global row);
//   2. each CTA's local winner writes its full record (Delta, index, rho, z_new,
//      y*, x*, w_{c*}) into its own shared slot (double-buffered by step parity);
//   3. barrier.cluster; warp 0 of each CTA reads both slot headers (DSMEM), picks
//      the same global winner on both SMs and copies its record locally;
//   4. every candidate: e_c, w_c[j] = e_c/rho, s_c -= w_c[j]^2, cov_c -= z_new w_c[j].
// Prediction (a5) from the maintained factor exactly as in alc_incremental.cu.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "launch.h"

namespace cg = cooperative_groups;

namespace lagp {

constexpr int CL_THREADS = 512;
constexpr int CL_NMAX = 64;  // n supported by this kernel (entries >= CL_R live in smem)

struct ClRec {
    double d1, d2, rho, znew, ystar;
    int i1, pos;
    double xstar[LAGP_PMAX];
    double w[CL_NMAX];
};

template <int P, int CL_R>  // CL_R: w_c entries in registers (multiple of 4)
__global__ void __launch_bounds__(CL_THREADS, 1)
alc_inc_cluster_kernel(AlcArgs A, int S) {
    extern __shared__ __align__(16) double sm[];
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned rank = cluster.block_rank();  // 0 or 1
    const int n = A.n, Np = A.Nprime, n0 = A.n0;
    constexpr int SPAD = CL_THREADS;  // smem entry stride (one column per thread)
    double *wsm = sm;                          // S × 512: entries [CL_R, CL_R + S)
    double *ytil = wsm + (size_t)S * SPAD;     // n (replicated on both CTAs)
    double *zv = ytil + CL_NMAX;               // n
    double *zc = zv + CL_NMAX;                 // 512: Z of this CTA's candidates
    double *red = zc + CL_THREADS;             // 160
    __shared__ ClRec slot[2];
    __shared__ ClRec cur;
    __shared__ double xq[LAGP_PMAX];
    __shared__ uint32_t fl;

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int c = (int)rank * CL_THREADS + tid;  // pool position owned by this thread
    const double eta = A.eta;
    const int G = n - n0;
    const int nclusters = gridDim.x / 2;
    const int cid = blockIdx.x / 2;

    for (int64_t xi = cid; xi < A.M; xi += nclusters) {
        const double rth = A.theta_vec ? 1.0 / A.theta_vec[xi] : A.rtheta;  // per-location theta (Fig 1 step 4)
        const int32_t *pool = A.pool + xi * (int64_t)Np;
        int32_t *idx = A.idx_out + xi * (int64_t)n;
        if (tid < P) xq[tid] = A.XX[xi * P + tid];
        if (tid == 0) fl = 0;
        if (rank == 0) {
            if (A.gap_out)
                for (int t = tid; t < G; t += blockDim.x)
                    A.gap_out[xi * G + t] = __longlong_as_double(0x7ff8000000000000LL);
            for (int t = tid; t < n; t += blockDim.x) idx[t] = (t < n0) ? pool[t] : -1;
        }
        __syncthreads();

        const bool valid = c < Np;
        bool chosen = false;
        const int gidx = valid ? pool[c] : 0x7fffffff;
        double xc[P];
        double d2 = 0.0;
#pragma unroll
        for (int k = 0; k < P; k++) {
            xc[k] = valid ? A.X[(int64_t)gidx * P + k] : 0.0;
            const double diff = __dsub_rn(xc[k], xq[k]);
            d2 = __fma_rn(diff, diff, d2);
        }
        double s = 1.0 + eta;
        double cov = valid ? corr_from_d2(d2, rth) : 0.0;  // kappa_c
        zc[tid] = valid ? A.Z[gidx] : 0.0;
        double wr[CL_R];
#pragma unroll
        for (int a = 0; a < CL_R; a++) wr[a] = 0.0;
        __syncthreads();

        int j = 0;
        for (; j < n; j++) {
            // ---- 1. local winner (forced NN order for j < n0)
            ArgTop loc;
            if (j < n0) {
                loc.d1 = 1.0;
                loc.d2 = 0.0;
                loc.i1 = (rank == 0) ? pool[j] : -1;
                loc.pos = (rank == 0) ? j : -1;
            } else {
                double bd1 = -1.0;
                int bi = -1;
                bool sentinel = false, nonfinite = false;
                if (valid && !chosen) {
                    if (!(s > kSMin)) {
                        sentinel = true;
                    } else {
                        const double dl = cov * cov / s;
                        if (!isfinite(dl)) nonfinite = true;
                        else { bd1 = dl; bi = gidx; }
                    }
                }
                if (__any_sync(0xffffffffu, sentinel) && lane == 0) atomicOr(&fl, (uint32_t)LAGP_FLAG_SENTINEL);
                if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(&fl, (uint32_t)LAGP_FLAG_NONFINITE);
                loc = block_argtop(bd1, bi, 0.0, c, red);
            }
            // ---- 2. the local winner publishes its record into slot[j & 1]
            ClRec &my = slot[j & 1];
            const bool mine = valid && !chosen && loc.i1 >= 0 && gidx == loc.i1;
            if (tid == 0 && loc.i1 < 0) {  // this CTA has no candidate left
                my.i1 = -1;
                my.d1 = -1.0;
                my.d2 = 0.0;
            }
            if (mine) {
                my.d1 = loc.d1;
                my.d2 = loc.d2;
                my.i1 = loc.i1;
                my.pos = c;
                const double rho = sqrt(s);
                my.rho = rho;
                my.znew = cov / rho;
                my.ystar = zc[tid];
#pragma unroll
                for (int k = 0; k < P; k++) my.xstar[k] = xc[k];
#pragma unroll
                for (int a = 0; a < CL_R; a++)
                    if (a < j) my.w[a] = wr[a];
                for (int a = CL_R; a < j; a++) my.w[a] = wsm[(size_t)(a - CL_R) * SPAD + tid];
            }
            cluster.sync();
            // ---- 3. both CTAs pick the same global winner, warp 0 copies its record
            if (wid == 0) {
                const ClRec *r0 = cluster.map_shared_rank(&slot[j & 1], 0);
                const ClRec *r1 = cluster.map_shared_rank(&slot[j & 1], 1);
                const double a1 = r0->d1, b1 = r1->d1;
                const int ai = r0->i1, bi = r1->i1;
                // (Delta, index) order; a missing record has i1 = -1
                bool take1;
                if (ai < 0) take1 = true;
                else if (bi < 0) take1 = false;
                else take1 = (b1 > a1) || (b1 == a1 && bi < ai);
                const ClRec *w = take1 ? r1 : r0;
                const ClRec *l = take1 ? r0 : r1;
                const int wi = w->i1;
                if (lane == 0) {
                    cur.i1 = wi;
                    if (wi >= 0) {
                        cur.d1 = w->d1;
                        // second best: the winner CTA's own second, or the other CTA's best
                        const double ld1 = l->i1 >= 0 ? l->d1 : 0.0;
                        cur.d2 = fmax(w->d2, ld1);
                        cur.pos = w->pos;
                        cur.rho = w->rho;
                        cur.znew = w->znew;
                        cur.ystar = w->ystar;
                    }
                }
                if (wi >= 0) {
                    for (int a = lane; a < j; a += 32) cur.w[a] = w->w[a];
                    if (lane < P) cur.xstar[lane] = w->xstar[lane];
                }
            }
            __syncthreads();
            if (cur.i1 < 0) {  // both CTAs exhausted
                if (tid == 0) fl |= LAGP_FLAG_EXHAUSTED;
                break;
            }
            if (j >= n0 && rank == 0 && tid == 0) {
                const double gap = top2_gap(cur.d1, cur.d2);
                if (!(cur.d1 > 0.0) || gap < kTieGap) fl |= LAGP_FLAG_NEAR_TIE;
                if (A.gap_out) A.gap_out[xi * G + (j - n0)] = gap;
                idx[j] = cur.i1;
            }
            if (c == cur.pos) chosen = true;
            const double rrho = 1.0 / cur.rho, znew = cur.znew;
            if (wid == 0) {  // a5 state: y~_j = (y* - w*^T y~)/rho, z_j = z_new
                double acc = 0.0;
                for (int a = lane; a < j; a += 32) acc = fma(cur.w[a], ytil[a], acc);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
                if (lane == 0) {
                    ytil[j] = (cur.ystar - acc) * rrho;
                    zv[j] = znew;
                }
            }
            // ---- 4. downdate every candidate
            if (valid) {
                double dd = 0.0;
#pragma unroll
                for (int k = 0; k < P; k++) {
                    const double diff = __dsub_rn(xc[k], cur.xstar[k]);
                    dd = __fma_rn(diff, diff, dd);
                }
                double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
#pragma unroll
                for (int a = 0; a < CL_R; a += 4) {  // cur.w[a >= j] are stale but wr[a >= j] = 0
                    const double2 w01 = *reinterpret_cast<const double2 *>(&cur.w[a]);
                    const double2 w23 = *reinterpret_cast<const double2 *>(&cur.w[a + 2]);
                    acc0 = fma(a < j ? w01.x : 0.0, wr[a], acc0);
                    acc1 = fma(a + 1 < j ? w01.y : 0.0, wr[a + 1], acc1);
                    acc2 = fma(a + 2 < j ? w23.x : 0.0, wr[a + 2], acc2);
                    acc3 = fma(a + 3 < j ? w23.y : 0.0, wr[a + 3], acc3);
                }
                for (int a = CL_R; a < j; a++) acc0 = fma(cur.w[a], wsm[(size_t)(a - CL_R) * SPAD + tid], acc0);
                const double e = corr_from_d2(dd, rth) - ((acc0 + acc1) + (acc2 + acc3));
                const double wn = e * rrho;
                if (j < CL_R) {
#pragma unroll
                    for (int b = 0; b < CL_R; b++)
                        if (b == j) wr[b] = wn;
                } else {
                    wsm[(size_t)(j - CL_R) * SPAD + tid] = wn;
                }
                s = fma(-wn, wn, s);
                cov = fma(-znew, wn, cov);
            }
            __syncthreads();
        }

        // ---- flags from both CTAs, then a5 on rank 0
        cluster.sync();
        if (rank == 0 && wid == 0) {
            const uint32_t f1 = *cluster.map_shared_rank(&fl, 1);
            double mu = 0.0, psi = 0.0, zz = 0.0;
            for (int a = lane; a < j; a += 32) {
                mu = fma(zv[a], ytil[a], mu);
                psi = fma(ytil[a], ytil[a], psi);
                zz = fma(zv[a], zv[a], zz);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                mu += __shfl_xor_sync(0xffffffffu, mu, off);
                psi += __shfl_xor_sync(0xffffffffu, psi, off);
                zz += __shfl_xor_sync(0xffffffffu, zz, off);
            }
            if (lane == 0) {
                const double sc = psi * (1.0 + eta - zz) / (double)j;
                const double vr = j > 2 ? sc * (double)j / (double)(j - 2) : __longlong_as_double(0x7ff8000000000000LL);
                uint32_t f = fl | (f1 & (LAGP_FLAG_SENTINEL | LAGP_FLAG_NONFINITE));
                if (!isfinite(mu) || !isfinite(sc)) f |= LAGP_FLAG_NONFINITE;
                A.mean[xi] = mu;
                A.s2[xi] = sc;
                if (A.var) A.var[xi] = vr;
                if (A.flags) A.flags[xi] = f;
                if (f & (LAGP_FLAG_EXHAUSTED | LAGP_FLAG_NONFINITE)) atomicAdd(A.n_partial, 1);
            }
        }
        cluster.sync();  // partner's flags read before the next location resets them
    }
}

// ---------------------------------------------------------------- host side
bool inc_cluster_supported(int n, int p, int Nprime) {
    return Nprime <= 2 * CL_THREADS && n <= CL_NMAX && (p == 2 || p == 3 || p == 8);
}

static size_t cl_smem(int n, int R) {
    const int S = n > R ? n - R : 0;
    return ((size_t)S * CL_THREADS + 2 * CL_NMAX + CL_THREADS + 160) * sizeof(double);
}

template <int P, int R>
static cudaError_t cl_launch_t(const AlcArgs &a, int clusters, cudaStream_t st) {
    const int S = a.n > R ? a.n - R : 0;
    const size_t smem = cl_smem(a.n, R);
    cudaError_t e = cudaFuncSetAttribute(alc_inc_cluster_kernel<P, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(CL_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, alc_inc_cluster_kernel<P, R>, a, S);
}

cudaError_t launch_alc_inc_cluster(const AlcArgs &a, int num_sms, cudaStream_t st) {
    int clusters = num_sms / 2;
    if ((int64_t)clusters > a.M) clusters = (int)a.M;
    if (clusters < 1) clusters = 1;
    switch (a.p) {
        // largest register share without spills at 128 registers per thread
        case 2: return cl_launch_t<2, 32>(a, clusters, st);
        case 3: return cl_launch_t<3, 32>(a, clusters, st);
        case 8: return cl_launch_t<8, 28>(a, clusters, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lagp
