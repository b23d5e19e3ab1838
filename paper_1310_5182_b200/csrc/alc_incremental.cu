// alc_incremental.cu — LAGP_ALC_INCREMENTAL: the same
// greedy ALC local design (Fig 1 step 2; Eq (5)-(6)) with
// per-candidate Schur-complement downdates, O(j) work per candidate per step
// instead of the O(j^2) quadratic form k_c^T K_j^{-1} k_c.
//
// With K_j = L_j L_j^T, every pool candidate c carries
//   w_c = L_j^{-1} k_j(x_c)   (j entries),
//   s_c = 1 + eta - ||w_c||^2 = m_j^{-1}(x_c)          (Eq 6)
//   cov_c = kappa_c - z^T w_c, z = L_j^{-1} h          (kappa_c = K(x_c, x))
// so Delta_c = cov_c^2 / s_c is exactly Eq (5) (App A.1). Appending the chosen
// x* (candidate c*, rho = sqrt(s_{c*})) is the partitioned-inverse step of a4
// applied to the factor: L_{j+1} = [[L_j, 0], [w_{c*}^T, rho]], and for every c
//   e_c = K(x_c, x*) - w_{c*}^T w_c          (= Cov_j(f(x_c), f(x*)))
//   w_c[j] = e_c / rho,  s_c -= (e_c/rho)^2,  cov_c -= (cov_{c*}/rho) (e_c/rho).
// The initial NN design X_{n0} enters by the same append, forced in NN order.
//
// a5 from the same factor (L_n is a Cholesky factor of K_n = C(X_n) + eta I,
// built column by column): with z = L^{-1} h and y~ = L^{-1} Y (one new entry
// per append, y~_j = (y* - w_{c*}^T y~)/rho),
//   mean = z^T y~,  psi = ||y~||^2,  s2 = psi (1 + eta - ||z||^2) / n   (Eq 1-2).
//
// B200 mapping: one CTA of 1024 threads per location (persistent grid, one CTA
// per SM), one pool candidate per thread when N' <= 1024. The candidate's state
// (x_c, s_c, cov_c and the first R entries of w_c) lives in registers, entries
// [R, R+S) in shared memory (entry-major, conflict-free), the rest in an HBM
// slab — so for the C1–C4 shapes almost all of the local state is on-chip and
// each step is one pass over the candidates: one exp, one j-term dot, one argmax.
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "launch.h"

namespace lagp {

constexpr int INC_THREADS = 1024;
// w_c entries kept in registers (1024 threads -> <= 64 registers per thread)
#ifndef INC_R8
#define INC_R8 8
#endif
#ifndef INC_R4
#define INC_R4 12
#endif

struct IncShared {
    double xstar[LAGP_PMAX];
    double xq[LAGP_PMAX];
    double rho, rrho, znew, ystar;
    uint32_t fl;
};

// smem (doubles): wsm S*Npad | wstar n4 | ytil n4 | zv n4 | zc Npad | red 160
__host__ __device__ inline int inc_n4(int n) { return (n + 3) & ~3; }

template <int R, int P, int CPT>
__global__ void __launch_bounds__(INC_THREADS, 1)
alc_incremental_kernel(AlcArgs A, int S) {
    extern __shared__ __align__(16) double sm[];
    const int n = A.n, Np = A.Nprime, Npad = A.Npad, n0 = A.n0;
    const int p = P ? P : A.p;
    double *wsm = sm;
    double *wstar = wsm + (size_t)S * Npad;
    double *ytil = wstar + inc_n4(n);
    double *zv = ytil + inc_n4(n);
    double *zc = zv + inc_n4(n);  // Z of the pool candidates (y* without an HBM round trip)
    double *red = zc + Npad;
    __shared__ IncShared sh;

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    double *gw = A.cache + (size_t)blockIdx.x * A.cache_stride;  // entries >= R+S: gw[(a-R-S)*Npad + c]
    double *coords = A.coords + (size_t)blockIdx.x * p * Npad;   // generic-p path only
    const double rth = A.rtheta, eta = A.eta;
    const int G = n - n0;
    const int RS = R + S;

    for (int64_t xi = blockIdx.x; xi < A.M; xi += gridDim.x) {
        const int32_t *pool = A.pool + xi * (int64_t)Np;
        int32_t *idx = A.idx_out + xi * (int64_t)n;
        if (tid < p) sh.xq[tid] = A.XX[xi * p + tid];
        if (tid == 0) sh.fl = 0;
        for (int t = tid; t < n; t += blockDim.x) wstar[t] = 0.0;
        if (A.gap_out)
            for (int t = tid; t < G; t += blockDim.x) A.gap_out[xi * G + t] = __longlong_as_double(0x7ff8000000000000LL);
        for (int t = tid; t < n; t += blockDim.x) idx[t] = (t < n0) ? pool[t] : -1;
        __syncthreads();

        // ---- per-candidate state
        double xc[CPT][P ? P : 1];
        double s[CPT], cov[CPT];
        double wr[CPT][R > 0 ? R : 1];
        bool chosen[CPT], valid[CPT];
        int gidx[CPT];
#pragma unroll
        for (int q = 0; q < CPT; q++) {
            const int c = tid + q * INC_THREADS;
            valid[q] = c < Np;
            chosen[q] = false;
            gidx[q] = valid[q] ? pool[c] : 0x7fffffff;
            double d2 = 0.0;
            if (P) {
#pragma unroll
                for (int k = 0; k < (P ? P : 1); k++) {
                    xc[q][k] = valid[q] ? A.X[(int64_t)gidx[q] * p + k] : 0.0;
                    double diff = __dsub_rn(xc[q][k], sh.xq[k]);
                    d2 = __fma_rn(diff, diff, d2);
                }
            } else if (valid[q]) {
                for (int k = 0; k < p; k++) {
                    const double v = A.X[(int64_t)gidx[q] * p + k];
                    coords[k * Npad + c] = v;
                    double diff = __dsub_rn(v, sh.xq[k]);
                    d2 = __fma_rn(diff, diff, d2);
                }
            }
            s[q] = 1.0 + eta;
            cov[q] = valid[q] ? corr_from_d2(d2, rth) : 0.0;  // kappa_c (z is empty at j = 0)
            if (valid[q]) zc[c] = A.Z[gidx[q]];
#pragma unroll
            for (int a = 0; a < (R > 0 ? R : 1); a++) wr[q][a] = 0.0;
        }
        __syncthreads();

        int j = 0;  // current design size
        for (; j < n; j++) {
            int cstar;
            if (j < n0) {
                cstar = j;  // forced NN append (a2), pool order = NN order
            } else {
                // ---- a3: argmax of Delta_c = cov_c^2 / s_c over valid, unchosen candidates
                double bd1 = -1.0, bd2 = 0.0;  // bd1 < 0: no candidate
                int bi = -1, bp = -1;
                bool sentinel = false, nonfinite = false;
#pragma unroll
                for (int q = 0; q < CPT; q++) {
                    if (valid[q] && !chosen[q]) {
                        if (!(s[q] > kSMin)) {
                            sentinel = true;
                        } else {
                            const double dl = cov[q] * cov[q] / s[q];
                            if (!isfinite(dl)) {
                                nonfinite = true;
                            } else if (dl > bd1 || (dl == bd1 && (unsigned)gidx[q] < (unsigned)bi)) {
                                bd2 = fmax(bd2, bd1);
                                bd1 = dl;
                                bi = gidx[q];
                                bp = tid + q * INC_THREADS;
                            } else {
                                bd2 = fmax(bd2, dl);
                            }
                        }
                    }
                }
                if (__any_sync(0xffffffffu, sentinel) && lane == 0) atomicOr(&sh.fl, (uint32_t)LAGP_FLAG_SENTINEL);
                if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(&sh.fl, (uint32_t)LAGP_FLAG_NONFINITE);
                const ArgTop best = block_argtop(bd1, bi, bd2, bp, red);
                if (best.i1 < 0) {
                    if (tid == 0) sh.fl |= LAGP_FLAG_EXHAUSTED;
                    break;
                }
                cstar = best.pos;
                if (tid == 0) {
                    const double gap = top2_gap(best.d1, best.d2);
                    if (!(best.d1 > 0.0) || gap < kTieGap) sh.fl |= LAGP_FLAG_NEAR_TIE;
                    if (A.gap_out) A.gap_out[xi * G + (j - n0)] = gap;
                    idx[j] = best.i1;
                }
            }
            // ---- a4 on the factor: publish w_{c*}, x*, rho, z_new, y*
            const int owner = cstar % INC_THREADS, oq = cstar / INC_THREADS;
            if (tid == owner) {
#pragma unroll
                for (int q = 0; q < CPT; q++) {
                    if (q == oq) {
#pragma unroll
                        for (int a = 0; a < R; a++)
                            if (a < j) wstar[a] = wr[q][a];
                        if (P) {
#pragma unroll
                            for (int k = 0; k < (P ? P : 1); k++) sh.xstar[k] = xc[q][k];
                        }
                        const double rho = sqrt(s[q]);
                        sh.rho = rho;
                        sh.rrho = 1.0 / rho;
                        sh.znew = cov[q] / rho;
                        sh.ystar = zc[cstar];
                        chosen[q] = true;
                        if (!(s[q] > 0.0)) atomicOr(&sh.fl, (uint32_t)LAGP_FLAG_NONFINITE);
                    }
                }
            }
            if (!P && tid < p) sh.xstar[tid] = coords[tid * Npad + cstar];
            for (int a = R + tid; a < j; a += blockDim.x)
                wstar[a] = (a < RS) ? wsm[(size_t)(a - R) * Npad + cstar] : gw[(size_t)(a - RS) * Npad + cstar];
            __syncthreads();
            const double rrho = sh.rrho, znew = sh.znew;
            if (wid == 0) {  // a5 state: y~_j = (y* - w*^T y~) / rho, z_j = z_new
                double acc = 0.0;
                for (int a = lane; a < j; a += 32) acc = fma(wstar[a], ytil[a], acc);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
                if (lane == 0) {
                    ytil[j] = (sh.ystar - acc) * rrho;
                    zv[j] = znew;
                }
            }
            // ---- every candidate: new entry of w_c, downdates of s_c and cov_c
#pragma unroll
            for (int q = 0; q < CPT; q++) {
                const int c = tid + q * INC_THREADS;
                if (!valid[q]) continue;
                // issue the HBM-slab loads first (independent, latency overlapped)
                double acc2 = 0.0, acc3 = 0.0;
                for (int a = RS; a < j; a += 4) {
                    const double g0 = gw[(size_t)(a - RS) * Npad + c];
                    const double g1 = a + 1 < j ? gw[(size_t)(a + 1 - RS) * Npad + c] : 0.0;
                    const double g2 = a + 2 < j ? gw[(size_t)(a + 2 - RS) * Npad + c] : 0.0;
                    const double g3 = a + 3 < j ? gw[(size_t)(a + 3 - RS) * Npad + c] : 0.0;
                    acc2 = fma(wstar[a], g0, acc2);
                    acc3 = fma(a + 1 < j ? wstar[a + 1] : 0.0, g1, acc3);
                    acc2 = fma(a + 2 < j ? wstar[a + 2] : 0.0, g2, acc2);
                    acc3 = fma(a + 3 < j ? wstar[a + 3] : 0.0, g3, acc3);
                }
                double d2 = 0.0;
                if (P) {
#pragma unroll
                    for (int k = 0; k < (P ? P : 1); k++) {
                        double diff = __dsub_rn(xc[q][k], sh.xstar[k]);
                        d2 = __fma_rn(diff, diff, d2);
                    }
                } else {
                    for (int k = 0; k < p; k++) {
                        double diff = __dsub_rn(coords[k * Npad + c], sh.xstar[k]);
                        d2 = __fma_rn(diff, diff, d2);
                    }
                }
                double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
                for (int a = 0; a < R; a += 2) {  // R even; wstar[a >= j] = 0, wr[a >= j] = 0
                    const double2 ws = reinterpret_cast<const double2 *>(wstar)[a >> 1];
                    acc0 = fma(ws.x, wr[q][a], acc0);
                    acc1 = fma(ws.y, wr[q][a + 1], acc1);
                }
                const int jr = j < RS ? j : RS;
                const double *wp = wsm + c;  // column of this candidate, entry a at wp[(a - R) * Npad]
                int a = R;
                for (; a + 3 < jr; a += 4) {  // R even -> a even: wstar pairs are 16-byte aligned
                    const double2 s01 = *reinterpret_cast<const double2 *>(wstar + a);
                    const double2 s23 = *reinterpret_cast<const double2 *>(wstar + a + 2);
                    const double *q0 = wp + (size_t)(a - R) * Npad;
                    acc0 = fma(s01.x, q0[0], acc0);
                    acc1 = fma(s01.y, q0[Npad], acc1);
                    acc0 = fma(s23.x, q0[2 * Npad], acc0);
                    acc1 = fma(s23.y, q0[3 * Npad], acc1);
                }
                for (; a < jr; a++) acc0 = fma(wstar[a], wp[(size_t)(a - R) * Npad], acc0);
                const double e = corr_from_d2(d2, rth) - ((acc0 + acc1) + (acc2 + acc3));
                const double wn = e * rrho;
                if (j < R) {
#pragma unroll
                    for (int b = 0; b < R; b++)
                        if (b == j) wr[q][b] = wn;
                } else if (j < RS) {
                    wsm[(size_t)(j - R) * Npad + c] = wn;
                } else {
                    gw[(size_t)(j - RS) * Npad + c] = wn;
                }
                s[q] = fma(-wn, wn, s[q]);
                cov[q] = fma(-znew, wn, cov[q]);
            }
            __syncthreads();  // wstar / sh / ytil reused next step
        }

        // ---- a5: mean = z^T y~, psi = ||y~||^2, s2 = psi (1 + eta - ||z||^2) / j
        __syncthreads();
        if (wid == 0) {
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
                uint32_t f = sh.fl;
                if (!isfinite(mu) || !isfinite(sc)) f |= LAGP_FLAG_NONFINITE;
                A.mean[xi] = mu;
                A.s2[xi] = sc;
                if (A.var) A.var[xi] = vr;
                if (A.flags) A.flags[xi] = f;
                if (f & (LAGP_FLAG_EXHAUSTED | LAGP_FLAG_NONFINITE)) atomicAdd(A.n_partial, 1);
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- host side
template <int R, int P, int CPT>
static cudaError_t inc_launch_t(const AlcArgs &a, int S, int grid, size_t smem, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(alc_incremental_kernel<R, P, CPT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    alc_incremental_kernel<R, P, CPT><<<grid, INC_THREADS, smem, st>>>(a, S);
    return cudaGetLastError();
}

// register entries per candidate by input dimension (1024 threads -> <= 64 regs/thread)
static int inc_R(int p, int cpt) {
    if (cpt > 1) return 0;
    if (p == 8) return INC_R8;
    if (p <= 4) return INC_R4;
    return 0;
}

IncPlan inc_plan(int n, int p, int Nprime, int Npad, size_t smem_optin) {
    IncPlan pl{};
    pl.cpt = (Nprime + INC_THREADS - 1) / INC_THREADS;
    if (pl.cpt > 8) {
        pl.ok = false;
        return pl;
    }
    pl.R = inc_R(p, pl.cpt);
    const size_t fixed = ((size_t)inc_n4(n) * 3 + Npad + 160) * sizeof(double);
    size_t avail = smem_optin > fixed + 1024 ? smem_optin - fixed - 1024 : 0;
    int S = (int)(avail / ((size_t)Npad * sizeof(double)));
    const int need = n - pl.R > 0 ? n - pl.R : 0;
    if (S > need) S = need;
    if (S < 0) S = 0;
    pl.S = S;
    pl.wsz = S * Npad;
    pl.smem = (size_t)S * Npad * sizeof(double) + fixed;
    pl.ok = pl.smem <= smem_optin;
    pl.global_entries = n - pl.R - S > 0 ? n - pl.R - S : 0;
    return pl;
}

cudaError_t launch_alc_incremental(const AlcArgs &a, const IncPlan &pl, int grid, cudaStream_t st) {
    const int p = a.p;
#define INC_DISPATCH_P(R_, CPT_)                                                     \
    switch (p) {                                                                     \
        case 1: return inc_launch_t<R_, 1, CPT_>(a, pl.S, grid, pl.smem, st);        \
        case 2: return inc_launch_t<R_, 2, CPT_>(a, pl.S, grid, pl.smem, st);        \
        case 3: return inc_launch_t<R_, 3, CPT_>(a, pl.S, grid, pl.smem, st);        \
        case 4: return inc_launch_t<R_, 4, CPT_>(a, pl.S, grid, pl.smem, st);        \
        case 8: return inc_launch_t<R_, 8, CPT_>(a, pl.S, grid, pl.smem, st);        \
        default: return inc_launch_t<0, 0, CPT_>(a, pl.S, grid, pl.smem, st);        \
    }
    if (pl.cpt == 1) {
        if (p == 8 && pl.R == INC_R8) { INC_DISPATCH_P(INC_R8, 1) }
        if (p <= 4 && pl.R == INC_R4) { INC_DISPATCH_P(INC_R4, 1) }
        INC_DISPATCH_P(0, 1)
    }
    if (pl.cpt == 2) { INC_DISPATCH_P(0, 2) }
    if (pl.cpt <= 4) { INC_DISPATCH_P(0, 4) }
    INC_DISPATCH_P(0, 8)
#undef INC_DISPATCH_P
}

}  // namespace lagp
