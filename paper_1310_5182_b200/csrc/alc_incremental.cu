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
    double rrho, znew, ystar;
};

// smem (doubles): wsm S*Npad | wst 2*n4 | ytil n4 | zv n4 | zc Npad | red 200
__host__ __device__ inline int inc_n4(int n) { return (n + 3) & ~3; }
__host__ __device__ inline int inc_wl(int n, int R) { return inc_n4(n > R ? n : R); }

template <int R, int P, int CPT>
__global__ void __launch_bounds__(INC_THREADS, 1)
alc_incremental_kernel(AlcArgs A, int S) {
    extern __shared__ __align__(16) double sm[];
    const int n = A.n, Np = A.Nprime, Npad = A.Npad, n0 = A.n0;
    const int p = P ? P : A.p;
    const int n4 = inc_n4(n);
    double *wsm = sm;                        // S x Npad: entries [R, R+S) of every w_c
    const int wl = inc_wl(n, R);             // publish slot length: covers n and R entries
    double *wst = wsm + (size_t)S * Npad;    // 2 x wl: the winner's register entries (by step parity)
    double *ytil = wst + 2 * wl;
    double *zv = ytil + n4;
    double *zc = zv + n4;                    // Z of the pool candidates (y* without an HBM round trip)
    double *red = zc + Npad;                 // 200 doubles: double-buffered argmax scratch
    __shared__ IncShared sh[2];              // publish slots by step parity
    __shared__ uint32_t fl;

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    double *gw = A.cache + (size_t)blockIdx.x * A.cache_stride;  // entries >= R+S: gw[(a-R-S)*Npad + c]
    double *coords = A.coords + (size_t)blockIdx.x * p * Npad;   // generic-p path only
    const double eta = A.eta;
    const int G = n - n0;
    const int RS = R + S;

    for (int64_t xi = blockIdx.x; xi < A.M; xi += gridDim.x) {
        const double rth = A.theta_vec ? 1.0 / A.theta_vec[xi] : A.rtheta;  // per-location theta (Fig 1 step 4)
        const int32_t *pool = A.pool + xi * (int64_t)Np;
        int32_t *idx = A.idx_out + xi * (int64_t)n;
        if (tid < p) sh[0].xq[tid] = A.XX[xi * p + tid];
        if (tid == 0) fl = 0;
        for (int t = tid; t < 2 * wl; t += blockDim.x) wst[t] = 0.0;
        if (A.gap_out)
            for (int t = tid; t < G; t += blockDim.x) A.gap_out[xi * G + t] = __longlong_as_double(0x7ff8000000000000LL);
        for (int t = tid; t < n; t += blockDim.x) idx[t] = (t < n0) ? pool[t] : -1;
        // shared entries not yet appended read as 0, so the dot below runs in
        // whole groups of 4 (S is a multiple of 4)
        for (int t = tid; t < S * Npad; t += blockDim.x) wsm[t] = 0.0;
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
                    double diff = __dsub_rn(xc[q][k], sh[0].xq[k]);
                    d2 = __fma_rn(diff, diff, d2);
                }
            } else if (valid[q]) {
                for (int k = 0; k < p; k++) {
                    const double v = A.X[(int64_t)gidx[q] * p + k];
                    coords[k * Npad + c] = v;
                    double diff = __dsub_rn(v, sh[0].xq[k]);
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

        // Two barriers per step: one in the argmax, one after the publish. The
        // publish slots and the argmax scratch alternate by step parity, so a slot
        // is rewritten only after every thread has passed the next step's barriers.
        int j = 0;  // current design size
        for (; j < n; j++) {
            const int par = j & 1;
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
                if (__any_sync(0xffffffffu, sentinel) && lane == 0) atomicOr(&fl, (uint32_t)LAGP_FLAG_SENTINEL);
                if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(&fl, (uint32_t)LAGP_FLAG_NONFINITE);
                const ArgTop best = block_argtop_1b(bd1, bi, bd2, bp, red, par);
                if (best.i1 < 0) {
                    if (tid == 0) fl |= LAGP_FLAG_EXHAUSTED;
                    break;
                }
                cstar = best.pos;
                if (tid == 0) {
                    const double gap = top2_gap(best.d1, best.d2);
                    if (!(best.d1 > 0.0) || gap < kTieGap) fl |= LAGP_FLAG_NEAR_TIE;
                    if (A.gap_out) A.gap_out[xi * G + (j - n0)] = gap;
                    idx[j] = best.i1;
                }
            }
            // ---- a4 on the factor: the owner publishes its register entries, x*, 1/rho,
            // z_new, y*; the winner's shared/HBM entries are read in place by everyone
            IncShared &pb = sh[par];
            double *ws = wst + par * wl;
            const int owner = cstar % INC_THREADS, oq = cstar / INC_THREADS;
            if (tid == owner) {
#pragma unroll
                for (int q = 0; q < CPT; q++) {
                    if (q == oq) {
#pragma unroll
                        for (int a = 0; a < R; a++) ws[a] = (a < j) ? wr[q][a] : 0.0;
                        if (P) {
#pragma unroll
                            for (int k = 0; k < (P ? P : 1); k++) pb.xstar[k] = xc[q][k];
                        }
                        const double rho = sqrt(s[q]);
                        pb.rrho = 1.0 / rho;
                        pb.znew = cov[q] / rho;
                        pb.ystar = zc[cstar];
                        chosen[q] = true;
                        if (!(s[q] > 0.0)) atomicOr(&fl, (uint32_t)LAGP_FLAG_NONFINITE);
                    }
                }
            }
            if (!P && tid < p) pb.xstar[tid] = coords[tid * Npad + cstar];
            __syncthreads();
            const double rrho = pb.rrho, znew = pb.znew;
            const double *wcs = wsm + cstar;  // winner's column, entry a at wcs[(a - R) * Npad]
            const double *wcg = gw + cstar;   // ... and in the slab, entry a at wcg[(a - RS) * Npad]
            if (wid == 0) {  // a5 state: y~_j = (y* - w*^T y~) / rho, z_j = z_new
                double acc = 0.0;
                for (int a = lane; a < j; a += 32) {
                    const double wa = a < R ? ws[a] : (a < RS ? wcs[(a - R) * Npad] : wcg[(a - RS) * Npad]);
                    acc = fma(wa, ytil[a], acc);
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
                if (lane == 0) {
                    ytil[j] = (pb.ystar - acc) * rrho;
                    zv[j] = znew;
                }
            }
            // ---- every candidate: new entry of w_c, downdates of s_c and cov_c
#pragma unroll
            for (int q = 0; q < CPT; q++) {
                const int c = tid + q * INC_THREADS;
                if (!valid[q]) continue;
                // HBM-slab entries first (independent loads, latency overlapped)
                double acc2 = 0.0, acc3 = 0.0;
                for (int a = RS; a < j; a += 2) {
                    const bool two = a + 1 < j;
                    const double g0 = gw[(a - RS) * Npad + c];
                    const double g1 = two ? gw[(a + 1 - RS) * Npad + c] : 0.0;
                    const double h0 = wcg[(a - RS) * Npad];
                    const double h1 = two ? wcg[(a + 1 - RS) * Npad] : 0.0;
                    acc2 = fma(h0, g0, acc2);
                    acc3 = fma(h1, g1, acc3);
                }
                double d2 = 0.0;
                if (P) {
#pragma unroll
                    for (int k = 0; k < (P ? P : 1); k++) {
                        double diff = __dsub_rn(xc[q][k], pb.xstar[k]);
                        d2 = __fma_rn(diff, diff, d2);
                    }
                } else {
                    for (int k = 0; k < p; k++) {
                        double diff = __dsub_rn(coords[k * Npad + c], pb.xstar[k]);
                        d2 = __fma_rn(diff, diff, d2);
                    }
                }
                double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
                for (int a = 0; a < R; a += 2) {  // R even; ws[a >= j] = 0 and wr[a >= j] = 0
                    const double2 w2 = reinterpret_cast<const double2 *>(ws)[a >> 1];
                    acc0 = fma(w2.x, wr[q][a], acc0);
                    acc1 = fma(w2.y, wr[q][a + 1], acc1);
                }
                // shared entries [R, min(j, R+S)) rounded up to 4: rows >= j are still 0 in
                // every column read here (the winner's included: chosen columns are frozen)
                const int e4 = (j < RS ? j - R + 3 : S) & ~3;
                const double *wp = wsm + c;  // this candidate's column
                for (int o = 0; o < e4 * Npad; o += 4 * Npad) {  // shared offsets fit 32 bits
                    acc0 = fma(wcs[o], wp[o], acc0);
                    acc1 = fma(wcs[o + Npad], wp[o + Npad], acc1);
                    acc0 = fma(wcs[o + 2 * Npad], wp[o + 2 * Npad], acc0);
                    acc1 = fma(wcs[o + 3 * Npad], wp[o + 3 * Npad], acc1);
                }
                const double e = corr_from_d2(d2, rth) - ((acc0 + acc1) + (acc2 + acc3));
                const double wn = e * rrho;
                if (j < R) {
#pragma unroll
                    for (int b = 0; b < R; b++)
                        if (b == j) wr[q][b] = wn;
                } else if (chosen[q]) {
                    // a chosen column is never read after its own step: keep its rows >= j
                    // at 0 so the padded dot above sees no write from this step
                } else if (j < RS) {
                    wsm[(j - R) * Npad + c] = wn;
                } else {
                    gw[(j - RS) * Npad + c] = wn;
                }
                s[q] = fma(-wn, wn, s[q]);
                cov[q] = fma(-znew, wn, cov[q]);
            }
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
                uint32_t f = fl;
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
    const size_t fixed = ((size_t)inc_n4(n) * 2 + 2 * (size_t)inc_wl(n, pl.R) + Npad + 200) * sizeof(double);
    size_t avail = smem_optin > fixed + 1024 ? smem_optin - fixed - 1024 : 0;
    int S = (int)(avail / ((size_t)Npad * sizeof(double)));
    const int need = n - pl.R > 0 ? n - pl.R : 0;
    if (S > inc_n4(need)) S = inc_n4(need);
    S &= ~3;  // the shared dot runs in groups of 4 entries
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
