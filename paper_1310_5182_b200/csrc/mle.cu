// mle.cu — row f2: the local MLE theta-hat_n(x) | D_n(x) of Fig 1
// step 3 on the concentrated likelihood Eq (3), by the
// safeguarded Newton of reading R21 on tau = log(theta), with the analytic
// derivatives of reading R20; then the step-5 prediction (Eq (1)-(2))
// at theta-hat on the same D_n(x).
//
//   l(theta)  = lgamma(n/2) - (n/2) log(2 pi) - (1/2) log|K| - (n/2) log(psi/2)
//   P = dK/dtau   = C o (D/theta),   Q = d2K/dtau2 = C o (D/theta) o (D/theta - 1)
//   dl/dtau   = -1/2 tr(A P) + (n/2) a^T P a / psi                 (A = K^{-1}, a = A Y)
//   d2l/dtau2 = -1/2 tr(A Q) + 1/2 tr(A P A P) - (n/2)(2 v^T A v - a^T Q a)/psi
//               + (n/2)(a^T P a / psi)^2                            (v = P a)
//
// B200 mapping: one CTA of 128 threads per location (persistent grid, four CTAs
// per SM at n = 50, so four locations' latency-bound factorizations overlap). Two
// n×n buffers hold everything, each split at the diagonal:
//   X: lower (with the diagonal) K -> L (Cholesky) -> A = K^{-1}; strict upper P = dK/dtau
//   Y: lower (with the diagonal) W = L^{-1};                   strict upper D (squared distances)
// in shared memory when they fit, else in a per-CTA HBM slab (L2-resident). Every
// evaluation: K (n^2/2 exp) and P = C o (D/theta) from the same exp values, a
// right-looking Cholesky with two columns per barrier, W by quad-parallel
// substitution in 2x2 block form, A = W^T W on DMMA, then the traces; tr(APAP) comes
// from pairs of 8x8 tiles of T = AP (DMMA) without storing T. The Newton iteration runs
// uniformly on block-reduced scalars. The prediction at theta-hat reuses W when the
// last evaluation was at theta-hat.
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "launch.h"

namespace lagp {

constexpr int MLE_THREADS = 128;
constexpr int MLE_NW = MLE_THREADS / 32;
constexpr int MLE_MAXIT = 64;

#ifdef LAGP_MLE_PROF
// phase clocks (profiling builds only): thread 0 of CTA b accumulates cycles per phase
// 0 K + Cholesky, 1 inverse, 2 W^T W, 3 a = A Y + psi, 4 v = P a, 5 tr(APAP), 6 traces,
// 7 evaluations counted
__device__ long long g_mle_ph[1024][8];
#define MLE_PH(k)                                                                   \
    do {                                                                            \
        if (threadIdx.x == 0 && blockIdx.x < 1024) {                                \
            long long t_;                                                           \
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_)::"memory");            \
            g_mle_ph[blockIdx.x][k] += t_ - ph_t0;                                  \
            ph_t0 = t_;                                                             \
        }                                                                           \
    } while (0)
#define MLE_PH0()                                                                   \
    long long ph_t0 = 0;                                                            \
    if (threadIdx.x == 0) {                                                         \
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(ph_t0)::"memory");             \
        if (blockIdx.x < 1024) g_mle_ph[blockIdx.x][7] += 1;                        \
    }
#else
#define MLE_PH(k) do {} while (0)
#define MLE_PH0() do {} while (0)
#endif

struct MleEval {
    double l, g, h, psi;
    bool ok;
};

// Per-location vectors (doubles): responses Yr[n], al[n] = A Yr, v[n] = P al, hv[n],
// rd[n] = 1/L_ii, Xn[n p], Tb[(n - h) h] (block-inverse temporary), tp[MLE_NW][64]
// (per-warp 8x8 transposes), red[8 * 8] (reductions)
__host__ __device__ inline size_t mle_vec_doubles(int n, int p) {
    const int h = n >= 24 ? n / 2 : n;
    return (size_t)5 * n + (size_t)n * p + (size_t)(n - h) * h + 64 * MLE_NW + 64 + 8;
}

// Sums of K values over the CTA; every thread gets them (warp shuffle tree, then the
// warp partials in warp order: deterministic)
template <int K>
__device__ __forceinline__ void cta_sum(double (&v)[K], double *red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; k++)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; k++) red[wid * K + k] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; k++) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < MLE_NW; w++) t += red[w * K + k];
        v[k] = t;
    }
    __syncthreads();
}

// row a of entry e of a lower triangle stored row by row (a(a+1)/2 <= e < (a+1)(a+2)/2):
// the float root, corrected in integers
__device__ __forceinline__ int tri_row(int e) {
    int a = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
    while (a * (a + 1) / 2 > e) a--;
    while ((a + 1) * (a + 2) / 2 <= e) a++;
    return a;
}

__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

// K = C + eta I into X's lower triangle (and, with deriv, P = C o (D/theta) into its strict
// upper triangle from the same exp values), then its Cholesky factor in place (lower,
// row-major). Returns false when a pivot is not positive.
__device__ bool mle_chol(const double *Y, double *X, int n, double rth, double eta, bool deriv) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // the n(n+1)/2 lower-triangle entries dealt over all threads (row a of entry e from
    // the triangular root, corrected in integers)
    const int ne = n * (n + 1) / 2;
    for (int e = tid; e < ne; e += blockDim.x) {
        const int a = tri_row(e);
        const int b = e - a * (a + 1) / 2;
        const double d = a == b ? 0.0 : Y[b * n + a];  // D_ab (upper storage)
        const double c = exp_nonpos(-d * rth);
        X[a * n + b] = c + (a == b ? eta : 0.0);
        if (deriv && b < a) X[b * n + a] = c * (d * rth);
    }
    __shared__ int bad;
    if (tid == 0) bad = 0;
    __syncthreads();
    // Two columns (k, k+1) per barrier. Every thread forms the pair's factors itself:
    // 1/sqrt(L_kk), l_{k+1,k} = L_{k+1,k}/sqrt(L_kk), the updated pivot
    // d = L_{k+1,k+1} - l_{k+1,k}^2 and 1/sqrt(d); each row then gets its two column
    // values on the fly and the trailing block its rank-2 update — the one-column
    // right-looking order operation for operation. The pair's columns are written one
    // step later (no thread reads them then).
    int kp = -1;
    bool ptwo = false;
    double prl = 0.0, pc10 = 0.0, prl2 = 0.0, pd2 = 0.0;
    for (int k = 0; k < n; k += 2) {
        const bool two = k + 1 < n;
        const double dkk = X[k * n + k];
        if (!(dkk > 0.0)) {
            if (tid == 0) bad = 1;
            break;  // uniform: every thread read the same pivot
        }
        const double rl = rsqrt_nr(dkk);
        double c10 = 0.0, d2 = 0.0, rl2 = 0.0;
        if (two) {
            c10 = X[(k + 1) * n + k] * rl;
            d2 = fma(-c10, c10, X[(k + 1) * n + (k + 1)]);
            if (!(d2 > 0.0)) {
                if (tid == 0) bad = 1;
                break;  // uniform
            }
            rl2 = rsqrt_nr(d2);
        }
        if (kp >= 0) {  // the previous pair's columns, rows >= k
            for (int i = k + tid; i < n; i += blockDim.x) {
                const double lik = X[i * n + kp] * prl;
                X[i * n + kp] = lik;
                if (ptwo) X[i * n + kp + 1] = fma(-lik, pc10, X[i * n + kp + 1]) * prl2;
            }
            if (tid == 0 && ptwo) {
                X[(kp + 1) * n + kp] = pc10;
                X[(kp + 1) * n + kp + 1] = pd2;
            }
        }
        const int j0 = k + (two ? 2 : 1);
        // this lane's trailing columns jj = j0 + lane + 32 m: their two factors formed once
        // per step (the same values for every row), then each row's rank-2 update
        if (two && ((n | j0) & 1) == 0) {
            // pairs of columns per lane (jj = j0 + 2 lane + 64 m, 16-byte aligned since n and
            // j0 are even): one LDS.128 / STS.128 per two entries. When jj = i the second
            // entry is in the strict upper triangle (P, untouched here) and is written back
            // unchanged. Same fma per entry as the scalar loop.
            const int nm2 = (n - j0 + 63) >> 6;  // (uniform)
            double lj[2][2], lj1[2][2];
#pragma unroll
            for (int m = 0; m < 2; m++)
#pragma unroll
                for (int h2 = 0; h2 < 2; h2++) {
                    const int jj = j0 + 2 * lane + 64 * m + h2;
                    lj[m][h2] = lj1[m][h2] = 0.0;
                    if (m < nm2 && jj < n) {
                        lj[m][h2] = X[jj * n + k] * rl;
                        lj1[m][h2] = fma(-lj[m][h2], c10, X[jj * n + k + 1]) * rl2;
                    }
                }
            for (int i = j0 + wid; i < n; i += MLE_NW) {
                const double lik = X[i * n + k] * rl;
                const double lik1 = fma(-lik, c10, X[i * n + k + 1]) * rl2;
#pragma unroll
                for (int m = 0; m < 2; m++) {
                    if (m >= nm2) break;  // (uniform)
                    const int jj = j0 + 2 * lane + 64 * m;
                    if (jj <= i) {
                        double2 *px = reinterpret_cast<double2 *>(X + i * n + jj);
                        double2 x = *px;
                        x.x = fma(-lik1, lj1[m][0], fma(-lik, lj[m][0], x.x));
                        if (jj + 1 <= i) x.y = fma(-lik1, lj1[m][1], fma(-lik, lj[m][1], x.y));
                        *px = x;
                    }
                }
            }
        } else {
            const int nm = (n - j0 + 31) >> 5;  // column blocks of 32 in the trailing part (uniform)
            double lj[4], lj1[4];
#pragma unroll
            for (int m = 0; m < 4; m++) {
                const int jj = j0 + lane + 32 * m;
                lj[m] = lj1[m] = 0.0;
                if (m < nm && jj < n) {
                    lj[m] = X[jj * n + k] * rl;
                    if (two) lj1[m] = fma(-lj[m], c10, X[jj * n + k + 1]) * rl2;
                }
            }
            for (int i = j0 + wid; i < n; i += MLE_NW) {
                const double lik = X[i * n + k] * rl;
                const double lik1 = two ? fma(-lik, c10, X[i * n + k + 1]) * rl2 : 0.0;
#pragma unroll
                for (int m = 0; m < 4; m++) {
                    if (m >= nm) break;  // (uniform)
                    const int jj = j0 + lane + 32 * m;
                    if (jj <= i) {
                        double v = fma(-lik, lj[m], X[i * n + jj]);
                        if (two) v = fma(-lik1, lj1[m], v);
                        X[i * n + jj] = v;
                    }
                }
            }
        }
        __syncthreads();
        kp = k;
        ptwo = two;
        prl = rl;
        pc10 = c10;
        prl2 = rl2;
        pd2 = d2;
    }
    if (kp >= 0) {  // the last pair (after a failed pivot: the pair before it, harmless)
        for (int i = kp + 2 + tid; i < n; i += blockDim.x) {
            const double lik = X[i * n + kp] * prl;
            X[i * n + kp] = lik;
            if (ptwo) X[i * n + kp + 1] = fma(-lik, pc10, X[i * n + kp + 1]) * prl2;
        }
        if (tid == 0 && ptwo) {
            X[(kp + 1) * n + kp] = pc10;
            X[(kp + 1) * n + kp + 1] = pd2;
        }
    }
    // every thread reads `bad` before any can leave the barrier
    if (__syncthreads_or(bad)) return false;
    for (int k = tid; k < n; k += blockDim.x) X[k * n + k] = sqrt(X[k * n + k]);
    __syncthreads();
    return true;
}

// W = L^{-1} into Y's lower triangle (L in X's lower triangle) by forward substitution,
// four lanes (a quad) per column, in 2x2 block form for n >= 24: W11 and W22 at the same
// time, then W21 = -W22 (L21 W11) on DMMA. The strict upper triangle of Y (D) is not
// touched: reads of W's upper part are guarded instead.
// Returns this thread's part of log|L| = sum_i log L_ii.
__device__ double mle_inverse(const double *X, double *Y, double *rd, double *Tb, int n) {
    const int tid = threadIdx.x;
    double ld = 0.0;
    for (int i = tid; i < n; i += blockDim.x) {
        rd[i] = 1.0 / X[i * n + i];
        ld += log(X[i * n + i]);
    }
    __syncthreads();
    const int h = n >= 24 ? n / 2 : n;
    const int sub = tid & 3;
    const unsigned qmask = 0xfu << (tid & 28);
    // Columns in descending order of their row counts (h-1-c for c < h, n-1-c above),
    // dealt to the quads in snake order (quad Q: positions Q, 2NQ-1-Q, 2NQ+Q, ...), so the
    // longest substitution chains do not queue behind each other on one quad
    const int nq4 = blockDim.x >> 2, d0 = n - 2 * h;
    for (int pos = tid >> 2, rnd = 0; pos < n; rnd++, pos = (rnd & 1) ? (rnd + 1) * nq4 - 1 - (tid >> 2) : rnd * nq4 + (tid >> 2)) {
        int c;
        if (h == n) {
            c = pos;
        } else if (pos < d0) {
            c = h + pos;
        } else {
            const int pi = (pos - d0) >> 1;
            c = ((pos - d0) & 1) ? pi : h + d0 + pi;
        }
        if (sub == 0) Y[c * n + c] = rd[c];
        __syncwarp(qmask);
        const int iend = c < h ? h : n;
        for (int i = c + 1; i < iend; i++) {
            double s = 0.0, s1 = 0.0;
            const double *pl = X + i * n + c + sub, *pw = Y + (c + sub) * n + c;
            int t = c + sub;
            for (; t + 4 < i; t += 8, pl += 8, pw += 8 * n) {
                s = fma(pl[0], pw[0], s);
                s1 = fma(pl[4], pw[4 * n], s1);
            }
            if (t < i) s = fma(pl[0], pw[0], s);
            s += s1;
            s += __shfl_xor_sync(qmask, s, 1);
            s += __shfl_xor_sync(qmask, s, 2);
            if (sub == 0) Y[i * n + c] = -s * rd[i];
            __syncwarp(qmask);
        }
    }
    __syncthreads();
    if (h < n) {
        // Tb = L21 W11 ((n-h) x h), then W21 = -W22 Tb, both on DMMA (8x8 tiles to warps)
        const int lane = tid & 31, g = lane >> 2, q = lane & 3;
        const int m1 = n - h, tr = (m1 + 7) >> 3, tc = (h + 7) >> 3;
        for (int tile = tid >> 5; tile < tr * tc; tile += MLE_NW) {
            const int r0 = (tile / tc) * 8, b0 = (tile - (tile / tc) * tc) * 8;
            const int ar = r0 + g, bc = b0 + g;
            double c0 = 0.0, c1 = 0.0;
            for (int kk = b0 & ~3; kk < h; kk += 4) {
                const int t = kk + q;
                const double av = (ar < m1 && t < h) ? X[(h + ar) * n + t] : 0.0;
                const double bv = (bc < h && t < h && t >= bc) ? Y[t * n + bc] : 0.0;
                dmma884(c0, c1, av, bv);
            }
            const int cc = b0 + 2 * q;
            if (ar < m1) {
                if (cc < h) Tb[ar * h + cc] = c0;
                if (cc + 1 < h) Tb[ar * h + cc + 1] = c1;
            }
        }
        __syncthreads();
        for (int tile = tid >> 5; tile < tr * tc; tile += MLE_NW) {
            const int r0 = (tile / tc) * 8, b0 = (tile - (tile / tc) * tc) * 8;
            const int ar = r0 + g, bc = b0 + g;
            const int kend = r0 + 8 < m1 ? r0 + 8 : m1;
            double c0 = 0.0, c1 = 0.0;
            for (int kk = 0; kk < kend; kk += 4) {
                const int u = kk + q;
                const double av = (ar < m1 && u < m1 && u <= ar) ? Y[(h + ar) * n + h + u] : 0.0;
                const double bv = (bc < h && u < m1) ? Tb[u * h + bc] : 0.0;
                dmma884(c0, c1, av, bv);
            }
            const int cc = b0 + 2 * q;
            if (ar < m1) {
                if (cc < h) Y[(h + ar) * n + cc] = -c0;
                if (cc + 1 < h) Y[(h + ar) * n + cc + 1] = -c1;
            }
        }
        __syncthreads();
    }
    return ld;
}

// A = W^T W into X's lower triangle (L is no longer needed), DMMA over the lower 8x8
// tiles; W lower triangular: tile (a0, b0) sums t >= max(a0, b0)
__device__ void mle_wtw(const double *Y, double *X, int n) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int g = lane >> 2, q = lane & 3, nt = (n + 7) >> 3, ntile = nt * (nt + 1) / 2;
    // two tiles per warp at a time (independent DMMA chains in one k loop; a tile's
    // products below its start are exact zeros, so its sums are unchanged)
    for (int tile = wid; tile < ntile; tile += 2 * MLE_NW) {
        int ar[2], bc[2], b0[2];
        bool has[2];
#pragma unroll
        for (int u = 0; u < 2; u++) {
            const int tl = tile + u * MLE_NW;
            has[u] = tl < ntile;
            const int ti = tri_row(tl);
            const int tj = tl - ti * (ti + 1) / 2;
            ar[u] = ti * 8 + g;
            b0[u] = tj * 8;
            bc[u] = tj * 8 + g;
        }
        const int a00 = (has[1] ? min(ar[0], ar[1]) : ar[0]) - g;  // the earlier tile row start
        double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        const int k0 = a00 & ~3;
        int oa[2], ob[2];  // offsets of W[t][ar], W[t][bc] (row-major Y), t = kk + q
#pragma unroll
        for (int u = 0; u < 2; u++) {
            oa[u] = (k0 + q) * n + ar[u];
            ob[u] = (k0 + q) * n + bc[u];
        }
        for (int kk = k0; kk < n; kk += 4) {
            const int t = kk + q;
#pragma unroll
            for (int u = 0; u < 2; u++) {
                if (u == 1 && !has[1]) break;  // (warp-uniform)
                const double av = (ar[u] < n && t < n && t >= ar[u]) ? Y[oa[u]] : 0.0;
                const double bv = (bc[u] < n && t < n && t >= bc[u]) ? Y[ob[u]] : 0.0;
                dmma884(c[u][0], c[u][1], av, bv);
                oa[u] += 4 * n;
                ob[u] += 4 * n;
            }
        }
#pragma unroll
        for (int u = 0; u < 2; u++) {
            const int cc = b0[u] + 2 * q;
            if (has[u] && ar[u] < n) {
                if (cc <= ar[u]) X[ar[u] * n + cc] = c[u][0];
                if (cc + 1 <= ar[u]) X[ar[u] * n + cc + 1] = c[u][1];
            }
        }
    }
    __syncthreads();
}

__device__ __forceinline__ double symA(const double *X, int n, int a, int b) {  // A = K^{-1}
    return a >= b ? X[a * n + b] : X[b * n + a];
}
__device__ __forceinline__ double symP(const double *X, int n, int a, int b) {  // P = dK/dtau
    return a < b ? X[a * n + b] : (a > b ? X[b * n + a] : 0.0);
}

// One evaluation of l (and with deriv, dl/dtau, d2l/dtau2) at theta = exp(tau). On return
// W = L^{-1} (Y lower), A = K^{-1} (X lower) and al = A Yr at that theta.
__device__ MleEval mle_eval(double tau, bool deriv, int n, double *X, double *Y, double *vec, double eta, int p,
                            int nv) {
    MleEval r{};
    r.l = -INFINITY;
    r.g = r.h = __longlong_as_double(0x7ff8000000000000LL);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // vectors at the kernel's stride nv (>= n, the valid prefix of an exhausted design)
    double *Yr = vec, *al = Yr + nv, *v = al + nv, *rd = v + 2 * nv;
    const int hv_ = nv >= 24 ? nv / 2 : nv;
    double *Tb = vec + 5 * nv + nv * p, *tp = Tb + (nv - hv_) * hv_, *red = tp + 64 * MLE_NW;
    const double theta = exp(tau), rth = 1.0 / theta;
    MLE_PH0();
    if (!mle_chol(Y, X, n, rth, eta, deriv)) {
        r.ok = false;
        return r;
    }
    MLE_PH(0);
    const double ld = mle_inverse(X, Y, rd, Tb, n);
    MLE_PH(1);
    mle_wtw(Y, X, n);
    MLE_PH(2);
    double pp[2] = {0.0, ld};
    // a = A Yr: two threads per row (adjacent lanes), each half of the b range (A[a][b]
    // from row a of the lower triangle for b <= a, from column a below it), halves added
    // by one shuffle
    const int bm = n >> 1;
    for (int a0 = 0; a0 < n; a0 += blockDim.x >> 1) {
        const int a = a0 + (tid >> 1), hh = tid & 1;
        double sa = 0.0;
        if (a < n) {
            const int b0 = hh ? bm : 0, b1 = hh ? n : bm, bs = a + 1 < b0 ? b0 : (a + 1 < b1 ? a + 1 : b1);
            for (int b = b0; b < bs; b++) sa = fma(X[a * n + b], Yr[b], sa);
            for (int b = bs; b < b1; b++) sa = fma(X[b * n + a], Yr[b], sa);
        }
        sa += __shfl_xor_sync(0xffffffffu, sa, 1);
        if (a < n && hh == 0) {
            al[a] = sa;
            pp[0] = fma(Yr[a], sa, pp[0]);
        }
    }
    cta_sum<2>(pp, red);  // (also orders the al writes)
    MLE_PH(3);
    const double psi = pp[0], logdet = 2.0 * pp[1];
    r.psi = psi;
    if (!(psi > 0.0)) {
        r.ok = false;
        return r;
    }
    const double hn = 0.5 * (double)n;
    r.l = lgamma(hn) - hn * log(2.0 * 3.14159265358979323846) - 0.5 * logdet - hn * log(0.5 * psi);
    r.ok = isfinite(r.l);
    if (!deriv || !r.ok) return r;
    // v = P al
    // (two threads per row as for a; P[a][b] from column a of the strict upper triangle
    // for b < a, from row a for b > a, 0 on the diagonal)
    for (int a0 = 0; a0 < n; a0 += blockDim.x >> 1) {
        const int a = a0 + (tid >> 1), hh = tid & 1;
        double sa = 0.0;
        if (a < n) {
            const int b0 = hh ? bm : 0, b1 = hh ? n : bm, bs = a < b0 ? b0 : (a < b1 ? a : b1);
            for (int b = b0; b < bs; b++) sa = fma(X[b * n + a], al[b], sa);
            for (int b = (bs > a ? bs : a + 1); b < b1; b++) sa = fma(X[a * n + b], al[b], sa);
        }
        sa += __shfl_xor_sync(0xffffffffu, sa, 1);
        if (a < n && hh == 0) v[a] = sa;
    }
    MLE_PH(4);
    // tr(APAP) = sum_ab T_ab T_ba with T = A P: 8x8 tiles of T on DMMA, a tile pair (I, J),
    // I <= J, per warp; the partner tile's transpose through the warp's 8x8 scratch
    double tTT = 0.0;
    {
        const int g = lane >> 2, q = lane & 3, nt = (n + 7) >> 3;
        double *tw = tp + 64 * wid;
        for (int pr = wid; pr < nt * (nt + 1) / 2; pr += MLE_NW) {
            const int ti = tri_row(pr);
            const int tj = pr - ti * (ti + 1) / 2;  // tj <= ti
            double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
            {
                // tiles (ti, tj) and (tj, ti) as two independent accumulation chains in one
                // k loop (each tile's k order unchanged)
                const bool two = ti != tj;  // (warp-uniform)
                const int ar0 = ti * 8 + g, bc0 = tj * 8 + g;
                // The four operands come from four offset streams of X (row-major):
                //   x1 = X[ar0][k], x2 = X[k][ar0], x3 = X[bc0][k], x4 = X[k][bc0]
                // A[ar0][k] = k <= ar0 ? x1 : x2    P[k][bc0] = k < bc0 ? x4 : (k > bc0 ? x3 : 0)
                // A[bc0][k] = k <= bc0 ? x3 : x4    P[k][ar0] = k < ar0 ? x2 : (k > ar0 ? x1 : 0)
                // (A in the lower triangle with the diagonal, P in the strict upper one).
                const bool ra = ar0 < n, rb = bc0 < n;
                int s1 = ar0 * n + q, s2 = q * n + ar0, s3 = bc0 * n + q, s4 = q * n + bc0;
                for (int kk = 0; kk < n; kk += 4, s1 += 4, s2 += 4 * n, s3 += 4, s4 += 4 * n) {
                    const int k = kk + q;
                    const bool kv = k < n;
                    const double x1 = (ra && kv) ? X[s1] : 0.0, x2 = (ra && kv) ? X[s2] : 0.0;
                    const double x3 = (rb && kv) ? X[s3] : 0.0, x4 = (rb && kv) ? X[s4] : 0.0;
                    const double av0 = k <= ar0 ? x1 : x2;
                    const double bv0 = k < bc0 ? x4 : (k > bc0 ? x3 : 0.0);
                    if (two) {
                        const double av1 = k <= bc0 ? x3 : x4;
                        const double bv1 = k < ar0 ? x2 : (k > ar0 ? x1 : 0.0);
                        dmma884(c[1][0], c[1][1], av1, bv1);
                    }
                    dmma884(c[0][0], c[0][1], av0, bv0);
                }
            }
            // tile (ti, tj) in c[0]; its partner (tj, ti) in c[1] (or c[0] on the diagonal)
            const int src = ti == tj ? 0 : 1;
            tw[g * 8 + 2 * q] = c[src][0];
            tw[g * 8 + 2 * q + 1] = c[src][1];
            __syncwarp();
            const double wgt = ti == tj ? 1.0 : 2.0;
            tTT = fma(wgt * c[0][0], tw[(2 * q) * 8 + g], tTT);
            tTT = fma(wgt * c[0][1], tw[(2 * q + 1) * 8 + g], tTT);
            __syncwarp();
        }
    }
    __syncthreads();  // v
    MLE_PH(5);
    double tAP = 0.0, tAQ = 0.0, aQa = 0.0, aPa = 0.0, vAv = 0.0;
    // the lower triangle (off-diagonal terms twice; P and Q vanish on the diagonal), its
    // entries dealt over all threads as in mle_chol
    const int ne = n * (n + 1) / 2;
    for (int e = tid; e < ne; e += blockDim.x) {
            const int a = tri_row(e);
            const int b = e - a * (a + 1) / 2;
            const double Aab = X[a * n + b];
            if (a == b) {
                vAv = fma(v[a] * Aab, v[a], vAv);
                continue;
            }
            const double Pab = X[b * n + a];
            const double Qab = Pab * (Y[b * n + a] * rth - 1.0);
            tAP = fma(2.0 * Aab, Pab, tAP);
            tAQ = fma(2.0 * Aab, Qab, tAQ);
            aQa = fma(2.0 * al[a] * Qab, al[b], aQa);
            aPa = fma(2.0 * al[a] * Pab, al[b], aPa);
            vAv = fma(2.0 * v[a] * Aab, v[b], vAv);
        }
    double t6[6] = {tAP, tAQ, tTT, aQa, aPa, vAv};
    cta_sum<6>(t6, red);
    MLE_PH(6);
    const double qv = t6[4] / psi;
    r.g = -0.5 * t6[0] + hn * qv;
    r.h = -0.5 * t6[1] + 0.5 * t6[2] - hn * (2.0 * t6[5] - t6[3]) / psi + hn * qv * qv;
    r.ok = isfinite(r.g) && isfinite(r.h);
    return r;
}

__global__ void __launch_bounds__(MLE_THREADS, 4)
mle_kernel(MleArgs A) {
    extern __shared__ __align__(16) double sm[];
    const int n = A.n, p = A.p;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const size_t vd = mle_vec_doubles(n, p);
    double *mats = A.use_smem ? sm : A.ws + (size_t)blockIdx.x * (2 * (size_t)n * n + vd);
    double *X = mats, *Y = X + (size_t)n * n, *vec = Y + (size_t)n * n;
    double *Yr = vec, *hv = vec + 3 * n, *Xn = vec + 5 * n, *red = vec + vd - 64 - 8;
    __shared__ int jn_s;
    const double lo = log(A.lo), hi = log(A.hi);

    for (int64_t xi = blockIdx.x; xi < A.M; xi += gridDim.x) {
        const int32_t *idx = A.idx + xi * (int64_t)n;
        if (tid == 0) jn_s = n;
        __syncthreads();
        for (int t = tid; t < n; t += blockDim.x)
            if (idx[t] < 0) atomicMin(&jn_s, t);
        __syncthreads();
        const int m = jn_s;  // the design's valid prefix (exhausted designs are shorter)
        double *Ym = Y;  // the buffers are laid out with stride m below
        for (int e = tid; e < m * p; e += blockDim.x) Xn[e] = A.X[(int64_t)idx[e / p] * p + (e % p)];
        for (int a = tid; a < m; a += blockDim.x) Yr[a] = A.Z[idx[a]];
        __syncthreads();
        for (int a = wid; a < m; a += MLE_NW)  // D into Y's strict upper triangle
            for (int b = a + 1 + lane; b < m; b += 32) Ym[a * m + b] = sqdist_fma(Xn + a * p, Xn + b * p, p);
        __syncthreads();

        const double theta0 = A.theta_in ? A.theta_in[xi] : A.theta0;
        double tau = fmin(fmax(log(theta0), lo), hi);
        uint32_t fl = 0;
        int it = 0;
        MleEval cur = mle_eval(tau, true, m, X, Ym, vec, A.eta, p, n);
        double last_tau = tau;
        bool last_ok = cur.ok;
        double theta_hat = theta0;
        if (!cur.ok) {
            fl |= LAGP_FLAG_MLE_FAIL;
        } else {
            for (it = 1; it <= MLE_MAXIT; it++) {
                if ((tau <= lo && cur.g <= 0.0) || (tau >= hi && cur.g >= 0.0)) break;
                if (cur.g == 0.0 && !(cur.h < 0.0)) break;
                double step = (cur.h < 0.0) ? -cur.g / cur.h : (cur.g > 0.0 ? 1.0 : -1.0);
                step = fmin(fmax(step, -1.0), 1.0);
                double tn = fmin(fmax(tau + step, lo), hi);
                MleEval nx = mle_eval(tn, true, m, X, Ym, vec, A.eta, p, n);
                last_tau = tn;
                last_ok = nx.ok;
                if (fabs(step) > 0.25 || !(cur.h < 0.0)) {
                    for (int t = 0; t < 40 && (!nx.ok || nx.l < cur.l); t++) {
                        tn = 0.5 * (tau + tn);
                        nx = mle_eval(tn, true, m, X, Ym, vec, A.eta, p, n);
                        last_tau = tn;
                        last_ok = nx.ok;
                    }
                    if (!nx.ok || nx.l < cur.l) break;  // no ascent: stay at tau
                } else if (!nx.ok) {
                    break;
                }
                const double dt = fabs(tn - tau);
                tau = tn;
                cur = nx;
                if (dt <= 1e-10 * fmax(1.0, fabs(tau))) break;
            }
            if (it > MLE_MAXIT) {
                fl |= LAGP_FLAG_MLE_MAXIT;
                it = MLE_MAXIT;
            }
            if (tau <= lo || tau >= hi) fl |= LAGP_FLAG_MLE_BOUND;
            theta_hat = exp(tau);
        }
        // Fig 1 step 5 at theta-hat (the incoming theta when the MLE failed), from the
        // factor: with W = L^{-1}, a = W h and b = W Y give mean = a.b, h^T K^{-1} h = a.a,
        // psi = b.b. W is still the one of the last evaluation when that was at tau_p.
        const double tau_p = cur.ok ? tau : log(theta0);
        bool fin_ok = last_ok;
        if (!(last_ok && last_tau == tau_p)) fin_ok = mle_eval(tau_p, false, m, X, Ym, vec, A.eta, p, n).ok;
        const double rth = 1.0 / exp(tau_p);
        const double *xq = A.XX + xi * p;
        for (int a = tid; a < m; a += blockDim.x) hv[a] = corr_from_d2(sqdist_fma(Xn + a * p, xq, p), rth);
        __syncthreads();
        double s3[3] = {0.0, 0.0, 0.0};
        for (int a = tid; a < m; a += blockDim.x) {
            double sa = 0.0, sb = 0.0;
            for (int b = 0; b <= a; b++) {
                sa = fma(Ym[a * m + b], hv[b], sa);
                sb = fma(Ym[a * m + b], Yr[b], sb);
            }
            s3[0] = fma(sa, sb, s3[0]);
            s3[1] = fma(sa, sa, s3[1]);
            s3[2] = fma(sb, sb, s3[2]);
        }
        cta_sum<3>(s3, red);
        const double mu = s3[0], hAh = s3[1], psi_p = s3[2];
        if (tid == 0) {
            const double sc = psi_p * (1.0 + A.eta - hAh) / (double)m;
            const double vr = m > 2 ? sc * (double)m / (double)(m - 2) : __longlong_as_double(0x7ff8000000000000LL);
            const double qnan = __longlong_as_double(0x7ff8000000000000LL);
            if (!fin_ok || !isfinite(mu) || !isfinite(sc)) fl |= LAGP_FLAG_NONFINITE;
            A.theta_out[xi] = theta_hat;
            if (A.loglik_out) A.loglik_out[xi] = cur.l;
            if (A.iters_out) A.iters_out[xi] = it;
            if (A.flags_out) A.flags_out[xi] |= fl;
            // K not positive definite at the prediction's theta: no factor, no
            // prediction (NaN, as oracle_predict reports it)
            if (A.mean) A.mean[xi] = fin_ok ? mu : qnan;
            if (A.s2) A.s2[xi] = fin_ok ? sc : qnan;
            if (A.var) A.var[xi] = fin_ok ? vr : qnan;
            if ((fl & LAGP_FLAG_NONFINITE) && A.n_partial) atomicAdd(A.n_partial, 1);
        }
        __syncthreads();
    }
}

size_t mle_smem_bytes(int n, int p) { return (2 * (size_t)n * n + mle_vec_doubles(n, p)) * sizeof(double); }

size_t mle_ws_bytes(int grid, int n, int p, bool use_smem) {
    if (use_smem) return 0;
    return (size_t)grid * (2 * (size_t)n * n + mle_vec_doubles(n, p)) * sizeof(double);
}

int mle_blocks_per_sm(int n, int p, bool use_smem) {
    const size_t smem = use_smem ? mle_smem_bytes(n, p) : 0;
    if (use_smem && cudaFuncSetAttribute(mle_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, mle_kernel, MLE_THREADS, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return b;
}

cudaError_t launch_mle(const MleArgs &a, int grid, cudaStream_t st) {
    const size_t smem = a.use_smem ? mle_smem_bytes(a.n, a.p) : 0;
    if (a.use_smem) {
        cudaError_t e = cudaFuncSetAttribute(mle_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    mle_kernel<<<grid, MLE_THREADS, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace lagp

#ifdef LAGP_MLE_PROF
extern "C" int lagp_mle_prof(long long *out, int reset) {
    if (reset) {
        static long long z[1024][8];
        return (int)cudaMemcpyToSymbol(lagp::g_mle_ph, z, sizeof(z));
    }
    return (int)cudaMemcpyFromSymbol(out, lagp::g_mle_ph, sizeof(lagp::g_mle_ph));
}
#endif
