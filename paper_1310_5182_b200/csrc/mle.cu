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
// B200 mapping: one CTA of 256 threads per location (persistent grid). The
// n×n matrices (D, K/L, W = L^{-1} then T = A P, A) live in shared memory when
// 4 n^2 doubles fit (n <= 80), else in a per-CTA HBM slab (L2-resident). Every
// evaluation: K from the stored D (n^2 exp), right-looking Cholesky with one
// barrier per column, W by per-column forward substitution, A = W^T W, then
// the traces and quadratic forms as block reductions. The Newton iteration is
// executed uniformly by all threads on block-reduced scalars.
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "launch.h"

namespace lagp {

constexpr int MLE_THREADS = 256;
constexpr int MLE_MAXIT = 64;

struct MleEval {
    double l, g, h, psi;
    bool ok;
};

// Sums of K values over the CTA in one pass (two barriers); every thread gets
// the sums. Warp partials by a fixed shuffle tree, then summed in warp order.
template <int K>
__device__ __forceinline__ void block_sum_n(double (&v)[K], double *scratch /* >= 8*K */) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < K; k++)
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; k++) scratch[wid * K + k] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; k++) {
        double t = 0.0;
        for (int w = 0; w < nw; w++) t += scratch[w * K + k];
        v[k] = t;
    }
    __syncthreads();
}

// K = C + eta I from D at 1/theta into L; Cholesky in place (lower, row-major).
// Returns false when a pivot is not positive.
__device__ bool mle_chol(const double *D, double *L, int n, double rth, double eta, double *scratch) {
    const int tid = threadIdx.x;
    for (int e = tid; e < n * n; e += blockDim.x) {
        const int a = e / n, b = e - a * n;
        if (b <= a) L[e] = exp_nonpos(-D[e] * rth) + (a == b ? eta : 0.0);
    }
    __shared__ int bad;
    if (tid == 0) bad = 0;
    __syncthreads();
    // Two columns (k, k+1) per barrier. Every thread forms the pair's factors itself:
    // 1/sqrt(L_kk), l_{k+1,k} = L_{k+1,k}/sqrt(L_kk), the updated pivot
    // d = L_{k+1,k+1} - l_{k+1,k}^2 and 1/sqrt(d); each row then gets its two column
    // values on the fly and the trailing block its rank-2 update. The arithmetic is
    // the one-column-per-step right-looking order operation for operation (the same
    // fmas, products and reciprocal square roots), so the factor is bitwise the same.
    // The pair's columns are written one step later (no thread reads them then).
    const int lane = tid & 31, nw = blockDim.x >> 5;
    int kp = -1;
    bool ptwo = false;
    double prl = 0.0, pc10 = 0.0, prl2 = 0.0, pd2 = 0.0;
    for (int k = 0; k < n; k += 2) {
        const bool two = k + 1 < n;
        const double dkk = L[k * n + k];
        if (!(dkk > 0.0)) {
            if (tid == 0) bad = 1;
            break;  // uniform: every thread read the same pivot
        }
        const double rl = rsqrt_nr(dkk);  // 1/sqrt(L_kk), seed + Newton (dkk > 0 here)
        double c10 = 0.0, d2 = 0.0, rl2 = 0.0;
        if (two) {
            c10 = L[(k + 1) * n + k] * rl;
            d2 = fma(-c10, c10, L[(k + 1) * n + (k + 1)]);
            if (!(d2 > 0.0)) {
                if (tid == 0) bad = 1;
                break;  // uniform
            }
            rl2 = rsqrt_nr(d2);
        }
        if (kp >= 0) {  // the previous pair's columns, rows >= k
            for (int i = k + tid; i < n; i += blockDim.x) {
                const double lik = L[i * n + kp] * prl;
                L[i * n + kp] = lik;
                if (ptwo) L[i * n + kp + 1] = fma(-lik, pc10, L[i * n + kp + 1]) * prl2;
            }
            if (tid == 0 && ptwo) {
                L[(kp + 1) * n + kp] = pc10;
                L[(kp + 1) * n + kp + 1] = pd2;
            }
        }
        // trailing update: rows to warps, columns to lanes (no index division)
        const int j0 = k + (two ? 2 : 1);
        for (int i = j0 + (tid >> 5); i < n; i += nw) {
            const double lik = L[i * n + k] * rl;
            const double lik1 = two ? fma(-lik, c10, L[i * n + k + 1]) * rl2 : 0.0;
            for (int jj = j0 + lane; jj <= i; jj += 32) {
                const double ljk = L[jj * n + k] * rl;
                double v = fma(-lik, ljk, L[i * n + jj]);
                if (two) v = fma(-lik1, fma(-ljk, c10, L[jj * n + k + 1]) * rl2, v);
                L[i * n + jj] = v;
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
            const double lik = L[i * n + kp] * prl;
            L[i * n + kp] = lik;
            if (ptwo) L[i * n + kp + 1] = fma(-lik, pc10, L[i * n + kp + 1]) * prl2;
        }
        if (tid == 0 && ptwo) {
            L[(kp + 1) * n + kp] = pc10;
            L[(kp + 1) * n + kp + 1] = pd2;
        }
    }
    // every thread reads `bad` before any can leave the barrier, so the next call's
    // reset (tid 0, before its own barrier) cannot race with these reads
    if (__syncthreads_or(bad)) return false;
    // every column below the diagonal is scaled (column n-1 has no such entries);
    // the diagonal takes its square roots last
    for (int k = tid; k < n; k += blockDim.x) L[k * n + k] = sqrt(L[k * n + k]);
    __syncthreads();
    (void)scratch;
    return true;
}

// W = L^{-1} (lower) by forward substitution, four lanes (a quad) per column: each
// row's dot is split over the quad and combined by two quad shuffles, which cuts
// the longest (column 0) dependent chain about 2-3x; then A = W^T W (symmetric,
// both triangles). Every lane of the quad writes the same W[i][c], so its own later
// reads of that entry need no synchronisation.
__device__ void mle_inverse(const double *L, double *W, double *A, int n) {
    const int tid = threadIdx.x;
    // 1/L_ii first (keeps the divisions off the substitution chains)
    for (int i = tid; i < n; i += blockDim.x) A[i] = 1.0 / L[i * n + i];
    __syncthreads();
    // 2x2 block form: L = [L11 0; L21 L22] -> W11 = L11^-1 and W22 = L22^-1 by the
    // substitution below at the same time (half the longest chain), then
    // W21 = -W22 (L21 W11) by two short parallel products
    const int h = n >= 24 ? n / 2 : n;
    const int sub = tid & 3;
    const unsigned qmask = 0xfu << (tid & 28);
    for (int c = tid >> 2; c < n; c += blockDim.x >> 2) {
        for (int i = sub; i < c; i += 4) W[i * n + c] = 0.0;
        W[c * n + c] = A[c];
        __syncwarp(qmask);  // every lane of the quad wrote the same values; order them for the reads
        const int iend = c < h ? h : n;
        for (int i = c + 1; i < iend; i++) {
            // two accumulators, pointer steps (the column-0 chain is the critical path)
            double s = 0.0, s1 = 0.0;
            const double *pl = L + i * n + c + sub, *pw = W + (c + sub) * n + c;
            int t = c + sub;
            for (; t + 4 < i; t += 8, pl += 8, pw += 8 * n) {
                s = fma(pl[0], pw[0], s);
                s1 = fma(pl[4], pw[4 * n], s1);
            }
            if (t < i) s = fma(pl[0], pw[0], s);
            s += s1;
            s += __shfl_xor_sync(qmask, s, 1);
            s += __shfl_xor_sync(qmask, s, 2);
            W[i * n + c] = -s * A[i];
            __syncwarp(qmask);
        }
    }
    __syncthreads();
    if (h < n) {
        // T = L21 W11 ((n-h) x h, in A's storage past the 1/L_ii entries; A is free until
        // W^T W), then W21 = -W22 T: both on the FP64 tensor path (mma.sync m8n8k4 f64,
        // 8x8 tiles to warps; W11 and W22 are lower triangular, so T's tile (., b0) sums
        // t >= b0 and W21's tile (a0, .) sums u <= a0 + 7)
        double *T = A + n;
        const int lane = tid & 31, nw = blockDim.x >> 5, g = lane >> 2, q = lane & 3;
        const int m1 = n - h, tr = (m1 + 7) >> 3, tc = (h + 7) >> 3;
        for (int tile = tid >> 5; tile < tr * tc; tile += nw) {
            const int r0 = (tile / tc) * 8, b0 = (tile - (tile / tc) * tc) * 8;
            const int ar = r0 + g, bc = b0 + g;  // ar: row of L21 / T, bc: column of W11 / T
            double c0 = 0.0, c1 = 0.0;
            for (int kk = b0 & ~3; kk < h; kk += 4) {
                const int t = kk + q;
                const double av = (ar < m1 && t < h) ? L[(h + ar) * n + t] : 0.0;
                const double bv = (bc < h && t < h) ? W[t * n + bc] : 0.0;
                asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                    : "+d"(c0), "+d"(c1)
                    : "d"(av), "d"(bv));
            }
            const int cc = b0 + 2 * q;
            if (ar < m1) {
                if (cc < h) T[ar * h + cc] = c0;
                if (cc + 1 < h) T[ar * h + cc + 1] = c1;
            }
        }
        __syncthreads();
        for (int tile = tid >> 5; tile < tr * tc; tile += nw) {
            const int r0 = (tile / tc) * 8, b0 = (tile - (tile / tc) * tc) * 8;
            const int ar = r0 + g, bc = b0 + g;  // ar: row of W22 / W21 (offset h), bc: column
            const int kend = r0 + 8 < m1 ? r0 + 8 : m1;
            double c0 = 0.0, c1 = 0.0;
            for (int kk = 0; kk < kend; kk += 4) {
                const int u = kk + q;  // column of W22 (offset h) = row of T
                const double av = (ar < m1 && u < m1) ? W[(h + ar) * n + h + u] : 0.0;
                const double bv = (bc < h && u < m1) ? T[u * h + bc] : 0.0;
                asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                    : "+d"(c0), "+d"(c1)
                    : "d"(av), "d"(bv));
            }
            const int cc = b0 + 2 * q;
            if (ar < m1) {
                if (cc < h) W[(h + ar) * n + cc] = -c0;
                if (cc + 1 < h) W[(h + ar) * n + cc + 1] = -c1;
            }
        }
        __syncthreads();
    }
    // A = W^T W on the FP64 tensor path (mma.sync m8n8k4 f64): the lower 8x8 tiles to
    // warps, mirrored; W is lower triangular, so tile (a0, b0) sums t >= max(a0, b0) only
    {
        const int lane = tid & 31, nw = blockDim.x >> 5;
        const int g = lane >> 2, q = lane & 3, nt = (n + 7) >> 3;
        for (int tile = tid >> 5; tile < nt * (nt + 1) / 2; tile += nw) {
            int ti = 0;
            while ((ti + 1) * (ti + 2) / 2 <= tile) ti++;  // lower-triangle tile (ti, tj)
            const int tj = tile - ti * (ti + 1) / 2;
            const int a0 = ti * 8, b0 = tj * 8, ar = a0 + g, bc = b0 + g;
            double c0 = 0.0, c1 = 0.0;
            for (int kk = a0 & ~3; kk < n; kk += 4) {
                const int t = kk + q;
                const double av = (ar < n && t < n) ? W[t * n + ar] : 0.0;
                const double bv = (bc < n && t < n) ? W[t * n + bc] : 0.0;
                asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                    : "+d"(c0), "+d"(c1)
                    : "d"(av), "d"(bv));
            }
            const int cc = b0 + 2 * q;
            if (ar < n) {
                if (cc < n && (ti != tj || cc <= ar)) {
                    A[ar * n + cc] = c0;
                    A[cc * n + ar] = c0;
                }
                if (cc + 1 < n && (ti != tj || cc + 1 <= ar)) {
                    A[ar * n + cc + 1] = c1;
                    A[(cc + 1) * n + ar] = c1;
                }
            }
        }
    }
    __syncthreads();
}

// One evaluation of l (and with deriv, dl/dtau, d2l/dtau2) at theta = exp(tau).
// On return A = K^{-1} and al = A Y at that theta.
__device__ MleEval mle_eval(double tau, bool deriv, int n, const double *D, double *L, double *W, double *A,
                            const double *Y, double *al, double *v, double eta, double *scratch) {
    MleEval r{};
    r.l = -INFINITY;
    r.g = r.h = __longlong_as_double(0x7ff8000000000000LL);
    const int tid = threadIdx.x;
    const double theta = exp(tau), rth = 1.0 / theta;
    if (!mle_chol(D, L, n, rth, eta, scratch)) {
        r.ok = false;
        return r;
    }
    double ld = 0.0;
    for (int k = tid; k < n; k += blockDim.x) ld += log(L[k * n + k]);
    const double logdet = 2.0 * block_sum(ld, scratch);
    mle_inverse(L, W, A, n);
    double pp = 0.0;
    for (int a = tid; a < n; a += blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < n; b++) s = fma(A[a * n + b], Y[b], s);
        al[a] = s;
        pp = fma(Y[a], s, pp);
    }
    const double psi = block_sum(pp, scratch);  // (also orders the al writes)
    r.psi = psi;
    if (!(psi > 0.0)) {
        r.ok = false;
        return r;
    }
    const double hn = 0.5 * (double)n;
    r.l = lgamma(hn) - hn * log(2.0 * 3.14159265358979323846) - 0.5 * logdet - hn * log(0.5 * psi);
    r.ok = isfinite(r.l);
    if (!deriv || !r.ok) return r;
    // P into L's storage (L no longer needed), then T = A P into W's storage
    for (int e = tid; e < n * n; e += blockDim.x) {
        const double q = D[e] * rth;
        L[e] = exp_nonpos(-q) * q;
    }
    __syncthreads();
    // T = A P on the FP64 tensor path (mma.sync m8n8k4 f64, SASS DMMA): 8x8 output tiles
    // to warps, k in steps of 4, zero-padded past n. Fragments (PTX ISA): A a = A[g][k],
    // B b = B[k][g], C {c0, c1} = C[g][2k], C[g][2k+1], with g = lane>>2, k = lane&3.
    {
        const int lane = tid & 31, nw = blockDim.x >> 5;
        const int g = lane >> 2, q = lane & 3, nt = (n + 7) >> 3;
        for (int tile = tid >> 5; tile < nt * nt; tile += nw) {
            const int a0 = (tile / nt) * 8, b0 = (tile - (tile / nt) * nt) * 8;
            const int ar = a0 + g, bc = b0 + g;
            double c0 = 0.0, c1 = 0.0;
            for (int kk = 0; kk < n; kk += 4) {
                const int k = kk + q;
                const double av = (ar < n && k < n) ? A[ar * n + k] : 0.0;
                const double bv = (k < n && bc < n) ? L[k * n + bc] : 0.0;
                asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                    : "+d"(c0), "+d"(c1)
                    : "d"(av), "d"(bv));
            }
            const int cc = b0 + 2 * q;
            if (ar < n) {
                if (cc < n) W[ar * n + cc] = c0;
                if (cc + 1 < n) W[ar * n + cc + 1] = c1;
            }
        }
    }
    // v = P a (P symmetric)
    for (int a = tid; a < n; a += blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < n; b++) s = fma(L[a * n + b], al[b], s);
        v[a] = s;
    }
    __syncthreads();
    double tAP = 0.0, tAQ = 0.0, tTT = 0.0, aQa = 0.0, aPa = 0.0, vAv = 0.0;
    for (int e = tid; e < n * n; e += blockDim.x) {
        const int a = e / n, b = e - a * n;
        const double Pab = L[e];
        const double Qab = Pab * (D[e] * rth - 1.0);
        tAP = fma(A[e], Pab, tAP);
        tAQ = fma(A[e], Qab, tAQ);
        tTT = fma(W[e], W[b * n + a], tTT);
        aQa = fma(al[a] * Qab, al[b], aQa);
        aPa = fma(al[a] * Pab, al[b], aPa);
        vAv = fma(v[a] * A[e], v[b], vAv);
    }
    {
        double t6[6] = {tAP, tAQ, tTT, aQa, aPa, vAv};
        block_sum_n<6>(t6, scratch);
        tAP = t6[0];
        tAQ = t6[1];
        tTT = t6[2];
        aQa = t6[3];
        aPa = t6[4];
        vAv = t6[5];
    }
    const double q = aPa / psi;
    r.g = -0.5 * tAP + hn * q;
    r.h = -0.5 * tAQ + 0.5 * tTT - hn * (2.0 * vAv - aQa) / psi + hn * q * q;
    r.ok = isfinite(r.g) && isfinite(r.h);
    return r;
}

__global__ void __launch_bounds__(MLE_THREADS, 2)
mle_kernel(MleArgs A) {
    extern __shared__ __align__(16) double sm[];
    const int n = A.n, p = A.p;
    const int tid = threadIdx.x;
    double *mats = A.use_smem ? sm : A.ws + (size_t)blockIdx.x * 4 * n * n;
    double *vecs = A.use_smem ? sm + 4 * n * n : A.ws + (size_t)gridDim.x * 4 * n * n + (size_t)blockIdx.x * (4 * n + n * p + 64);
    double *D = mats, *L = D + n * n, *W = L + n * n, *Am = W + n * n;
    double *Y = vecs, *al = Y + n, *v = al + n, *hv = v + n, *Xn = hv + n;
    __shared__ double scratch[64];
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
        for (int e = tid; e < m * p; e += blockDim.x) Xn[e] = A.X[(int64_t)idx[e / p] * p + (e % p)];
        for (int a = tid; a < m; a += blockDim.x) Y[a] = A.Z[idx[a]];
        __syncthreads();
        for (int e = tid; e < m * m; e += blockDim.x) {
            const int a = e / m, b = e - a * m;
            D[e] = sqdist_fma(Xn + a * p, Xn + b * p, p);
        }
        __syncthreads();

        const double theta0 = A.theta_in ? A.theta_in[xi] : A.theta0;
        double tau = fmin(fmax(log(theta0), lo), hi);
        uint32_t fl = 0;
        int it = 0;
        MleEval cur = mle_eval(tau, true, m, D, L, W, Am, Y, al, v, A.eta, scratch);
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
                MleEval nx = mle_eval(tn, true, m, D, L, W, Am, Y, al, v, A.eta, scratch);
                if (fabs(step) > 0.25 || !(cur.h < 0.0)) {
                    for (int t = 0; t < 40 && (!nx.ok || nx.l < cur.l); t++) {
                        tn = 0.5 * (tau + tn);
                        nx = mle_eval(tn, true, m, D, L, W, Am, Y, al, v, A.eta, scratch);
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
        // psi = b.b (the triangular-solve form of Eq (1)-(2), not the explicit inverse)
        const double tau_p = cur.ok ? tau : log(theta0);
        const MleEval fin = mle_eval(tau_p, false, m, D, L, W, Am, Y, al, v, A.eta, scratch);
        const double rth = 1.0 / exp(tau_p);
        const double *xq = A.XX + xi * p;
        for (int a = tid; a < m; a += blockDim.x) hv[a] = corr_from_d2(sqdist_fma(Xn + a * p, xq, p), rth);
        __syncthreads();
        double pm = 0.0, ph = 0.0, pp = 0.0;
        for (int a = tid; a < m; a += blockDim.x) {
            double sa = 0.0, sb = 0.0;
            for (int b = 0; b <= a; b++) {
                sa = fma(W[a * m + b], hv[b], sa);
                sb = fma(W[a * m + b], Y[b], sb);
            }
            pm = fma(sa, sb, pm);
            ph = fma(sa, sa, ph);
            pp = fma(sb, sb, pp);
        }
        double s3[3] = {pm, ph, pp};
        block_sum_n<3>(s3, scratch);
        const double mu = s3[0], hAh = s3[1], psi_p = s3[2];
        if (tid == 0) {
            const double sc = psi_p * (1.0 + A.eta - hAh) / (double)m;
            const double vr = m > 2 ? sc * (double)m / (double)(m - 2) : __longlong_as_double(0x7ff8000000000000LL);
            const double qnan = __longlong_as_double(0x7ff8000000000000LL);
            if (!fin.ok || !isfinite(mu) || !isfinite(sc)) fl |= LAGP_FLAG_NONFINITE;
            A.theta_out[xi] = theta_hat;
            if (A.loglik_out) A.loglik_out[xi] = cur.l;
            if (A.iters_out) A.iters_out[xi] = it;
            if (A.flags_out) A.flags_out[xi] |= fl;
            // K not positive definite at the prediction's theta: no factor, no
            // prediction (NaN, as oracle_predict reports it)
            if (A.mean) A.mean[xi] = fin.ok ? mu : qnan;
            if (A.s2) A.s2[xi] = fin.ok ? sc : qnan;
            if (A.var) A.var[xi] = fin.ok ? vr : qnan;
            if ((fl & LAGP_FLAG_NONFINITE) && A.n_partial) atomicAdd(A.n_partial, 1);
        }
        __syncthreads();
    }
}

size_t mle_smem_bytes(int n, int p) { return ((size_t)4 * n * n + 4 * n + (size_t)n * p + 64) * sizeof(double); }

size_t mle_ws_bytes(int grid, int n, int p, bool use_smem) {
    if (use_smem) return 0;
    return (size_t)grid * ((size_t)4 * n * n + 4 * n + (size_t)n * p + 64) * sizeof(double);
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
