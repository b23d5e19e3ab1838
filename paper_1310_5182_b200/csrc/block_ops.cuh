// block_ops.cuh — CTA-level building blocks for the local GP state kept in
// shared memory: reductions, the partitioned-inverse append (row a4) and the
// fresh-Cholesky prediction (row a5). Used by the fused local-design kernels
// and by the single-row diagnostic kernels.
#pragma once
#include "lagp_internal.cuh"

namespace lagp {

// Sum over the CTA (blockDim.x multiple of 32, <= 1024). `scratch` >= 33 doubles.
// Deterministic: fixed shuffle tree, then warp partials summed in warp order.
__device__ __forceinline__ double block_sum(double v, double *scratch) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    if (wid == 0) {  // second level: warp 0 over the warp partials (fixed tree)
        const int nw = blockDim.x >> 5;
        double s = lane < nw ? scratch[lane] : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) scratch[32] = s;
    }
    __syncthreads();
    const double s = scratch[32];
    __syncthreads();
    return s;
}

// Block-wide merge of per-thread Top2 records; every thread receives the result.
__device__ __forceinline__ Top2 block_top2(Top2 t, double *scratch /* >= 132 doubles */) {
    warp_merge_top2(t);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) {
        scratch[4 * wid + 0] = t.d1;
        scratch[4 * wid + 1] = t.d2;
        scratch[4 * wid + 2] = int_bits_to_double(t.i1);
        scratch[4 * wid + 3] = int_bits_to_double(t.pos);
    }
    __syncthreads();
    if (wid == 0) {  // second level: warp 0 merges the warp results (fixed tree)
        const int nw = blockDim.x >> 5;
        Top2 r;
        r.init();
        if (lane < nw) {
            r.d1 = scratch[4 * lane + 0];
            r.d2 = scratch[4 * lane + 1];
            r.i1 = double_bits_to_int(scratch[4 * lane + 2]);
            r.pos = double_bits_to_int(scratch[4 * lane + 3]);
        }
        warp_merge_top2(r);
        if (lane == 0) {
            scratch[128] = r.d1;
            scratch[129] = r.d2;
            scratch[130] = int_bits_to_double(r.i1);
            scratch[131] = int_bits_to_double(r.pos);
        }
    }
    __syncthreads();
    Top2 r;
    r.d1 = scratch[128];
    r.d2 = scratch[129];
    r.i1 = double_bits_to_int(scratch[130]);
    r.pos = double_bits_to_int(scratch[131]);
    __syncthreads();
    return r;
}

// Fast block argmax for non-negative scores: each thread brings its best (d1, i1)
// and its own second best d2 (d = score >= 0; invalid = no candidate). The warp
// and block levels use redux.sync max/min on the 64-bit pattern of the doubles
// (non-negative doubles order like their bits) instead of shuffle trees:
//   d1 = max score, i1 = lowest global index among exact maxima (R7),
//   d2 = max of everything else (for the top-2 gap). Every thread gets the result;
// i1 = INT_MAX when no thread had a candidate. `scratch` >= 100 doubles.
struct ArgTop {
    double d1, d2;
    int i1;   // global index of the winner, -1 if none
    int pos;  // caller's payload of the winner (pool position)
};
__device__ __forceinline__ void warp_argtop(unsigned long long &k1, unsigned &i1, unsigned long long &k2, int &pos) {
    const unsigned full = 0xffffffffu;
    const unsigned hi = (unsigned)(k1 >> 32), lo = (unsigned)k1;
    const unsigned mhi = __reduce_max_sync(full, hi);
    const unsigned mlo = __reduce_max_sync(full, hi == mhi ? lo : 0u);
    const bool ismax = (hi == mhi && lo == mlo);
    const unsigned mi = __reduce_min_sync(full, ismax ? i1 : 0xffffffffu);
    const bool win = ismax && i1 == mi;
    const unsigned wb = __ballot_sync(full, win);
    pos = __shfl_sync(full, pos, wb ? __ffs(wb) - 1 : 0);
    // second: the winner contributes its own second, everyone else its best
    const unsigned long long c2 = (win && (__ffs(wb) - 1) == (int)(threadIdx.x & 31)) ? k2 : k1;
    const unsigned shi = __reduce_max_sync(full, (unsigned)(c2 >> 32));
    const unsigned slo = __reduce_max_sync(full, (unsigned)(c2 >> 32) == shi ? (unsigned)c2 : 0u);
    k1 = ((unsigned long long)mhi << 32) | mlo;
    i1 = mi;
    k2 = ((unsigned long long)shi << 32) | slo;
}
__device__ __forceinline__ ArgTop block_argtop(double d1, int i1, double d2, int pos, double *scratch) {
    // invalid entries carry key 0 and index 0xffffffff (lose every tie)
    unsigned long long k1 = (unsigned long long)__double_as_longlong(d1 > 0.0 ? d1 : 0.0);
    unsigned long long k2 = (unsigned long long)__double_as_longlong(d2 > 0.0 ? d2 : 0.0);
    unsigned ii = (unsigned)i1;
    warp_argtop(k1, ii, k2, pos);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long *sk = reinterpret_cast<unsigned long long *>(scratch);
    __syncthreads();
    if (lane == 0) {
        sk[3 * wid + 0] = k1;
        sk[3 * wid + 1] = ((unsigned long long)(unsigned)pos << 32) | ii;
        sk[3 * wid + 2] = k2;
    }
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        unsigned long long a1 = 0, a2 = 0;
        unsigned ai = 0xffffffffu;
        int ap = -1;
        if (lane < nw) {
            a1 = sk[3 * lane + 0];
            ai = (unsigned)sk[3 * lane + 1];
            ap = (int)(unsigned)(sk[3 * lane + 1] >> 32);
            a2 = sk[3 * lane + 2];
        }
        warp_argtop(a1, ai, a2, ap);
        if (lane == 0) {
            sk[96] = a1;
            sk[97] = ((unsigned long long)(unsigned)ap << 32) | ai;
            sk[98] = a2;
        }
    }
    __syncthreads();
    ArgTop r;
    r.d1 = __longlong_as_double((long long)sk[96]);
    r.i1 = (int)(unsigned)sk[97];
    r.pos = (int)(unsigned)(sk[97] >> 32);
    r.d2 = __longlong_as_double((long long)sk[98]);
    __syncthreads();
    return r;
}

// block_argtop with the scratch double-buffered by `parity` (alternate calls
// must alternate parity) and no trailing barrier: two __syncthreads instead of
// three. `scratch` >= 200 doubles. Safe when at least one other barrier
// separates two calls with the same parity.
__device__ __forceinline__ ArgTop block_argtop_db(double d1, int i1, double d2, int pos, double *scratch,
                                                  int parity) {
    unsigned long long k1 = (unsigned long long)__double_as_longlong(d1 > 0.0 ? d1 : 0.0);
    unsigned long long k2 = (unsigned long long)__double_as_longlong(d2 > 0.0 ? d2 : 0.0);
    unsigned ii = (unsigned)i1;
    warp_argtop(k1, ii, k2, pos);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long *sk = reinterpret_cast<unsigned long long *>(scratch) + parity * 100;
    if (lane == 0) {
        sk[3 * wid + 0] = k1;
        sk[3 * wid + 1] = ((unsigned long long)(unsigned)pos << 32) | ii;
        sk[3 * wid + 2] = k2;
    }
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        unsigned long long a1 = 0, a2 = 0;
        unsigned ai = 0xffffffffu;
        int ap = -1;
        if (lane < nw) {
            a1 = sk[3 * lane + 0];
            ai = (unsigned)sk[3 * lane + 1];
            ap = (int)(unsigned)(sk[3 * lane + 1] >> 32);
            a2 = sk[3 * lane + 2];
        }
        warp_argtop(a1, ai, a2, ap);
        if (lane == 0) {
            sk[96] = a1;
            sk[97] = ((unsigned long long)(unsigned)ap << 32) | ai;
            sk[98] = a2;
        }
    }
    __syncthreads();
    ArgTop r;
    r.d1 = __longlong_as_double((long long)sk[96]);
    r.i1 = (int)(unsigned)sk[97];
    r.pos = (int)(unsigned)(sk[97] >> 32);
    r.d2 = __longlong_as_double((long long)sk[98]);
    return r;
}

// block_argtop with ONE barrier: lane 0 of every warp posts the warp's result,
// then every warp reduces the posts itself (redundantly). `scratch` >= 200
// doubles, double-buffered by `parity`; safe when at least one other barrier
// separates two calls with the same parity.
__device__ __forceinline__ ArgTop block_argtop_1b(double d1, int i1, double d2, int pos, double *scratch,
                                                  int parity) {
    unsigned long long k1 = (unsigned long long)__double_as_longlong(d1 > 0.0 ? d1 : 0.0);
    unsigned long long k2 = (unsigned long long)__double_as_longlong(d2 > 0.0 ? d2 : 0.0);
    unsigned ii = (unsigned)i1;
    warp_argtop(k1, ii, k2, pos);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long *sk = reinterpret_cast<unsigned long long *>(scratch) + parity * 100;
    if (lane == 0) {
        sk[3 * wid + 0] = k1;
        sk[3 * wid + 1] = ((unsigned long long)(unsigned)pos << 32) | ii;
        sk[3 * wid + 2] = k2;
    }
    __syncthreads();
    const int nw = blockDim.x >> 5;
    unsigned long long a1 = 0, a2 = 0;
    unsigned ai = 0xffffffffu;
    int ap = -1;
    if (lane < nw) {
        a1 = sk[3 * lane + 0];
        ai = (unsigned)sk[3 * lane + 1];
        ap = (int)(unsigned)(sk[3 * lane + 1] >> 32);
        a2 = sk[3 * lane + 2];
    }
    warp_argtop(a1, ai, a2, ap);
    ArgTop r;
    r.d1 = __longlong_as_double((long long)a1);
    r.i1 = (int)ai;
    r.pos = ap;
    r.d2 = __longlong_as_double((long long)a2);
    return r;
}

// Partitioned-inverse append (a4; Eq (6)): given the
// explicit K_j^{-1} in Kinv (leading dimension ld, symmetric), k = k_j(x_new)
// and kdiag = K(x_new,x_new) + eta, overwrite Kinv with K_{j+1}^{-1}:
//   u = K^{-1} k,  s = kdiag - k^T u,
//   K_{j+1}^{-1} = [[K^{-1} + u u^T / s, -u/s], [-u^T/s, 1/s]].
// Entry (a,b) and (b,a) use the same IEEE operations, so symmetry is exact.
// `u` is scratch (>= j+1). Returns s (<= 0 means K_{j+1} is not PD).
__device__ inline double pinv_append(double *Kinv, int ld, int j, const double *k, double kdiag, double *u,
                              double *scratch) {
    const int tid = threadIdx.x;
    for (int a = tid; a < j; a += blockDim.x) {
        double acc = 0.0;
        const double *row = Kinv + a * ld;
        for (int b = 0; b < j; b++) acc = fma(row[b], k[b], acc);
        u[a] = acc;
    }
    __syncthreads();
    double part = 0.0;
    for (int a = tid; a < j; a += blockDim.x) part = fma(k[a], u[a], part);
    const double s = kdiag - block_sum(part, scratch);
    const int jj = j * j;
    for (int e = tid; e < jj; e += blockDim.x) {
        int a = e / j, b = e - a * j;
        Kinv[a * ld + b] = __dadd_rn(Kinv[a * ld + b], __ddiv_rn(__dmul_rn(u[a], u[b]), s));
    }
    for (int a = tid; a < j; a += blockDim.x) {
        double v = -__ddiv_rn(u[a], s);
        Kinv[a * ld + j] = v;
        Kinv[j * ld + a] = v;
    }
    if (tid == 0) Kinv[j * ld + j] = __ddiv_rn(1.0, s);
    __syncthreads();
    return s;
}

// w = Kinv * h for the leading j×j block.
__device__ __forceinline__ void block_matvec(const double *Kinv, int ld, int j, const double *h, double *w) {
    for (int a = threadIdx.x; a < j; a += blockDim.x) {
        double acc = 0.0;
        const double *row = Kinv + a * ld;
        for (int b = 0; b < j; b++) acc = fma(row[b], h[b], acc);
        w[a] = acc;
    }
    __syncthreads();
}

// a5 — Eq (1)-(2) with N -> n on D_n(x) (Fig 1 step 5):
// fresh Cholesky of K_n = C(X_n) + eta I built in `A` (n×n, ld), then
//   mean = h^T K^{-1} Y, psi = Y^T K^{-1} Y, s2 = psi (1 + eta - h^T K^{-1} h)/n,
//   var = s2 n/(n-2) (NaN if n <= 2).
// Xn [n×p] (row-major, smem or global), Yn [n], h [n]; y1,y2 scratch [n].
// Returns false if K_n is not numerically PD.
__device__ inline bool block_predict(double *A, int ld, int n, int p, const double *Xn, const double *Yn,
                              const double *h, double rtheta, double eta, double *y1, double *y2,
                              double *scratch, double *mean, double *s2, double *var) {
    const int tid = threadIdx.x;
    for (int e = tid; e < n * n; e += blockDim.x) {
        int a = e / n, b = e - a * n;
        if (b <= a) {
            double v = corr_from_d2(sqdist_fma(Xn + a * p, Xn + b * p, p), rtheta);
            if (a == b) v += eta;
            A[a * ld + b] = v;
        }
    }
    __syncthreads();
    // right-looking Cholesky, lower triangle in place
    __shared__ int bad;
    if (tid == 0) bad = 0;
    __syncthreads();
    for (int k = 0; k < n; k++) {
        if (tid == 0) {
            double dkk = A[k * ld + k];
            if (!(dkk > 0.0)) bad = 1;
            A[k * ld + k] = sqrt(dkk);
        }
        __syncthreads();
        const double lkk = A[k * ld + k];
        for (int i = k + 1 + tid; i < n; i += blockDim.x) A[i * ld + k] /= lkk;
        __syncthreads();
        const int m = n - k - 1;  // trailing (m×m lower) update
        const int tri = m * (m + 1) / 2;
        for (int e = tid; e < tri; e += blockDim.x) {
            // map e -> (r, c) with c <= r in the trailing block
            int r = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
            while ((r + 1) * (r + 2) / 2 <= e) r++;
            while (r * (r + 1) / 2 > e) r--;
            int c = e - r * (r + 1) / 2;
            int i = k + 1 + r, jj = k + 1 + c;
            A[i * ld + jj] = fma(-A[i * ld + k], A[jj * ld + k], A[i * ld + jj]);
        }
        __syncthreads();
    }
    // forward / back substitution, warp 0 on h, warp 1 on Y
    const int lane = tid & 31, wid = tid >> 5;
    if (wid < 2) {
        const double *b = (wid == 0) ? h : Yn;
        double *y = (wid == 0) ? y1 : y2;
        for (int i = 0; i < n; i++) {
            double acc = 0.0;
            for (int t = lane; t < i; t += 32) acc = fma(A[i * ld + t], y[t], acc);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) y[i] = (b[i] - acc) / A[i * ld + i];
            __syncwarp();
        }
        for (int i = n - 1; i >= 0; i--) {
            double acc = 0.0;
            for (int t = i + 1 + lane; t < n; t += 32) acc = fma(A[t * ld + i], y[t], acc);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) y[i] = (y[i] - acc) / A[i * ld + i];
            __syncwarp();
        }
    }
    __syncthreads();
    double pm = 0.0, pp = 0.0, ph = 0.0;
    for (int i = tid; i < n; i += blockDim.x) {
        pm = fma(h[i], y2[i], pm);
        pp = fma(Yn[i], y2[i], pp);
        ph = fma(h[i], y1[i], ph);
    }
    double mu = block_sum(pm, scratch);
    double psi = block_sum(pp, scratch);
    double hKh = block_sum(ph, scratch);
    double sc = psi * (1.0 + eta - hKh) / (double)n;
    *mean = mu;
    *s2 = sc;
    *var = (n > 2) ? sc * (double)n / (double)(n - 2) : __longlong_as_double(0x7ff8000000000000LL);
    return bad == 0;
}

}  // namespace lagp
