// nn.cu — row a1: the N' nearest-neighbour candidate pool of every predictive
// location (PAPER.md P:250-253 NN sub-design; Fig 1 step 2(a) P:365; the N'
// NN candidate restriction P:484-487), exact by the key (d^2, row index) with
// d^2 accumulated by fma in the order k = 0..p-1 (reading R8).
//
// B200 design: a persistent grid of CTAs, each handling NN_Q
// queries at a time. One pass streams X through registers (coalesced rows) and
// evaluates all NN_Q queries per row, so X is read from L2 once per NN_Q
// queries. Selection is threshold-then-sort: a strided sample of X gives a
// per-query threshold tau at ~1.5 N' expected survivors; the filter pass
// appends (d^2, i) with d^2 <= tau to a per-query buffer; the buffer is
// bitonic-sorted in shared memory by (key bits, index) and its first N' rows
// are the pool. If the count lands outside [N', NN_CAP] the threshold is
// re-chosen from the sample; after a few misses the query falls back to an
// exact 8-bit radix select over the 64-bit keys (robust to massive ties).
#include <cuda_runtime.h>

#include "lagp_internal.cuh"
#include "launch.h"

namespace lagp {

constexpr int NN_THREADS = 256;
constexpr int NN_Q = 8;
constexpr int NN_SAMPLE = 2048;
constexpr int NN_CAP = 8192;
constexpr int NN_MAX_ROUNDS = 6;

struct NNSmem {
    uint64_t key[NN_CAP];
    int32_t idx[NN_CAP];
    double qx[NN_Q][LAGP_PMAX];
    double tau[NN_Q];
    int cnt[NN_Q];
    int rank[NN_Q];
    int state[NN_Q];  // 0 = active, 1 = done, 2 = fallback
    unsigned hist[256];
    int scan[NN_THREADS / 32];
    int misc[4];
};

__device__ __forceinline__ bool key_less(uint64_t ka, int ia, uint64_t kb, int ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// Bitonic sort of s.key/s.idx[0..n) ascending, n a power of two <= NN_CAP.
__device__ void bitonic_sort(NNSmem &s, int n) {
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = threadIdx.x; t < (n >> 1); t += blockDim.x) {
                int i = 2 * t - (t & (j - 1));  // lower element of the pair
                int l = i + j;
                bool up = ((i & k) == 0);
                uint64_t ki = s.key[i], kl = s.key[l];
                int ii = s.idx[i], il = s.idx[l];
                bool sw = up ? key_less(kl, il, ki, ii) : key_less(ki, ii, kl, il);
                if (sw) {
                    s.key[i] = kl;
                    s.key[l] = ki;
                    s.idx[i] = il;
                    s.idx[l] = ii;
                }
            }
            __syncthreads();
        }
    }
}

template <int P>
__device__ __forceinline__ void load_row(const double *__restrict__ X, int64_t row, int p, double *xr) {
    const double *src = X + row * (int64_t)p;
#pragma unroll
    for (int k = 0; k < (P ? P : LAGP_PMAX); k++)
        if (P || k < p) xr[k] = __ldg(src + k);
}

template <int P>
__device__ __forceinline__ double row_d2(const double *xr, const double *q, int p) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < (P ? P : LAGP_PMAX); k++) {
        if (P || k < p) {
            double diff = __dsub_rn(q[k], xr[k]);
            acc = __fma_rn(diff, diff, acc);
        }
    }
    return acc;
}

// Exact fallback for one query (index q within the group): radix select of the
// Nprime-th smallest 64-bit key, then an ordered collection that takes every
// key below it plus the lowest-index rows equal to it. Leaves s.key/s.idx
// holding exactly Nprime entries (unsorted).
template <int P>
__device__ void nn_exact_select(NNSmem &s, const double *__restrict__ X, int64_t N, int p, int q,
                                int Nprime) {
    const int tid = threadIdx.x;
    uint64_t prefix = 0;
    int need = Nprime;  // rank (1-based) of the target within the current prefix bucket
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int b = tid; b < 256; b += blockDim.x) s.hist[b] = 0;
        __syncthreads();
        const uint64_t hmask = (shift == 56) ? 0ull : (~0ull << (shift + 8));
        for (int64_t r = tid; r < N; r += blockDim.x) {
            double xr[P ? P : LAGP_PMAX];
            load_row<P>(X, r, p, xr);
            uint64_t k = d2_key(row_d2<P>(xr, s.qx[q], p));
            if ((k & hmask) == prefix) atomicAdd(&s.hist[(k >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid == 0) {
            unsigned acc = 0;
            int b = 0;
            for (; b < 256; b++) {
                if (acc + s.hist[b] >= (unsigned)need) break;
                acc += s.hist[b];
            }
            s.misc[0] = b;
            s.misc[1] = need - (int)acc;
        }
        __syncthreads();
        prefix |= ((uint64_t)s.misc[0]) << shift;
        need = s.misc[1];
        __syncthreads();
    }
    const uint64_t tau = prefix;  // exact key of the Nprime-th smallest
    // ordered collection: keys < tau (count = Nprime - need) and the first
    // `need` rows (by index) with key == tau.
    if (tid == 0) { s.misc[2] = 0; s.misc[3] = 0; }
    __syncthreads();
    const int lane = tid & 31, wid = tid >> 5;
    for (int64_t base = 0; base < N; base += blockDim.x) {
        int64_t r = base + tid;
        uint64_t k = ~0ull;
        if (r < N) {
            double xr[P ? P : LAGP_PMAX];
            load_row<P>(X, r, p, xr);
            k = d2_key(row_d2<P>(xr, s.qx[q], p));
        }
        bool lt = (r < N) && k < tau;
        bool eq = (r < N) && k == tau;
        if (lt) {
            int pos = atomicAdd(&s.misc[2], 1);
            s.key[pos] = k;
            s.idx[pos] = (int)r;
        }
        unsigned bal = __ballot_sync(0xffffffffu, eq);
        if (lane == 0) s.scan[wid] = __popc(bal);
        __syncthreads();
        int before = s.misc[3];
        for (int w = 0; w < wid; w++) before += s.scan[w];
        int rk = before + __popc(bal & ((1u << lane) - 1u));
        if (eq && rk < need) {
            int pos = (Nprime - need) + rk;
            s.key[pos] = k;
            s.idx[pos] = (int)r;
        }
        __syncthreads();
        if (tid == 0) {
            int tot = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); w++) tot += s.scan[w];
            s.misc[3] += tot;
        }
        __syncthreads();
        if (s.misc[3] >= need && s.misc[2] >= Nprime - need) break;  // uniform: both sets complete
    }
    __syncthreads();
}

template <int P>
__global__ void __launch_bounds__(NN_THREADS)
nn_pool_kernel(const double *__restrict__ X, int64_t N, int p, const double *__restrict__ XX, int64_t M,
               int Nprime, int32_t *__restrict__ pool_out, double *__restrict__ d2_out,
               double *__restrict__ samp_ws, uint64_t *__restrict__ bufk_ws, int32_t *__restrict__ bufi_ws,
               int *__restrict__ fallback_count) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    NNSmem &s = *reinterpret_cast<NNSmem *>(smem_raw);
    const int tid = threadIdx.x;
    const int64_t ngroups = (M + NN_Q - 1) / NN_Q;
    const int S = (int)(N < NN_SAMPLE ? N : NN_SAMPLE);
    double *samp = samp_ws + (size_t)blockIdx.x * NN_Q * NN_SAMPLE;
    uint64_t *bufk = bufk_ws + (size_t)blockIdx.x * NN_Q * NN_CAP;
    int32_t *bufi = bufi_ws + (size_t)blockIdx.x * NN_Q * NN_CAP;

    for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        const int64_t q0 = grp * NN_Q;
        const int nq = (int)((M - q0) < NN_Q ? (M - q0) : NN_Q);
        for (int e = tid; e < NN_Q * LAGP_PMAX; e += blockDim.x) {
            int q = e / LAGP_PMAX, k = e % LAGP_PMAX;
            s.qx[q][k] = (q < nq && k < p) ? XX[(q0 + q) * p + k] : 0.0;
        }
        __syncthreads();

        // ---- sample phase: sorted strided sample of d^2 per query
        for (int q = 0; q < nq; q++) {
            int npow = 1;
            while (npow < S) npow <<= 1;
            for (int t = tid; t < npow; t += blockDim.x) {
                if (t < S) {
                    int64_t r = (int64_t)t * N / S;
                    double xr[P ? P : LAGP_PMAX];
                    load_row<P>(X, r, p, xr);
                    s.key[t] = d2_key(row_d2<P>(xr, s.qx[q], p));
                    s.idx[t] = (int)r;
                } else {
                    s.key[t] = ~0ull;
                    s.idx[t] = 0x7fffffff;
                }
            }
            __syncthreads();
            bitonic_sort(s, npow);
            for (int t = tid; t < S; t += blockDim.x) samp[q * NN_SAMPLE + t] = __longlong_as_double((long long)s.key[t]);
            __syncthreads();
            if (tid == 0) {
                // target ~1.5 N' survivors (+ a few sample ranks of slack)
                double want = 1.5 * (double)Nprime * (double)S / (double)N;
                int r = (int)ceil(want) + 12;
                if (Nprime >= N || r >= S) r = S;  // tau = +inf: take every row
                s.rank[q] = r;
                s.state[q] = 0;
            }
            __syncthreads();
        }
        if (tid == 0)
            for (int q = nq; q < NN_Q; q++) s.state[q] = 1;
        __syncthreads();

        // ---- filter rounds
        for (int round = 0; round < NN_MAX_ROUNDS; round++) {
            if (tid < NN_Q && s.state[tid] == 0) {  // only queries still searching
                int q = tid;
                s.cnt[q] = 0;
                int r = s.rank[q];
                s.tau[q] = (r >= S) ? INFINITY : samp[q * NN_SAMPLE + r];
            }
            __syncthreads();
            bool any = false;
            for (int q = 0; q < NN_Q; q++) any |= (s.state[q] == 0);
            if (!any) break;
            for (int64_t r = tid; r < N; r += blockDim.x) {
                double xr[P ? P : LAGP_PMAX];
                load_row<P>(X, r, p, xr);
#pragma unroll
                for (int q = 0; q < NN_Q; q++) {
                    if (s.state[q] != 0) continue;
                    double d2 = row_d2<P>(xr, s.qx[q], p);
                    if (d2 <= s.tau[q]) {
                        int pos = atomicAdd(&s.cnt[q], 1);
                        if (pos < NN_CAP) {
                            bufk[q * NN_CAP + pos] = d2_key(d2);
                            bufi[q * NN_CAP + pos] = (int)r;
                        }
                    }
                }
            }
            __syncthreads();
            if (tid < NN_Q && s.state[tid] == 0) {
                int q = tid;
                int c = s.cnt[q];
                int r = s.rank[q];
                if (c >= Nprime && c <= NN_CAP) {
                    s.state[q] = 1;
                } else if (c < Nprime) {
                    int nr = (int)ceil((double)(r + 1) * 1.5 * (double)Nprime / (double)(c > 0 ? c : 1)) + 16;
                    if (nr <= r) nr = r + 1;
                    if (nr >= S) nr = S;
                    if (r >= S) s.state[q] = 2; else s.rank[q] = nr;
                } else {  // too many survivors
                    int nr = (int)floor((double)r * 0.7 * (double)NN_CAP / (double)c);
                    if (r >= S) nr = (int)floor((double)(S - 1) * 0.7 * (double)NN_CAP / (double)c);
                    if (nr >= r || nr < 0) s.state[q] = 2; else s.rank[q] = nr;
                }
            }
            __syncthreads();
        }
        // queries still active after the rounds fall back as well
        if (tid < NN_Q && s.state[tid] == 0) s.state[tid] = 2;
        __syncthreads();

        // ---- per-query sort and output
        for (int q = 0; q < nq; q++) {
            int c;
            if (s.state[q] == 2) {
                if (tid == 0) atomicAdd(fallback_count, 1);
                nn_exact_select<P>(s, X, N, p, q, Nprime);
                c = Nprime;
            } else {
                c = s.cnt[q];
                for (int t = tid; t < c; t += blockDim.x) {
                    s.key[t] = bufk[q * NN_CAP + t];
                    s.idx[t] = bufi[q * NN_CAP + t];
                }
            }
            int npow = 1;
            while (npow < c) npow <<= 1;
            for (int t = c + tid; t < npow; t += blockDim.x) {
                s.key[t] = ~0ull;
                s.idx[t] = 0x7fffffff;
            }
            __syncthreads();
            bitonic_sort(s, npow);
            int32_t *po = pool_out + (q0 + q) * (int64_t)Nprime;
            for (int t = tid; t < Nprime; t += blockDim.x) {
                po[t] = s.idx[t];
                if (d2_out) d2_out[(q0 + q) * (int64_t)Nprime + t] = __longlong_as_double((long long)s.key[t]);
            }
            __syncthreads();
        }
    }
}

size_t nn_smem_bytes() { return sizeof(NNSmem); }

// Host launcher. Workspace is allocated by the caller (abi.cu) via nn_ws_bytes.
size_t nn_ws_bytes(int grid) {
    return (size_t)grid * NN_Q * (NN_SAMPLE * sizeof(double) + NN_CAP * (sizeof(uint64_t) + sizeof(int32_t))) + 256;
}

template <int P>
static cudaError_t launch_nn_t(const double *X, int64_t N, int p, const double *XX, int64_t M, int Nprime,
                               int32_t *pool, double *d2, void *ws, int grid, int *fb, cudaStream_t st) {
    size_t smem = sizeof(NNSmem);
    cudaError_t e = cudaFuncSetAttribute(nn_pool_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    char *w = (char *)ws;
    double *samp = (double *)w;
    w += (size_t)grid * NN_Q * NN_SAMPLE * sizeof(double);
    uint64_t *bk = (uint64_t *)w;
    w += (size_t)grid * NN_Q * NN_CAP * sizeof(uint64_t);
    int32_t *bi = (int32_t *)w;
    nn_pool_kernel<P><<<grid, NN_THREADS, smem, st>>>(X, N, p, XX, M, Nprime, pool, d2, samp, bk, bi, fb);
    return cudaGetLastError();
}

int nn_grid(int64_t M, int num_sms) {
    int64_t groups = (M + NN_Q - 1) / NN_Q;
    int64_t g = 2LL * num_sms;  // 2 CTAs/SM fit (~110 KB smem each)
    return (int)(groups < g ? (groups > 0 ? groups : 1) : g);
}

cudaError_t launch_nn(const double *X, int64_t N, int p, const double *XX, int64_t M, int Nprime, int32_t *pool,
                      double *d2, void *ws, int grid, int *fb, cudaStream_t st) {
    switch (p) {
        case 1: return launch_nn_t<1>(X, N, p, XX, M, Nprime, pool, d2, ws, grid, fb, st);
        case 2: return launch_nn_t<2>(X, N, p, XX, M, Nprime, pool, d2, ws, grid, fb, st);
        case 3: return launch_nn_t<3>(X, N, p, XX, M, Nprime, pool, d2, ws, grid, fb, st);
        case 4: return launch_nn_t<4>(X, N, p, XX, M, Nprime, pool, d2, ws, grid, fb, st);
        case 8: return launch_nn_t<8>(X, N, p, XX, M, Nprime, pool, d2, ws, grid, fb, st);
        default: return launch_nn_t<0>(X, N, p, XX, M, Nprime, pool, d2, ws, grid, fb, st);
    }
}

}  // namespace lagp
