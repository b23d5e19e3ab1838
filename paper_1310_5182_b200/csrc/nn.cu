// nn.cu — row a1: the N' nearest-neighbour candidate pool of every predictive
// location (PAPER.md P:250-253 NN sub-design; Fig 1 step 2(a) P:365; the N'
// NN candidate restriction P:484-487), exact by the key (d^2, row index) with
// d^2 accumulated by fma in the order k = 0..p-1 (reading R8).
//
// B200 design: a persistent grid of CTAs (two per SM), each handling
// a group of 8 or 16 spatially neighbouring queries at a time. Rows of X are stored
// cell by cell: a two-axis grid for p <= 3, a multi-axis grid (slabs on up to 8
// coordinates) for p >= 4. Per group: a two-level strided sample of X gives each query
// a threshold tau at ~1.15-1.25 N' expected survivors; a paired-FP32 (FFMA2, sm_100)
// prefilter on an FP32 copy of X with a rigorous rounding margin visits only the cells
// that can hold a row with d^2 <= tau (per-query cell lists from rounded-down per-axis
// gap bounds on the multi-axis grid, merged cell-column runs on the two-axis one);
// survivors get the exact FP64 key, which alone decides membership. Selection: one
// value-bin histogram pass locates ranks N' and n0 (radix select as the fallback), or
// a bitonic sort for the sorted pool of laGP_nn_pool. A count outside [N', bufcap]
// re-scales tau; after a few misses the query falls back to an exact 8-bit radix
// select over the 64-bit keys of all rows (robust to massive ties).
#include <cuda_runtime.h>
#include <stdlib.h>

#include <type_traits>

#include "lagp_internal.cuh"
#include "launch.h"

namespace lagp {

constexpr int NN_THREADS = 256;
constexpr int NN_Q = 16;
constexpr int NN_CAP = 8192;
constexpr int NN_MAX_ROUNDS = 6;
// T2 sample rows per N/N' and expected survivors per N' under the sampled threshold.
// Two-axis grid: 128 and 1.25 (measured: 64 -> 128, C2/C4/C3 NN -5/-6/-9 % with that
// filter). Multi-axis grid, whose filter costs less per survivor: 64 and 1.15 (C2 NN
// 1.94 -> 1.85 ms, C4 19.4 -> 18.8 ms per 65,536 queries; 1-2 % of groups take a second
// filter round). Sparse pools (N >= 500 N', e.g. C4) take 32 N/N' rows: there the
// cell-list filter evaluates ~10 % of the rows per query, so the sample is a large share
// of the work (C4 18.6 -> 17.3 ms per 65,536 queries; C2 prefers 64: 1.80 vs 1.84 ms).
#ifndef NN_S2F
#define NN_S2F 128
#endif
#ifndef NN_S2F_MULTI
#define NN_S2F_MULTI 64
#endif
#ifndef NN_S2F_SPARSE
#define NN_S2F_SPARSE 32
#endif
#ifndef NN_TGT
#define NN_TGT 1.25
#endif
#ifndef NN_TGT_MULTI
#define NN_TGT_MULTI 1.15
#endif

#ifdef LAGP_NN_PROF
// phase clocks (profiling builds only): thread 0 of CTA b accumulates cycles per phase:
// 0 group setup + T1, 1 T2, 2 cell list / runs, 3 filter, 4 exact pass, 5 rescale,
// 6 selection + output, 7 groups (count); 8 rounds (count)
__device__ long long g_nn_ph[1024][12];
#define NN_PH(k)                                                                    \
    do {                                                                            \
        if (threadIdx.x == 0 && blockIdx.x < 1024) {                                \
            long long t_;                                                           \
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_)::"memory");            \
            g_nn_ph[blockIdx.x][k] += t_ - ph_t0;                                   \
            ph_t0 = t_;                                                             \
        }                                                                           \
    } while (0)
#define NN_PHC(k)                                                                   \
    do {                                                                            \
        if (threadIdx.x == 0 && blockIdx.x < 1024) g_nn_ph[blockIdx.x][k] += 1;     \
    } while (0)
#define NN_PH0()                                                                    \
    long long ph_t0 = 0;                                                            \
    if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%clock64;" : "=l"(ph_t0)::"memory");
#else
#define NN_PH(k) do {} while (0)
#define NN_PHC(k) do {} while (0)
#define NN_PH0() do {} while (0)
#endif

struct NNSmem {
    uint64_t key[NN_CAP];
    int32_t idx[NN_CAP];
    double qx[NN_Q][LAGP_PMAX];
    float nqf[NN_Q][LAGP_PMAX];  // -(query coords) in FP32 for the sampling distances
    float qf[NN_Q][LAGP_PMAX];   // query coords in FP32 for the dot-form prefilter
    float qn2f[NN_Q];            // ||q~||^2 in FP32
    double tau[NN_Q];
    float thrf[NN_Q];            // FP32 prefilter threshold: tau + rounding margin, rounded up
    float thq[NN_Q];             // thrf - ||q~||^2, rounded up (the FFMA2 filter's test)
    double qn2[NN_Q];            // ||x_q||^2 (for the margin)
    int cnt[NN_Q];
    int rank[NN_Q];
    int state[NN_Q];  // 0 = active, 1 = done, 2 = fallback
    int valid[NN_Q];  // survivors with exact d2 <= tau
    unsigned hist[256];
    unsigned whist[NN_THREADS / 32][256];  // per-warp histograms (sample quantiles)
    unsigned long long redk[NN_THREADS / 32];
    int redi[NN_THREADS / 32];
    int scan[NN_THREADS / 32];
    int misc[4];
    unsigned long long n0k[LAGP_NMAX];  // the n0 nearest (select_pool)
    int n0i[LAGP_NMAX];
    int wcnt[NN_THREADS / 32][NN_Q];    // filter appends per (warp segment, query)
    int fcnt[NN_Q];                     // filter appends per query (multi-axis cell list)
    int ovf[NN_Q];                      // a warp segment overflowed
    int nrng;                           // filter row ranges (in s.hist during the filter)
    int qid[NN_Q];                      // the group's query indices (cell order)
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

// Warp 0 finds the bin of a 256-bin histogram holding the need-th element
// (1-based): misc[0] = bin, misc[1] = rank within the bin, misc[2] = bin count.
__device__ __forceinline__ void warp_pick_bin(const unsigned *hist, int need, int *misc) {
    const int lane = threadIdx.x & 31;
    unsigned loc[8], tot = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) { loc[i] = hist[lane * 8 + i]; tot += loc[i]; }
    unsigned incl = tot;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
    }
    const unsigned excl = incl - tot;
    if (excl < (unsigned)need && incl >= (unsigned)need) {
        unsigned acc = excl;
        for (int i = 0; i < 8; i++) {
            if (acc + loc[i] >= (unsigned)need) {
                misc[0] = lane * 8 + i;
                misc[1] = need - (int)acc;
                misc[2] = (int)loc[i];
                break;
            }
            acc += loc[i];
        }
    }
}

// Exact fallback for one query (index q within the group): radix select of the
// Nprime-th smallest 64-bit key, then an ordered collection that takes every
// key below it plus the lowest-index rows equal to it. Leaves ok/oi (global
// buffers of the query) holding exactly Nprime entries (unsorted).
template <int P>
__device__ void nn_exact_select(NNSmem &s, const double *__restrict__ X, int64_t N, int p, int q, int Nprime,
                                uint64_t *ok, int32_t *oi) {
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
        if (tid < 32) warp_pick_bin(s.hist, need, s.misc);
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
            ok[pos] = k;
            oi[pos] = (int)r;
        }
        unsigned bal = __ballot_sync(0xffffffffu, eq);
        if (lane == 0) s.scan[wid] = __popc(bal);
        __syncthreads();
        int before = s.misc[3];
        for (int w = 0; w < wid; w++) before += s.scan[w];
        int rk = before + __popc(bal & ((1u << lane) - 1u));
        if (eq && rk < need) {
            int pos = (Nprime - need) + rk;
            ok[pos] = k;
            oi[pos] = (int)r;
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

// FP32 copy of X for the prefilter and B = max_i ||X_i||^2 (as ordered uint64 bits).
// order-preserving map of doubles onto uint64 (min/max by integer atomics; deterministic)
__device__ __forceinline__ unsigned long long d_ordkey(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double d_from_ordkey(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

// per-dimension min / max of X (the prefilter's centre c = (min + max) / 2)
__global__ void nn_bounds_kernel(const double *__restrict__ X, int64_t N, int p, unsigned long long *__restrict__ kmin,
                                 unsigned long long *__restrict__ kmax) {
    // one pass over the rows; thread-strided over the flat array so the loads coalesce
    // (element e belongs to dimension e % p; each thread's stride is a multiple of p
    // when blockDim*gridDim % p == 0, else the dimension is recomputed)
    __shared__ unsigned long long slo[LAGP_PMAX], shi[LAGP_PMAX];
    if (threadIdx.x < LAGP_PMAX) {
        slo[threadIdx.x] = ~0ull;
        shi[threadIdx.x] = 0ull;
    }
    __syncthreads();
    const int64_t tot = N * p, stride = (int64_t)gridDim.x * blockDim.x;
    unsigned long long lo[LAGP_PMAX], hi[LAGP_PMAX];
#pragma unroll
    for (int k = 0; k < LAGP_PMAX; k++) {
        lo[k] = ~0ull;
        hi[k] = 0ull;
    }
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += stride) {
        const int k = (int)(e % p);
        const unsigned long long o = d_ordkey(X[e]);
#pragma unroll
        for (int kk = 0; kk < LAGP_PMAX; kk++)
            if (kk == k) {
                lo[kk] = o < lo[kk] ? o : lo[kk];
                hi[kk] = o > hi[kk] ? o : hi[kk];
            }
    }
    for (int k = 0; k < p; k++) {  // warp reduction, then one shared atomic per warp
        unsigned long long l = lo[k], h = hi[k];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const unsigned long long a = __shfl_xor_sync(0xffffffffu, l, off), c = __shfl_xor_sync(0xffffffffu, h, off);
            l = a < l ? a : l;
            h = c > h ? c : h;
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(slo + k, l);
            atomicMax(shi + k, h);
        }
    }
    __syncthreads();
    if (threadIdx.x < p) {
        atomicMin(kmin + threadIdx.x, slo[threadIdx.x]);
        atomicMax(kmax + threadIdx.x, shi[threadIdx.x]);
    }
}

__device__ __forceinline__ double nn_centre(const unsigned long long *kmin, const unsigned long long *kmax, int k) {
    return 0.5 * (d_from_ordkey(kmin[k]) + d_from_ordkey(kmax[k]));
}

// The prefilter works on x~ = x - c (distances are translation invariant): the
// rounding margins scale with ||x~||^2 + ||q~||^2, smallest around the centre.
//
// Spatial cells ("cell pruning"): the bounding box of X is cut into
// gx x gy cells on coordinates 0 and 1 (gy = 1 when p = 1) and the rows of the FP32
// copy are stored cell by cell (row-major cell order; perm maps a stored position back
// to the row of X); the queries of a chunk are ordered the same way, so the 16
// queries of a group are spatial neighbours. Since d^2 >= (x_k - q_k)^2, a row can
// pass the filter only if |x_k - q_k| <= sqrt(thr) on both cell coordinates: the
// filter visits only the cells that meet the group's box (one margin cell on every
// side absorbs the rounding of the cell arithmetic).
__device__ __forceinline__ double nn_lo(const unsigned long long *kmin, int k) { return d_from_ordkey(kmin[k]); }
__device__ __forceinline__ double nn_invw(const unsigned long long *kmin, const unsigned long long *kmax, int k, int G) {
    const double w = d_from_ordkey(kmax[k]) - d_from_ordkey(kmin[k]);
    return (G > 1 && w > 0.0 && w < INFINITY) ? (double)G / w : 0.0;
}
// cell of a coordinate, clamped to [0, G); NaN -> lo (a point) or hi (a box edge)
__device__ __forceinline__ int nn_cell_lo(double v, double lo, double invw, int G) {
    if (invw == 0.0) return 0;
    const double t = (v - lo) * invw;
    if (!(t >= 0.0)) return 0;
    return t >= (double)G ? G - 1 : (int)t;
}
__device__ __forceinline__ int nn_cell_hi(double v, double lo, double invw, int G) {
    if (invw == 0.0) return 0;
    const double t = (v - lo) * invw;
    if (!(t < (double)G)) return G - 1;
    return t < 0.0 ? 0 : (int)t;
}
// The cell grid: s[k] equal-width slabs on coordinate k < nd (mixed-radix cell id,
// coordinate 0 most significant). The two-axis grid (nd <= 2, the filter visits runs
// of cell columns) is s = {gx, gy}; the multi-axis grid (multi = 1, p >= 4) cuts up to
// NN_CELL_DIMS coordinates and the filter visits a per-query list of cells (see the
// filter rounds).
constexpr int NN_CELL_DIMS = 8;
constexpr int NN_CELL_SMAX = 16;    // slabs per coordinate (multi-axis grid)
constexpr int NN_CELL_LIST = 8192;  // cells of the multi-axis grid (the list lives in s.key / s.idx)
struct NNGrid {
    int s[NN_CELL_DIMS];
    int nd;
    int multi;
    int ncell;
};
__device__ __forceinline__ int nn_cell_of(const double *x, int p, const unsigned long long *kmin,
                                          const unsigned long long *kmax, const NNGrid &g) {
    int c = 0;
    for (int k = 0; k < g.nd && k < p; k++) {
        const int G = g.s[k];
        c = c * G + nn_cell_lo(x[k], nn_lo(kmin, k), nn_invw(kmin, kmax, k, G), G);
    }
    return c;
}

// cell histogram of n points (rows of X, or a chunk of query locations)
__global__ void nn_cell_hist_kernel(const double *__restrict__ X, int64_t n, int p, const unsigned long long *__restrict__ kmin,
                                    const unsigned long long *__restrict__ kmax, NNGrid g, int32_t *__restrict__ counts) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(counts + nn_cell_of(X + r * p, p, kmin, kmax, g), 1);
}

// exclusive scan of C <= 16384 cell counts by one block of 1024 threads:
// start[0..C] (start[C] = n) and the scatter cursors cur[c] = start[c]
__global__ void __launch_bounds__(1024) nn_cell_scan_kernel(const int32_t *__restrict__ counts, int C,
                                                            int32_t *__restrict__ start, int32_t *__restrict__ cur) {
    __shared__ int wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int per = (C + 1023) / 1024, c0 = tid * per;
    int loc = 0;
    for (int c = c0; c < c0 + per && c < C; c++) loc += counts[c];
    int x = loc;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int v = wsum[lane];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, v, off);
            if (lane >= off) v += y;
        }
        wsum[lane] = v;
    }
    __syncthreads();
    int run = x - loc + (wid > 0 ? wsum[wid - 1] : 0);
    for (int c = c0; c < c0 + per && c < C; c++) {
        start[c] = run;
        cur[c] = run;
        run += counts[c];
    }
    if (tid == 1023) start[C] = run;
}

// query locations in cell order: qperm[position] = location
__global__ void nn_cell_scatter_kernel(const double *__restrict__ XX, int64_t n, int p, const unsigned long long *__restrict__ kmin,
                                       const unsigned long long *__restrict__ kmax, NNGrid g, int32_t *__restrict__ cur,
                                       int32_t *__restrict__ qperm) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        qperm[atomicAdd(cur + nn_cell_of(XX + r * p, p, kmin, kmax, g), 1)] = (int32_t)r;
}

// FP32 centred copy of X in cell order (perm[position] = row), its FP32 norms, the
// FP64 rows in cell order (the exact keys read them without the perm indirection) and
// B = max ||x~||^2 in FP64 (the margin's bound)
__global__ void nn_prep_kernel(const double *__restrict__ X, int64_t N, int p, float *__restrict__ X32,
                               float *__restrict__ rn2f, unsigned long long *__restrict__ maxn2,
                               const unsigned long long *__restrict__ kmin, const unsigned long long *__restrict__ kmax,
                               NNGrid g, int32_t *__restrict__ cur, int32_t *__restrict__ perm,
                               double *__restrict__ X64c) {
    double mx = 0.0;
    double c[LAGP_PMAX];
    for (int k = 0; k < p; k++) c[k] = nn_centre(kmin, kmax, k);
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < N; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t pos = atomicAdd(cur + nn_cell_of(X + r * p, p, kmin, kmax, g), 1);
        perm[pos] = (int32_t)r;
        double n2 = 0.0;
        float f2 = 0.f;
        for (int k = 0; k < p; k++) {
            X64c[pos * p + k] = X[r * p + k];
            const double v = X[r * p + k] - c[k];
            const float vf = (float)v;
            X32[pos * p + k] = vf;
            f2 = fmaf(vf, vf, f2);
            n2 = fma(v, v, n2);
        }
        rn2f[pos] = f2;
        mx = fmax(mx, n2);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if ((threadIdx.x & 31) == 0) atomicMax(maxn2, (unsigned long long)__double_as_longlong(mx));
}

__device__ __forceinline__ uint32_t f32_to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

// D = A B (m16n8k8, TF32 inputs, FP32 accumulate from 0) — the warp-level tensor path
__device__ __forceinline__ void mma_tf32_16x8x8(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                                uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%10, %10, %10, %10};\n"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(0.f));
}

// FP32 row of the prefilter copy (P compile-time, 0 = generic)
template <int P>
__device__ __forceinline__ void load_row32(const float *__restrict__ X32, int64_t row, int p, float *xf) {
    const float *src = X32 + row * (int64_t)(P ? P : p);
    if (P == 8) {
        const float4 a = __ldg(reinterpret_cast<const float4 *>(src));
        const float4 b = __ldg(reinterpret_cast<const float4 *>(src) + 1);
        xf[0] = a.x; xf[1] = a.y; xf[2] = a.z; xf[3] = a.w;
        xf[4] = b.x; xf[5] = b.y; xf[6] = b.z; xf[7] = b.w;
    } else if (P == 4) {
        const float4 a = __ldg(reinterpret_cast<const float4 *>(src));
        xf[0] = a.x; xf[1] = a.y; xf[2] = a.z; xf[3] = a.w;
    } else if (P == 2) {
        const float2 a = __ldg(reinterpret_cast<const float2 *>(src));
        xf[0] = a.x; xf[1] = a.y;
    } else {
#pragma unroll
        for (int k = 0; k < (P ? P : LAGP_PMAX); k++)
            if (P || k < p) xf[k] = __ldg(src + k);
    }
}

// paired-FP32 prefilter distance: sum_k (x_k - q_k)^2 with FFMA2 (nq = -q)
template <int P>
__device__ __forceinline__ float row_d2f(const float *xf, const float *nq, int p) {
    constexpr int PP = P ? P : LAGP_PMAX;
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k + 1 < PP; k += 2) {
        if (P || k + 1 < p) {
            const float2 d = __fadd2_rn(make_float2(xf[k], xf[k + 1]), make_float2(nq[k], nq[k + 1]));
            acc = __ffma2_rn(d, d, acc);
        } else if (!P && k < p) {
            const float d = xf[k] + nq[k];
            acc.x = fmaf(d, d, acc.x);
        }
    }
    if (PP & 1) {
        const int k = PP - 1;
        if (P || k < p) {
            const float d = xf[k] + nq[k];
            acc.x = fmaf(d, d, acc.x);
        }
    }
    return acc.x + acc.y;
}

// Upper edge of the 16-bit (sign+exponent+7 mantissa bits) bin holding the r-th
// smallest (1-based) of S non-negative floats, by a two-pass warp radix select.
// Used only to pick a threshold; an over-estimate just admits a few more rows.
__device__ float warp_quantile(const float *__restrict__ v, int S, int r, unsigned *hist) {
    const int lane = threadIdx.x & 31;
    if (r > S) return INFINITY;
    unsigned prefix = 0;
    int need = r;
    for (int pass = 0; pass < 2; pass++) {
        const int sh = pass == 0 ? 24 : 16;
        for (int b = lane; b < 256; b += 32) hist[b] = 0;
        __syncwarp();
        for (int t = lane; t < S; t += 32) {
            const unsigned bits = __float_as_uint(v[t]);
            if (pass == 0 || (bits >> 24) == prefix) atomicAdd(&hist[(bits >> sh) & 255u], 1u);
        }
        __syncwarp();
        unsigned loc[8], tot = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) { loc[i] = hist[lane * 8 + i]; tot += loc[i]; }
        unsigned incl = tot;  // inclusive warp scan of per-lane totals
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
        }
        const unsigned excl = incl - tot;
        int bin = -1, below = 0;
        if (excl < (unsigned)need && incl >= (unsigned)need) {
            unsigned acc = excl;
#pragma unroll
            for (int i = 0; i < 8; i++) {
                if (bin < 0 && acc + loc[i] >= (unsigned)need) { bin = lane * 8 + i; below = (int)acc; }
                acc += loc[i];
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, bin >= 0);
        const int src = __ffs(m) - 1;
        bin = __shfl_sync(0xffffffffu, bin, src);
        below = __shfl_sync(0xffffffffu, below, src);
        need -= below;
        prefix = pass == 0 ? (unsigned)bin : ((prefix << 8) | (unsigned)bin);
        __syncwarp();
    }
    return __uint_as_float((prefix << 16) | 0xFFFFu);
}

// (key, idx) composite order
__device__ __forceinline__ bool kv_less(unsigned long long ka, int ia, unsigned long long kb, int ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// Radix select over the live entries of K/I[0..c) (K != ~0): the composite
// (kth, ith) of the rank-th smallest (key, idx) (1-based), so that an entry is
// among the `rank` smallest iff (K, I) <= (kth, ith). The digits start below the
// bits shared by every live key (kmin/kmax), 8 bits at a time, and stop as soon
// as the bucket holding the target is taken whole (then ith = INT_MAX and kth
// has all lower bits set); only a fully tied key goes on to index digits.
// Histogram increments are aggregated per warp (match.any): the leading digits
// of nearby d^2 values collide heavily.
__device__ void radix_select_kv(NNSmem &s, const uint64_t *K, const int32_t *I, int c, int rank, uint64_t kmin,
                                uint64_t kmax, unsigned long long &kth_out, int &ith_out) {
    const int tid = threadIdx.x, lane = tid & 31;
    const uint64_t diff = kmin ^ kmax;
    int sh = diff ? 64 - __clzll((long long)diff) : 0;  // bits [sh, 64) are common to all live keys
    unsigned long long prefix = sh >= 64 ? 0ull : (kmin & (~0ull << sh));
    int need = rank, cnt = c;
    bool whole = false;
    while (sh > 0) {
        const int w = sh >= 8 ? 8 : sh;
        const int lo = sh - w;
        for (int b = tid; b < 256; b += blockDim.x) s.hist[b] = 0;
        __syncthreads();
        const unsigned long long hm = sh >= 64 ? 0ull : (~0ull << sh);
        for (int base = tid - lane; base < c; base += blockDim.x) {
            const int t = base + lane;
            const unsigned long long k = t < c ? K[t] : ~0ull;
            const bool live = k != ~0ull && (k & hm) == prefix;
            const unsigned bin = live ? (unsigned)((k >> lo) & ((1u << w) - 1u)) : 0x100u;
            const unsigned m = __match_any_sync(0xffffffffu, bin);
            if (live && (__ffs(m) - 1) == lane) atomicAdd(&s.hist[bin], (unsigned)__popc(m));
        }
        __syncthreads();
        if (tid < 32) warp_pick_bin(s.hist, need, s.misc);
        __syncthreads();
        prefix |= ((unsigned long long)s.misc[0]) << lo;
        need = s.misc[1];
        cnt = s.misc[2];
        sh = lo;
        __syncthreads();
        if (cnt == need) {  // the whole bucket is in
            whole = true;
            break;
        }
    }
    int ith = 0x7fffffff;
    if (whole) {
        prefix |= sh > 0 ? ((1ull << sh) - 1ull) : 0ull;
    } else if (cnt > need) {  // the target key is tied: select on the index
        unsigned ip = 0;
        for (int ish = 24; ish >= 0; ish -= 8) {
            for (int b = tid; b < 256; b += blockDim.x) s.hist[b] = 0;
            __syncthreads();
            const unsigned hmi = (ish == 24) ? 0u : (~0u << (ish + 8));
            for (int t = tid; t < c; t += blockDim.x)
                if (K[t] == prefix && ((unsigned)I[t] & hmi) == ip) atomicAdd(&s.hist[((unsigned)I[t] >> ish) & 255u], 1u);
            __syncthreads();
            if (tid < 32) warp_pick_bin(s.hist, need, s.misc);
            __syncthreads();
            ip |= ((unsigned)s.misc[0]) << ish;
            need = s.misc[1];
            __syncthreads();
        }
        ith = (int)ip;
    }
    kth_out = prefix;
    ith_out = ith;
}

// Exact selection of the Nprime smallest (key, idx) of the c survivors held in
// K/I[0..c) (entries with K = ~0 are dead): one radix select for rank Nprime
// (membership) and one for rank n0, whose n0 members are ranked by counting and
// written first (pool[0..n0) = X_{n0}(x) in NN order); the rest of the members
// follow in any order (positions >= n0 never affect results: every candidate's
// score and the (Delta, index) argmax are order-independent).
// K/I may be shared or global memory (large pools select in the global buffers).
//
// With dmax (every live key's d2 <= dmax, finite, > 0) the two ranks are found in one
// pass: a histogram over NN_SB value bins bin(d2) = min(NN_SB - 1, floor(d2 NN_SB / dmax))
// (monotone in the key), the bins holding rank Nprime and rank n0 gathered to shared
// memory and ranked there by counting under the (key, index) order. Bins too full for
// the shared lists fall back to the radix selects.
constexpr int NN_SB = 512;     // value bins (in s.whist)
constexpr int NN_SB_L1 = 256;  // gathered entries of the rank-Nprime bin (in s.whist)
__device__ void select_pool(NNSmem &s, uint64_t *K, int32_t *I, int c, int Nprime, int n0,
                            int32_t *__restrict__ po, double dmax) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    unsigned long long kth, k0th;
    int ith, i0th;
#ifndef NN_FASTSEL
#define NN_FASTSEL 1
#endif
    bool fast = NN_FASTSEL && dmax > 0.0 && dmax < INFINITY;  // uniform
    if (fast) {
        unsigned *hb = &s.whist[0][0];
        uint64_t *l1k = reinterpret_cast<uint64_t *>(hb + NN_SB);
        int32_t *l1i = reinterpret_cast<int32_t *>(l1k + NN_SB_L1);
        const double sc = (double)NN_SB / dmax;
        for (int b = tid; b < NN_SB; b += blockDim.x) hb[b] = 0;
        if (tid == 0) { s.misc[2] = 0; s.misc[3] = 0; }
        __syncthreads();
        for (int base = tid - lane; base < c; base += blockDim.x) {  // warp-uniform bound
            const int t = base + lane;
            const unsigned long long k = t < c ? K[t] : ~0ull;
            const bool live = k != ~0ull;
            const unsigned bin = live ? (unsigned)min(NN_SB - 1, (int)(__longlong_as_double((long long)k) * sc)) : 0xffffu;
            const unsigned m = __match_any_sync(0xffffffffu, bin);
            if (live && (__ffs(m) - 1) == lane) atomicAdd(&hb[bin], (unsigned)__popc(m));
        }
        __syncthreads();
        if (wid == 0) {  // bins of rank Nprime and rank n0: scan[0..2] / scan[3..5] = bin, rank in bin, count
            constexpr int PL = NN_SB / 32;
            unsigned loc[PL], tot = 0;
#pragma unroll
            for (int i = 0; i < PL; i++) { loc[i] = hb[lane * PL + i]; tot += loc[i]; }
            unsigned incl = tot;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += y;
            }
            const unsigned excl = incl - tot;
#pragma unroll
            for (int r = 0; r < 2; r++) {
                const unsigned need = r == 0 ? (unsigned)Nprime : (unsigned)n0;
                if (need > 0 && excl < need && incl >= need) {
                    unsigned acc = excl;
                    for (int i = 0; i < PL; i++) {
                        if (acc + loc[i] >= need) {
                            s.scan[3 * r] = lane * PL + i;
                            s.scan[3 * r + 1] = (int)(need - acc);
                            s.scan[3 * r + 2] = (int)loc[i];
                            break;
                        }
                        acc += loc[i];
                    }
                }
            }
            if (lane == 31 && incl < (unsigned)Nprime) s.scan[2] = 1 << 30;  // (never: c >= Nprime live keys)
        }
        __syncthreads();
        const int b1 = s.scan[0], r1 = s.scan[1], c1 = s.scan[2];
        const int b0 = n0 > 0 ? s.scan[3] : -1, r0 = s.scan[4], c0 = n0 > 0 ? s.scan[5] : 0;
        fast = c1 <= NN_SB_L1 && c0 <= LAGP_NMAX;  // uniform
        if (fast) {
            for (int t = tid; t < c; t += blockDim.x) {
                const unsigned long long k = K[t];
                if (k == ~0ull) continue;
                const int bin = min(NN_SB - 1, (int)(__longlong_as_double((long long)k) * sc));
                if (bin == b1) {
                    const int pos = atomicAdd(&s.misc[2], 1);
                    l1k[pos] = k;
                    l1i[pos] = I[t];
                }
                if (bin == b0) {
                    const int pos = atomicAdd(&s.misc[3], 1);
                    s.n0k[pos] = k;
                    s.n0i[pos] = I[t];
                }
            }
            __syncthreads();
            for (int t = tid; t < c1 + c0; t += blockDim.x) {  // rank by counting inside the bin
                const bool one = t < c1;
                const int u = one ? t : t - c1, cn = one ? c1 : c0;
                const uint64_t *bk = one ? l1k : reinterpret_cast<const uint64_t *>(s.n0k);
                const int32_t *bi = one ? l1i : s.n0i;
                const unsigned long long k = bk[u];
                const int i = bi[u];
                int r = 0;
                for (int v = 0; v < cn; v++) r += kv_less(bk[v], bi[v], k, i) ? 1 : 0;
                if (r == (one ? r1 : r0) - 1) {
                    s.redk[one ? 0 : 1] = k;
                    s.redi[one ? 0 : 1] = i;
                }
            }
            __syncthreads();
            kth = s.redk[0];
            ith = s.redi[0];
            if (n0 > 0) {
                k0th = s.redk[1];
                i0th = s.redi[1];
            } else {
                k0th = 0ull;
                i0th = -1;
            }
            __syncthreads();
        }
    }
    if (!fast) {
    // range of the live keys
    unsigned long long kmin = ~0ull, kmax = 0ull;
    for (int t = tid; t < c; t += blockDim.x) {
        const unsigned long long k = K[t];
        if (k != ~0ull) {
            kmin = k < kmin ? k : kmin;
            kmax = k > kmax ? k : kmax;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmin, off);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, kmax, off);
        kmin = a < kmin ? a : kmin;
        kmax = b > kmax ? b : kmax;
    }
    if (lane == 0) { s.redk[wid] = kmin; s.redi[wid] = (int)(kmax >> 32); s.scan[wid] = (int)(unsigned)kmax; }
    __syncthreads();
    kmin = ~0ull;
    kmax = 0ull;
    for (int w = 0; w < nw; w++) {
        const unsigned long long a = s.redk[w];
        const unsigned long long b = ((unsigned long long)(unsigned)s.redi[w] << 32) | (unsigned)s.scan[w];
        kmin = a < kmin ? a : kmin;
        kmax = b > kmax ? b : kmax;
    }
    __syncthreads();
    radix_select_kv(s, K, I, c, Nprime, kmin, kmax, kth, ith);
    if (n0 > 0) {
        radix_select_kv(s, K, I, c, n0, kmin, kmax, k0th, i0th);
    } else {
        k0th = 0ull;
        i0th = -1;  // no entry is <= (0, -1)
    }
    }
    if (tid == 0) { s.misc[2] = 0; s.misc[3] = n0; }
    __syncthreads();
    // the n0 nearest to shared memory (exactly n0: the composite order is total);
    // the other members straight to the pool
    for (int t = tid; t < c; t += blockDim.x) {
        const unsigned long long k = K[t];
        const int i = I[t];
        if (k == ~0ull) continue;
        if (kv_less(k, i, k0th, i0th) || (k == k0th && i == i0th)) {
            const int pos = atomicAdd(&s.misc[2], 1);
            s.n0k[pos] = k;
            s.n0i[pos] = i;
        } else if (kv_less(k, i, kth, ith) || (k == kth && i == ith)) {
            po[atomicAdd(&s.misc[3], 1)] = i;
        }
    }
    __syncthreads();
    for (int a = tid; a < n0; a += blockDim.x) {  // rank by counting
        const unsigned long long k = s.n0k[a];
        const int i = s.n0i[a];
        int r = 0;
        for (int b = 0; b < n0; b++) r += kv_less(s.n0k[b], s.n0i[b], k, i) ? 1 : 0;
        po[r] = i;
    }
    __syncthreads();
}

// paired-FP32 dot product x~ . q~ (FFMA2)
template <int P>
__device__ __forceinline__ float row_dotf(const float *xf, const float *qf, int p) {
    constexpr int PP = P ? P : LAGP_PMAX;
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k + 1 < PP; k += 2) {
        if (P || k + 1 < p) acc = __ffma2_rn(make_float2(xf[k], xf[k + 1]), make_float2(qf[k], qf[k + 1]), acc);
        else if (!P && k < p) acc.x = fmaf(xf[k], qf[k], acc.x);
    }
    if (PP & 1) {
        const int k = PP - 1;
        if (P || k < p) acc.x = fmaf(xf[k], qf[k], acc.x);
    }
    return acc.x + acc.y;
}

// MMA = true (p = 8 only): the filter's dot products on the tensor path in TF32 —
// worth it when survivors are rare (N'/N small, e.g. C4), since every hit costs a
// serial append; the FFMA2 path is faster for denser pools (C2: 3.3 vs 3.9 ms).
template <int P, bool MMA>
__global__ void __launch_bounds__(NN_THREADS, 2)
nn_pool_kernel(const double *__restrict__ X, const float *__restrict__ X32, const float *__restrict__ rn2f,
               const unsigned long long *maxn2_bits, const unsigned long long *__restrict__ kmin,
               const unsigned long long *__restrict__ kmax, int64_t N, int p, const double *__restrict__ XX, int64_t M, int Nprime, int n0, int bufcap,
               int sorted, int32_t *__restrict__ pool_out, double *__restrict__ d2_out, int32_t *__restrict__ bufc_ws,
               uint64_t *__restrict__ bufk_ws, int32_t *__restrict__ bufi_ws, int *__restrict__ fallback_count, NNGrid cg,
               const int32_t *__restrict__ cstart, const int32_t *__restrict__ perm,
               const int32_t *__restrict__ qperm, int qg, const double *__restrict__ X64c,
               unsigned long long *__restrict__ pairc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    NNSmem &s = *reinterpret_cast<NNSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const int gx = cg.s[0], gy = cg.nd > 1 ? cg.s[1] : 1;  // two-axis grid (runs of cell columns)
    const int64_t ngroups = (M + qg - 1) / qg;  // qg = 8 or 16 query locations per group
    // sample sizes and target ranks (see the threshold phase)
    const int S1 = (int)(N < 1024 ? N : 1024);
    const int s2f = !cg.multi ? NN_S2F : (N >= 500 * (int64_t)Nprime ? NN_S2F_SPARSE : NN_S2F_MULTI);
    int64_t s2 = (int64_t)s2f * N / (Nprime > 0 ? Nprime : 1);
    if (s2 < S1) s2 = S1;
    if (s2 > 65536) s2 = 65536;
    if (s2 > N) s2 = N;
    const int S2 = (int)s2;
    const int r2 = (int)ceil((cg.multi ? NN_TGT_MULTI : NN_TGT) * (double)Nprime * (double)S2 / (double)N) + 12;
    int r1 = (int)ceil(4.0 * (double)r2 * (double)S1 / (double)S2) + 4;
    if (Nprime >= N) r1 = S1 + 1;
    // per query: bufi = filter survivors (stored positions, cell order) in NN_THREADS/32 warp segments of segcap rows;
    // bufk/bufc = the exact survivors (key, row), compacted
    uint64_t *bufk = bufk_ws + (size_t)blockIdx.x * NN_Q * bufcap;
    int32_t *bufi = bufi_ws + (size_t)blockIdx.x * NN_Q * bufcap;
    int32_t *bufc = bufc_ws + (size_t)blockIdx.x * NN_Q * bufcap;
    const int segcap = bufcap / nw;
    const double Bn2 = __longlong_as_double((long long)*maxn2_bits);
    const double u32 = 5.9604644775390625e-08;  // 2^-24, FP32 unit roundoff

    // the pool of query q from its c exact survivors K/I (global, or s.key/s.idx):
    // sorted (laGP_nn_pool: bitonic sort in shared memory) or selected (select_pool)
    auto emit = [&](int q, uint64_t *K, int32_t *I, int c) {
        int32_t *po = pool_out + (int64_t)s.qid[q] * Nprime;
        if (sorted) {  // c <= NN_CAP here (bufcap is capped for the sorted output)
            if (K != s.key)
                for (int t = tid; t < c; t += blockDim.x) {
                    s.key[t] = K[t];
                    s.idx[t] = I[t];
                }
            int npow = 1;
            while (npow < c) npow <<= 1;
            for (int t = c + tid; t < npow; t += blockDim.x) {
                s.key[t] = ~0ull;
                s.idx[t] = 0x7fffffff;
            }
            __syncthreads();
            bitonic_sort(s, npow);
            for (int t = tid; t < Nprime; t += blockDim.x) {
                po[t] = s.idx[t];
                if (d2_out) d2_out[(int64_t)s.qid[q] * Nprime + t] = __longlong_as_double((long long)s.key[t]);
            }
            __syncthreads();
        } else {
            select_pool(s, K, I, c, Nprime, n0, po, s.state[q] == 2 ? -1.0 : s.tau[q]);
        }
    };

    // multi-axis grid: the list of cells (stored-row range [lst_a, lst_b), mask lst_m of the
    // queries in actm it can hold a row with d^2 <= thrf for) in s.key / s.idx (free
    // between the threshold samples and the exact pass); count in s.nrng
    int *lst_a = reinterpret_cast<int *>(s.key), *lst_b = lst_a + NN_CELL_LIST;
    unsigned *lst_m = reinterpret_cast<unsigned *>(s.idx);
    auto build_list = [&](unsigned act) {
        // A row of cell c has |x_k - q_k| >= gap_k(c, q) on every cut coordinate, so
        // d^2(x, q) >= lb(c, q) = sum_k gap_k^2; a cell is listed for query q unless
        // lb > thr (>= tau). Per-coordinate terms gap_k^2 are tabulated per query and
        // slab (rounded down; the slab box is widened by a margin that covers the
        // rounding of the cell arithmetic) and summed with round-down adds, so the
        // computed lb never exceeds the exact one: no row with d^2 <= tau is pruned.
        float *dlb = reinterpret_cast<float *>(&s.whist[0][0]);  // [NN_Q][NN_CELL_DIMS][NN_CELL_SMAX]
        for (int e = tid; e < NN_Q * NN_CELL_DIMS * NN_CELL_SMAX; e += blockDim.x) {
            const int q = e / (NN_CELL_DIMS * NN_CELL_SMAX), k = (e / NN_CELL_SMAX) % NN_CELL_DIMS,
                      i = e % NN_CELL_SMAX;
            float v = 0.f;
            if (k < cg.nd && i < cg.s[k] && ((act >> q) & 1u)) {
                const int G = cg.s[k];
                const double lo = nn_lo(kmin, k), iw = nn_invw(kmin, kmax, k, G);
                if (iw > 0.0) {
                    const double rw = 1.0 / iw;
                    const double mg = 1e-6 * rw + 1e-14 * (fabs(lo) + (double)G * rw);
                    const double blo = i == 0 ? -INFINITY : lo + (double)i * rw - mg;
                    const double bhi = i == G - 1 ? INFINITY : lo + (double)(i + 1) * rw + mg;
                    const double qk = s.qx[q][k];
                    const double gp = fmax(0.0, fmax(blo - qk, qk - bhi)) * (1.0 - 0x1p-40);
                    v = __double2float_rd(gp * gp);
                }
            }
            dlb[e] = v;
        }
        if (tid == 0) s.nrng = 0;
        __syncthreads();
        const int C = cg.ncell, per = (C + (int)blockDim.x - 1) / (int)blockDim.x;
        const int c0 = tid * per, c1 = min(c0 + per, C);
        int dg[NN_CELL_DIMS];  // mixed-radix digits of cell c (odometer)
        {
            int c = c0;
#pragma unroll
            for (int k = NN_CELL_DIMS - 1; k >= 0; k--) {
                dg[k] = 0;
                if (k < cg.nd) {
                    dg[k] = c % cg.s[k];
                    c /= cg.s[k];
                }
            }
        }
        for (int c = c0; c < c1; c++) {
            unsigned m = 0, aq = act;
            while (aq) {
                const int q = __ffs(aq) - 1;
                aq &= aq - 1;
                const float *dq = dlb + q * NN_CELL_DIMS * NN_CELL_SMAX;
                float lb = 0.f;
#pragma unroll
                for (int k = 0; k < NN_CELL_DIMS; k++)
                    if (k < cg.nd) lb = __fadd_rd(lb, dq[k * NN_CELL_SMAX + dg[k]]);
                if (!(lb > s.thrf[q])) m |= 1u << q;
            }
            if (m) {
                const int a = cstart[c], b = cstart[c + 1];
                if (b > a) {
                    const int e = atomicAdd(&s.nrng, 1);
                    lst_a[e] = a;
                    lst_b[e] = b;
                    lst_m[e] = m;
                }
            }
            bool carry = true;  // next cell: increment the odometer
#pragma unroll
            for (int k = NN_CELL_DIMS - 1; k >= 0; k--)
                if (carry && k < cg.nd) {
                    dg[k]++;
                    carry = dg[k] >= cg.s[k];
                    if (carry) dg[k] = 0;
                }
        }
        __syncthreads();
    };

    for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        NN_PH0();
        NN_PHC(7);
        const int64_t q0 = grp * qg;
        const int nq = (int)((M - q0) < qg ? (M - q0) : qg);
        if (tid < NN_Q) s.qid[tid] = tid < nq ? (qperm ? qperm[q0 + tid] : (int32_t)(q0 + tid)) : 0;
        __syncthreads();
        for (int e = tid; e < NN_Q * LAGP_PMAX; e += blockDim.x) {
            int q = e / LAGP_PMAX, k = e % LAGP_PMAX;
            const double v = (q < nq && k < p) ? XX[(int64_t)s.qid[q] * p + k] : 0.0;
            const double vc = (q < nq && k < p) ? v - nn_centre(kmin, kmax, k) : 0.0;  // centred (prefilter)
            s.qx[q][k] = v;  // raw (exact keys)
            s.nqf[q][k] = -(float)vc;
            s.qf[q][k] = (float)vc;
        }
        __syncthreads();
        if (tid < NN_Q) {
            double n2 = 0.0;
            for (int k = 0; k < p; k++) {
                const double vc = s.qx[tid][k] - nn_centre(kmin, kmax, k);
                n2 = fma(vc, vc, n2);
            }
            s.qn2[tid] = n2;
            float f2 = 0.f;
            for (int k = 0; k < p; k++) f2 = fmaf(s.qf[tid][k], s.qf[tid][k], f2);
            s.qn2f[tid] = f2;
        }
        // ---- threshold phase, two-level sampling (all 16 queries per row load).
        // T1: S1 <= 1024 strided rows; tau1 at a generous rank (about 4x the final
        //     target, so it bounds the T2 order statistic with margin).
        // T2: S2 = min(N, 64 N / N') strided rows; the T2 distances below tau1 are
        //     listed (~4 r2 per query) and tau = their r2-th smallest, where r2 puts
        //     ~NN_TGT N' expected survivors under tau (relative spread ~1/sqrt(r2) ~ 6 %).
        {
            float *t1 = reinterpret_cast<float *>(s.key);  // NN_Q x 1024 floats (64 KB)
            const double step1 = (double)N / (double)S1;
            for (int t = tid; t < S1; t += blockDim.x) {  // each sample row loaded once for all queries
                int64_t r = (int64_t)((double)t * step1);
                float xf[P ? P : LAGP_PMAX];
                load_row32<P>(X32, r < N ? r : N - 1, p, xf);
#pragma unroll 1
                for (int q = 0; q < nq; q++) t1[q * 1024 + t] = row_d2f<P>(xf, s.nqf[q], p);
            }
            __syncthreads();
            for (int q = wid; q < NN_Q; q += nw) {
                const float tq = (q >= nq || r1 > S1) ? INFINITY : warp_quantile(t1 + q * 1024, S1, r1, s.whist[wid]);
                if (lane == 0) {
                    s.tau[q] = (double)tq;
                    s.state[q] = q < nq ? 0 : 1;
                    s.cnt[q] = 0;
                }
            }
            __syncthreads();
            NN_PH(0);
            if (S2 > S1 && r2 <= S2) {
                float *lst = reinterpret_cast<float *>(bufk);  // per query bufcap floats
                const double step2 = (double)N / (double)S2;
                // 4 sample rows per thread per pass, each query's coordinates read from
                // shared memory once per 4 rows (as in the filter pass); the T2 distances
                // <= tau1 are listed
                auto t2_eval = [&](const float (&xf)[4][P ? P : LAGP_PMAX], const bool (&ok)[4], unsigned qm) {
                    while (qm) {
                        const int q = __ffs(qm) - 1;
                        qm &= qm - 1;
                        float qv[P ? P : LAGP_PMAX];
#pragma unroll
                        for (int k = 0; k < (P ? P : LAGP_PMAX); k++) qv[k] = s.nqf[q][k];
                        const float tq = (float)s.tau[q];
                        float d2f[4];
                        unsigned m[4];
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            d2f[u] = row_d2f<P>(xf[u], qv, p);
                            m[u] = __ballot_sync(0xffffffffu, ok[u] && d2f[u] <= tq);
                        }
                        if (m[0] | m[1] | m[2] | m[3]) {  // one shared atomic per warp and query
                            int pos = 0;
                            if (lane == 0) pos = atomicAdd(&s.cnt[q], __popc(m[0]) + __popc(m[1]) + __popc(m[2]) + __popc(m[3]));
                            pos = __shfl_sync(0xffffffffu, pos, 0);
                            const unsigned lt = (1u << lane) - 1u;
#pragma unroll
                            for (int u = 0; u < 4; u++) {
                                const int pu = pos + __popc(m[u] & lt);
                                if (((m[u] >> lane) & 1u) && pu < bufcap) lst[(size_t)q * bufcap + pu] = d2f[u];
                                pos += __popc(m[u]);
                            }
                        }
                    }
                };
                const unsigned allq = nq < 32 ? (1u << nq) - 1u : ~0u;
                if (pairc && tid == 0) atomicAdd(pairc + 1, (unsigned long long)S2 * (unsigned)nq);
                for (int64_t wb = (int64_t)wid * 128; wb < S2; wb += (int64_t)nw * 128) {
                    float xf[4][P ? P : LAGP_PMAX];
                    bool ok[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const int64_t t = wb + 32 * u + lane;
                        ok[u] = t < S2;
                        if (ok[u]) {
                            int64_t r = (int64_t)((double)t * step2);  // strided sample row (no 64-bit division)
                            load_row32<P>(X32, r < N ? r : N - 1, p, xf[u]);
                        } else {
#pragma unroll
                            for (int k = 0; k < (P ? P : LAGP_PMAX); k++) xf[u][k] = 0.f;
                        }
                    }
                    t2_eval(xf, ok, allq);
                }
                __syncthreads();
                for (int q = wid; q < NN_Q; q += nw) {
                    const int c2 = s.cnt[q];
                    if (c2 >= r2 && c2 <= bufcap) {  // else keep tau1; the filter rounds adapt it
                        const float tq = warp_quantile(lst + (size_t)q * bufcap, c2, r2, s.whist[wid]);
                        if (lane == 0) s.tau[q] = (double)tq;
                    }
                }
                __syncthreads();
            } else if (r2 > S2) {
                if (tid < NN_Q) s.tau[tid] = INFINITY;  // N' close to N: every row
                __syncthreads();
            } else {  // S2 == S1: T1 already has the target resolution
                for (int q = wid; q < nq; q += nw) {
                    const float tq = warp_quantile(t1 + q * 1024, S1, r2 <= S1 ? r2 : S1, s.whist[wid]);
                    if (lane == 0) s.tau[q] = (double)tq;
                }
                __syncthreads();
            }
        }

        NN_PH(1);
        // ---- filter rounds
        for (int round = 0; round < NN_MAX_ROUNDS; round++) {
            for (int e = tid; e < nw * NN_Q; e += blockDim.x) (&s.wcnt[0][0])[e] = 0;
            if (tid < NN_Q) {
                s.ovf[tid] = 0;
                s.fcnt[tid] = 0;
            }
            if (tid < NN_Q && s.state[tid] == 0) {  // only queries still searching
                const int q = tid;
                s.cnt[q] = 0;
                const double tau = s.tau[q];
                // FP32 prefilter threshold for the dot form d2 ~ ||x~||^2 + ||q~||^2 - 2 x~.q~
                // (x~, q~ the FP32-rounded inputs, u = 2^-24): rounding the inputs moves d2 by
                // <= 4u(||x||^2 + ||q||^2) and the FP32 evaluation by <= 2(p+3)u(||x||^2 + ||q||^2)
                // (first order), i.e. <= (2p+10)u(||x||^2 + ||q||^2); the margin doubles it, so
                // every row with exact d2 <= tau passes and the FP64 key alone decides.
                // MMA: TF32 inputs (10-bit mantissas) and FP32 accumulation bound the dot-form
                // error by (2^-10 + p 2^-20 + (2p+10) 2^-24)(||x~||^2 + ||q~||^2), doubled
                const double thr = MMA
                    ? tau + 2.0 * (9.765625e-04 + p * 9.5367431640625e-07 + (2.0 * p + 10.0) * u32) * (s.qn2[q] + Bn2)
                    : tau + (4.0 * p + 20.0) * u32 * (s.qn2[q] + Bn2);
                s.thrf[q] = isfinite(thr) ? __double2float_ru(thr) : INFINITY;
            }
            if (tid < NN_Q && s.state[tid] != 0) s.thrf[tid] = __int_as_float(0x7fc00000);  // NaN: inactive
            if (tid < NN_Q) s.thq[tid] = __fsub_ru(s.thrf[tid], s.qn2f[tid]);
            __syncthreads();
            unsigned act = 0;
            for (int q = 0; q < NN_Q; q++) act |= (s.state[q] == 0 ? 1u : 0u) << q;
            if (!act) break;
            // the cells that meet the active queries' box |x_k - q_k| <= sqrt(thr), k = 0, 1,
            // as maximal runs of stored rows (cell order is row-major: one run per cell column)
            int *rng_a = reinterpret_cast<int *>(s.hist), *rng_b = rng_a + 128;
            if (cg.multi) build_list(act);
            if (!cg.multi && wid == 0) {
                double lo0 = INFINITY, hi0 = -INFINITY, lo1 = INFINITY, hi1 = -INFINITY;
                if (lane < NN_Q && s.state[lane] == 0) {
                    const double r = sqrt((double)s.thrf[lane]);
                    lo0 = s.qx[lane][0] - r;
                    hi0 = s.qx[lane][0] + r;
                    if (p > 1) {
                        lo1 = s.qx[lane][1] - r;
                        hi1 = s.qx[lane][1] + r;
                    }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {  // fmin/fmax drop a NaN operand: NaN r -> whole axis below
                    lo0 = fmin(lo0, __shfl_xor_sync(0xffffffffu, lo0, off));
                    hi0 = fmax(hi0, __shfl_xor_sync(0xffffffffu, hi0, off));
                    lo1 = fmin(lo1, __shfl_xor_sync(0xffffffffu, lo1, off));
                    hi1 = fmax(hi1, __shfl_xor_sync(0xffffffffu, hi1, off));
                }
                bool anynan = false;
                if (lane < NN_Q && s.state[lane] == 0) anynan = isnan(s.thrf[lane]) || isnan(s.qx[lane][0]) || (p > 1 && isnan(s.qx[lane][1]));
                anynan = __any_sync(0xffffffffu, anynan);
                int cx0 = 0, cx1 = gx - 1, cy0 = 0, cy1 = gy - 1;
                if (!anynan) {
                    const double l0 = nn_lo(kmin, 0), iw0 = nn_invw(kmin, kmax, 0, gx);
                    cx0 = max(nn_cell_lo(lo0, l0, iw0, gx) - 1, 0);
                    cx1 = min(nn_cell_hi(hi0, l0, iw0, gx) + 1, gx - 1);
                    if (gy > 1) {
                        const double l1 = nn_lo(kmin, 1), iw1 = nn_invw(kmin, kmax, 1, gy);
                        cy0 = max(nn_cell_lo(lo1, l1, iw1, gy) - 1, 0);
                        cy1 = min(nn_cell_hi(hi1, l1, iw1, gy) + 1, gy - 1);
                    }
                }
                if (gy == 1) {  // one run
                    if (lane == 0) {
                        rng_a[0] = cstart[cx0];
                        rng_b[0] = cstart[cx1 + 1];
                        s.nrng = 1;
                    }
                } else {  // gx <= 128 columns: load the runs in parallel, merge adjacent ones
                    for (int cx = cx0 + lane; cx <= cx1; cx += 32) {
                        rng_a[cx - cx0] = cstart[cx * gy + cy0];
                        rng_b[cx - cx0] = cstart[cx * gy + cy1 + 1];
                    }
                    __syncwarp();
                    if (lane == 0) {
                        int nr = 0;
                        for (int i = 0; i <= cx1 - cx0; i++) {
                            const int a = rng_a[i], b = rng_b[i];
                            if (b <= a) continue;
                            if (nr > 0 && rng_b[nr - 1] == a) {
                                rng_b[nr - 1] = b;
                            } else {
                                rng_a[nr] = a;
                                rng_b[nr] = b;
                                nr++;
                            }
                        }
                        s.nrng = nr;
                    }
                }
            }
            __syncthreads();
            NN_PH(2);
            NN_PHC(8);
            const int nrng = s.nrng;
            // 4 rows per thread per iteration: each query's coordinates are loaded
            // from shared memory once per 4 rows
            // (the loop bound is warp-uniform: the ballots below need whole warps)
            // per-warp append counters in registers: lane q holds this warp's count for query q
            int wcr = 0;
            if (cg.multi) {
                // The listed cells, one warp per cell, in passes of 128 rows (4 per lane)
                // and a 64- or 32-row pass for the cell's tail; only the cell's listed
                // queries are evaluated; appends through a shared per-query counter (one
                // atomic per warp, query and pass with a hit).
                const unsigned lt = (1u << lane) - 1u;
                constexpr int PP = P ? P : LAGP_PMAX;
                unsigned long long npair = 0;  // lane 0: (row, query) pairs this warp evaluated
                auto pass = [&](auto uc, int base, int b, unsigned m) {
                    constexpr int U = decltype(uc)::value;
                    npair += (unsigned long long)min(32 * U, b - base) * (unsigned)__popc(m);
                    float xf[U][PP], rn[U];
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int r = base + 32 * u + lane;
                        if (r < b) {
                            load_row32<P>(X32, r, p, xf[u]);
                            rn[u] = __ldg(rn2f + r);
                        } else {
#pragma unroll
                            for (int k = 0; k < PP; k++) xf[u][k] = 0.f;
                            rn[u] = __int_as_float(0x7fc00000);  // NaN: never <= thr
                        }
                    }
                    // two listed queries per iteration (independent dot chains)
                    auto append = [&](int q, const bool (&hit)[U], const unsigned (&mm)[U], unsigned tot) {
                        if (tot) {
                            int pos = 0;
                            if (lane == 0) pos = atomicAdd(&s.fcnt[q], (int)tot);
                            pos = __shfl_sync(0xffffffffu, pos, 0);
                            int32_t *qb = bufi + q * bufcap;
#pragma unroll
                            for (int u = 0; u < U; u++) {
                                const int pu = pos + __popc(mm[u] & lt);
                                if (hit[u] && pu < bufcap) qb[pu] = base + 32 * u + lane;
                                pos += __popc(mm[u]);
                            }
                        }
                    };
                    while (m) {
                        const int q = __ffs(m) - 1;
                        m &= m - 1;
                        const int q2 = m ? __ffs(m) - 1 : q;  // (uniform)
                        const bool two = m != 0;
                        if (two) m &= m - 1;
                        float qv[PP], qv2[PP];
#pragma unroll
                        for (int k = 0; k < PP; k++) {
                            qv[k] = s.qf[q][k];
                            qv2[k] = s.qf[q2][k];
                        }
                        const float thq = s.thq[q], thq2 = s.thq[q2];
                        bool hit[U], hit2[U];
                        unsigned mm[U], mm2[U], tot = 0, tot2 = 0;
#pragma unroll
                        for (int u = 0; u < U; u++) {
                            hit[u] = fmaf(-2.f, row_dotf<P>(xf[u], qv, p), rn[u]) <= thq;
                            hit2[u] = two && fmaf(-2.f, row_dotf<P>(xf[u], qv2, p), rn[u]) <= thq2;
                        }
#pragma unroll
                        for (int u = 0; u < U; u++) {
                            mm[u] = __ballot_sync(0xffffffffu, hit[u]);
                            mm2[u] = __ballot_sync(0xffffffffu, hit2[u]);
                            tot += __popc(mm[u]);
                            tot2 += __popc(mm2[u]);
                        }
                        append(q, hit, mm, tot);
                        append(q2, hit2, mm2, tot2);
                    }
                };
                for (int e = wid; e < nrng; e += nw) {  // warp-uniform
                    const int b = lst_b[e];
                    const unsigned m = lst_m[e];
                    int base = lst_a[e];
                    for (; b - base > 96; base += 128) pass(std::integral_constant<int, 4>{}, base, b, m);
                    if (b - base > 32) {
                        pass(std::integral_constant<int, 2>{}, base, b, m);
                        base += 64;
                    }
                    if (b - base > 0) pass(std::integral_constant<int, 1>{}, base, b, m);
                }
                if (pairc && lane == 0 && npair) atomicAdd(pairc, npair);
            } else if constexpr (MMA && P == 8) {
                // Tensor-core filter (mma.sync m16n8k8 TF32): a warp takes 16 rows x 8
                // queries per MMA, D = X~[16x8] Q~^T[8x8]; MMA coordinate k is x~ coordinate
                // perm(k), perm(t) = 2t, perm(t + 4) = 2t + 1, so each thread's A elements
                // are one float2 of its row. Lane (g = lane/4, t = lane%4) holds
                // d[0..3] = dot(rows g, g+8; queries 2t, 2t+1).
                const int g = lane >> 2, t = lane & 3;
                uint32_t bq[2][2];
                float qn_l[2][2], thr_l[2][2];
#pragma unroll
                for (int gr = 0; gr < 2; gr++) {
                    bq[gr][0] = f32_to_tf32(s.qf[8 * gr + g][2 * t]);
                    bq[gr][1] = f32_to_tf32(s.qf[8 * gr + g][2 * t + 1]);
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        qn_l[gr][h] = s.qn2f[8 * gr + 2 * t + h];
                        thr_l[gr][h] = s.thrf[8 * gr + 2 * t + h];  // NaN for inactive queries
                    }
                }
                // 4 tiles (64 rows) per warp iteration: all loads issued before any MMA
                constexpr int NT = 4;
                for (int ri = 0; ri < nrng; ri++) {
                const int64_t ra = rng_a[ri], rend = rng_b[ri];
                for (int64_t rb = ra + (int64_t)wid * 16 * NT; rb < rend; rb += (int64_t)nw * 16 * NT) {
                    if (pairc && lane == 0)
                        atomicAdd(pairc, (unsigned long long)(rend - rb < 16 * NT ? rend - rb : 16 * NT) * (unsigned)__popc(act));
                    float2 xa[NT], xb[NT];
                    float rnA[NT], rnB[NT];
#pragma unroll
                    for (int u = 0; u < NT; u++) {
                        const int64_t rA = rb + 16 * u + g, rB = rA + 8;
                        xa[u] = make_float2(0.f, 0.f);
                        xb[u] = make_float2(0.f, 0.f);
                        rnA[u] = __int_as_float(0x7fc00000);
                        rnB[u] = __int_as_float(0x7fc00000);
                        if (rA < rend) {
                            xa[u] = __ldg(reinterpret_cast<const float2 *>(X32 + rA * 8) + t);
                            rnA[u] = __ldg(rn2f + rA);
                        }
                        if (rB < rend) {
                            xb[u] = __ldg(reinterpret_cast<const float2 *>(X32 + rB * 8) + t);
                            rnB[u] = __ldg(rn2f + rB);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < NT; u++) {
                        const int64_t r0 = rb + 16 * u;
                        const uint32_t a0 = f32_to_tf32(xa[u].x), a1 = f32_to_tf32(xb[u].x), a2 = f32_to_tf32(xa[u].y),
                                       a3 = f32_to_tf32(xb[u].y);
#pragma unroll
                        for (int gr = 0; gr < 2; gr++) {
                            float d[4];
                            mma_tf32_16x8x8(d, a0, a1, a2, a3, bq[gr][0], bq[gr][1]);
                            bool h[4];
                            h[0] = fmaf(-2.f, d[0], rnA[u] + qn_l[gr][0]) <= thr_l[gr][0];
                            h[1] = fmaf(-2.f, d[1], rnA[u] + qn_l[gr][1]) <= thr_l[gr][1];
                            h[2] = fmaf(-2.f, d[2], rnB[u] + qn_l[gr][0]) <= thr_l[gr][0];
                            h[3] = fmaf(-2.f, d[3], rnB[u] + qn_l[gr][1]) <= thr_l[gr][1];
                            if (__any_sync(0xffffffffu, h[0] | h[1] | h[2] | h[3])) {
                                // rare: walk the hits in a fixed order (deterministic segments)
#pragma unroll
                                for (int v = 0; v < 4; v++) {
                                    unsigned m = __ballot_sync(0xffffffffu, h[v]);
                                    while (m) {
                                        const int l = __ffs(m) - 1;
                                        m &= m - 1;
                                        const int q = 8 * gr + 2 * (l & 3) + (v & 1);
                                        const int64_t row = r0 + (l >> 2) + 8 * (v >> 1);
                                        const int pos = __shfl_sync(0xffffffffu, wcr, q);
                                        if (lane == 0 && pos < segcap) bufi[q * bufcap + wid * segcap + pos] = (int)row;
                                        if (lane == q) wcr++;
                                    }
                                }
                            }
                        }
                    }
                }
                }
            } else {
                for (int ri = 0; ri < nrng; ri++) {
                const int64_t ra = rng_a[ri], rend = rng_b[ri];
                for (int64_t wbase = ra + tid - lane; wbase < rend; wbase += 4 * (int64_t)blockDim.x) {
                    const int64_t base = wbase + lane;
                    if (pairc && lane == 0) {
                        long long rows = 0;
                        for (int u = 0; u < 4; u++) {
                            const long long r0 = wbase + u * (int64_t)blockDim.x;
                            rows += r0 >= rend ? 0 : (rend - r0 < 32 ? rend - r0 : 32);
                        }
                        if (rows) atomicAdd(pairc, (unsigned long long)rows * (unsigned)__popc(act));
                    }
                    float xf[4][P ? P : LAGP_PMAX];
                    float rn[4];
    #pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const int64_t r = base + u * (int64_t)blockDim.x;
                        if (r < rend) {
                            load_row32<P>(X32, r, p, xf[u]);
                            rn[u] = __ldg(rn2f + r);
                        } else {
    #pragma unroll
                            for (int k = 0; k < (P ? P : LAGP_PMAX); k++) xf[u][k] = 0.f;
                            rn[u] = __int_as_float(0x7fc00000);  // NaN: never <= thr, even thr = +inf
                        }
                    }
    #pragma unroll 1
                    for (int q = 0; q < nq; q++) {  // inactive queries have thr = NaN: no candidates
                        float qv[P ? P : LAGP_PMAX];
    #pragma unroll
                        for (int k = 0; k < (P ? P : LAGP_PMAX); k++) qv[k] = s.qf[q][k];
                        // ||x~||^2 - 2 x~.q~ <= thr - ||q~||^2 (rounded up): one rounding fewer than
                        // evaluating ||q~||^2 + ||x~||^2 first, inside the margin's factor 2
                        const float thq = s.thq[q];
                        bool hit[4];
                        unsigned mm[4];
    #pragma unroll
                        for (int u = 0; u < 4; u++) {
                            hit[u] = fmaf(-2.f, row_dotf<P>(xf[u], qv, p), rn[u]) <= thq;
                            mm[u] = __ballot_sync(0xffffffffu, hit[u]);
                        }
                        // append to this warp's own segment of the query's buffer: the warp
                        // owns its counter, so positions come from ballots alone (no atomics);
                        // only the 4-row groups with a hit do any work
                        if (mm[0] | mm[1] | mm[2] | mm[3]) {
                            int wc = __shfl_sync(0xffffffffu, wcr, q);
                            const unsigned lt = (1u << lane) - 1u;
                            int32_t *seg = bufi + q * bufcap + wid * segcap;
    #pragma unroll
                            for (int u = 0; u < 4; u++) {
                                if (mm[u]) {
                                    const int pos = wc + __popc(mm[u] & lt);
                                    if (hit[u] && pos < segcap) seg[pos] = (int)(base + u * (int64_t)blockDim.x);
                                    wc += __popc(mm[u]);
                                }
                            }
                            if (lane == q) wcr = wc;
                        }
                    }
                }
                }
            }
            if (cg.multi) {  // one segment (warp 0's) of up to bufcap rows per query
                __syncthreads();
                if (tid < NN_Q) {
                    s.wcnt[0][tid] = s.fcnt[tid];
                    if (s.fcnt[tid] > bufcap) s.ovf[tid] = 1;
                }
            } else if (lane < NN_Q) {
                s.wcnt[wid][lane] = wcr;
                if (wcr > segcap) s.ovf[lane] = 1;
            }
            __syncthreads();
            NN_PH(3);
            // dense exact pass over the prefilter survivors (the warp segments read as
            // one range): FP64 key, keep d2 <= tau, compacted into shared memory (s.key /
            // s.idx) when the prefilter count fits, else into bufk/bufc; a query whose count
            // lands in [N', bufcap] is selected and written at once (state 3)
            for (int q = 0; q < NN_Q; q++) {
                if (!((act >> q) & 1u)) continue;
                if (s.ovf[q]) {  // too many survivors: rescale below
                    __syncthreads();
                    if (tid == 0) { s.cnt[q] = bufcap + 1; s.valid[q] = 0; }
                    __syncthreads();
                    continue;
                }
                int tot = 0;
                for (int w = 0; w < nw; w++) tot += s.wcnt[w][q];
                const bool in_smem = tot <= NN_CAP;  // uniform
                if (pairc && tid == 0) atomicAdd(pairc + 2, (unsigned long long)tot);
                uint64_t *ok_k = in_smem ? s.key : bufk + (size_t)q * bufcap;
                int32_t *ok_i = in_smem ? s.idx : bufc + (size_t)q * bufcap;
                if (tid == 0) s.misc[3] = 0;
                __syncthreads();
                // the stored position of the thread's next survivor is loaded one iteration
                // ahead (its L2 round trip overlaps this iteration's row loads and key)
                auto surv_sp = [&](int t) -> int {
                    if (t >= tot) return -1;
                    int w = 0, off = t;
                    while (off >= s.wcnt[w][q]) { off -= s.wcnt[w][q]; w++; }
                    return bufi[q * bufcap + w * segcap + off];  // stored position
                };
                int sp_next = surv_sp(tid);
                for (int tb = tid - lane; tb < tot; tb += blockDim.x) {  // warp-uniform bound
                    const int t = tb + lane;
                    const int sp = sp_next;
                    sp_next = surv_sp(t + blockDim.x);
                    bool ok = false;
                    int r = 0;
                    double d2 = 0.0;
                    if (t < tot) {
                        r = __ldg(perm + sp);                                // -> row of X
                        double xr[P ? P : LAGP_PMAX];
                        load_row<P>(X64c, sp, p, xr);  // = row r of X
                        d2 = row_d2<P>(xr, s.qx[q], p);
                        ok = d2 <= s.tau[q];
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, ok);
                    if (m) {
                        int pos = 0;
                        if (lane == 0) pos = atomicAdd(&s.misc[3], __popc(m));
                        pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(m & ((1u << lane) - 1u));
                        if (ok) {
                            ok_k[pos] = d2_key(d2);
                            ok_i[pos] = r;
                        }
                    }
                }
                __syncthreads();
                const int c = s.misc[3];
                if (tid == 0) {
                    s.valid[q] = c;  // exact d2 <= tau, all of them in ok_k/ok_i
                    s.cnt[q] = c;
                }
                if (in_smem && c >= Nprime && c <= bufcap) {
#ifdef LAGP_NN_PROF
                    long long te0 = 0;
                    if (tid == 0) asm volatile("mov.u64 %0, %%clock64;" : "=l"(te0)::"memory");
#endif
                    emit(q, s.key, s.idx, c);
#ifdef LAGP_NN_PROF
                    if (tid == 0 && blockIdx.x < 1024) {
                        long long te1;
                        asm volatile("mov.u64 %0, %%clock64;" : "=l"(te1)::"memory");
                        g_nn_ph[blockIdx.x][9] += te1 - te0;
                        g_nn_ph[blockIdx.x][10] += 1;
                    }
#endif
                    if (tid == 0) s.state[q] = 3;
                }
                __syncthreads();
            }
            NN_PH(4);
            // missed queries: rescale tau (the count of rows inside the d^2 <= tau ball
            // grows like tau^(p/2)), aiming at ~1.5 N' survivors
            if (tid < NN_Q && s.state[tid] == 0) {
                const int q = tid;
                const int c = s.cnt[q] > bufcap ? s.cnt[q] : s.valid[q];  // overflow -> too many
                const double tau = s.tau[q];
                if (c >= Nprime && c <= bufcap) {
                    s.state[q] = 1;
                } else if (!isfinite(tau) || tau <= 0.0) {
                    s.state[q] = 2;  // cannot rescale (massive ties at 0, or already +inf)
                } else {
                    const double target = c < Nprime ? 1.5 * Nprime : 0.7 * bufcap;
                    double f = pow(target / (double)(c > 0 ? c : 1), 2.0 / (double)p);
                    if (c < Nprime && f < 1.05) f = 1.05;
                    if (c > bufcap && f > 0.95) f = 0.95;
                    s.tau[q] = tau * f;
                }
            }
            __syncthreads();
        }
        NN_PH(5);
        // queries still active after the rounds fall back as well
        if (tid < NN_Q && s.state[tid] == 0) s.state[tid] = 2;
        __syncthreads();

        // ---- per-query exact selection and output (queries not written yet)
        for (int q = 0; q < nq; q++) {
            if (s.state[q] == 3) continue;
            int c;
            uint64_t *qk = bufk + (size_t)q * bufcap;
            int32_t *qi = bufc + (size_t)q * bufcap;
            if (s.state[q] == 2) {
                if (tid == 0) atomicAdd(fallback_count, 1);
                nn_exact_select<P>(s, X, N, p, q, Nprime, qk, qi);
                c = Nprime;
            } else {
                c = s.cnt[q];
            }
            __syncthreads();
            emit(q, qk, qi, c);
        }
        NN_PH(6);
    }
}

size_t nn_smem_bytes() { return sizeof(NNSmem); }

// the NN work counters in the workspace header (after maxn2 and the bounds keys):
// [0] prefilter (row, query) pairs evaluated, [1] threshold-sample pairs, [2] exact keys
unsigned long long *nn_pair_counters(void *ws) {
    return reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(ws) + 384);
}

// per-query global survivor buffer: enough for ~1.5 N' plus sampling noise
// (capped at the shared-memory sort capacity when the sorted pool is requested)
static int nn_bufcap(int Nprime, bool sorted) {
    int c = 3 * Nprime;
    if (c < 2048) c = 2048;
    if (sorted && c > NN_CAP) c = NN_CAP;
    return c;
}

// Cell grid (see nn_cell_of).
// Two-axis grid (p <= 3, or the tensor-core filter): gx x gy cells on coordinates 0
// and 1, ~64 rows per cell; gx <= 128 when gy > 1 (the filter loads one run per cell
// column in parallel).
// Multi-axis grid (p >= 4): slabs on up to NN_CELL_DIMS coordinates, ~NN_CELL_ROWS rows
// per cell, one more slab at a time on the coordinate with the fewest (lowest first):
// C2 (N = 10^5, p = 8) 3 x 2^7 = 384 cells, C4 (N = 10^6) 3^6 x 2^2 = 2,916 cells.
// LAGP_NN_CELLS (A/B): 0 = one cell (no pruning), 2 = the two-axis grid.
// rows per cell: 96 up to N = 5e5, else 256 (measured at C2: NN 1.76 / 1.81 / 2.17 ms at
// 96 / 128 / 64 rows, 2.10 at 256; C4 18.2 vs 20.9 ms per 65,536 queries at 256 vs 128,
// where the 6,561-cell list costs more than the finer cells save); LAGP_NN_CR overrides
// (A/B)
static int nn_cell_rows(int64_t N) {
    const char *ev = getenv("LAGP_NN_CR");
    const int v = ev ? atoi(ev) : 0;
    return v >= 16 ? v : (N > 500000 ? 256 : 96);
}
static NNGrid nn_cells(int64_t N, int p, bool mma) {
    NNGrid g{};
    for (int k = 0; k < NN_CELL_DIMS; k++) g.s[k] = 1;
    g.nd = 1;
    g.multi = 0;
    const char *ev = getenv("LAGP_NN_CELLS");
    if (ev && ev[0] == '0') {
        // one cell
    } else if (p >= 4 && !mma && !(ev && ev[0] == '2')) {
        const int nd = p < NN_CELL_DIMS ? p : NN_CELL_DIMS;
        const double R = (double)nn_cell_rows(N);
        int64_t prod = 1;
        for (;;) {
            int k = 0;
            for (int t = 1; t < nd; t++)
                if (g.s[t] < g.s[k]) k = t;
            if (g.s[k] + 1 > NN_CELL_SMAX) break;
            const int64_t np = prod / g.s[k] * (g.s[k] + 1);
            if ((double)N / (double)np < R || np > NN_CELL_LIST) break;
            prod = np;
            g.s[k]++;
        }
        g.nd = 1;
        for (int k = 0; k < nd; k++)
            if (g.s[k] > 1) g.nd = k + 1;
        g.multi = 1;
    } else if (p == 1) {
        int64_t c = N / 64;
        g.s[0] = (int)(c < 1 ? 1 : (c > 16384 ? 16384 : c));
    } else {
        int c = (int)sqrt((double)N / 64.0);
        c = c < 1 ? 1 : (c > 128 ? 128 : c);
        g.s[0] = c;
        g.s[1] = c;
        g.nd = 2;
    }
    g.ncell = 1;
    for (int k = 0; k < g.nd; k++) g.ncell *= g.s[k];
    return g;
}
// the tensor-core filter (two-axis grid) when survivors are rare and the grid is not
// multi-axis; LAGP_NN_MMA=1 forces it (with the two-axis grid), 0 disables it
static bool nn_use_mma(int64_t N, int p, int Nprime) {
    if (p != 8) return false;
    const char *evm = getenv("LAGP_NN_MMA");
    if (evm) return evm[0] == '1';
    const char *ev = getenv("LAGP_NN_CELLS");
    const bool two_axis = ev && (ev[0] == '0' || ev[0] == '2');
    return two_axis && (double)Nprime <= 0.004 * (double)N;
}

// Workspace layout: [maxn2 bits, per-dimension min / max keys (512 B)] [X32: N*p floats] [rn2f: N floats]
// [perm: N] [cell counts, starts (C+1), cursors] for the rows and again for the queries [qperm: Mmax]
// [X64c: N*p doubles, X in cell order]
// [compacted rows] [survivor keys] [filter rows], the last three bufcap per query
struct NNLayout {
    size_t x32, rn2f, perm, rcnt, rstart, rcur, qcnt, qstart, qcur, qperm, x64c, rest;
    NNGrid g;
    bool mma;
};
static inline size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }
static NNLayout nn_layout(int64_t N, int p, int64_t Mmax, int Nprime) {
    NNLayout L;
    L.mma = nn_use_mma(N, p, Nprime);
    L.g = nn_cells(N, p, L.mma);
    const size_t C = (size_t)L.g.ncell;
    size_t o = 512;
    L.x32 = o; o += al256((size_t)N * p * sizeof(float));
    L.rn2f = o; o += al256((size_t)N * sizeof(float));
    L.perm = o; o += al256((size_t)N * sizeof(int32_t));
    L.rcnt = o; o += al256(C * sizeof(int32_t));
    L.rstart = o; o += al256((C + 1) * sizeof(int32_t));
    L.rcur = o; o += al256(C * sizeof(int32_t));
    L.qcnt = o; o += al256(C * sizeof(int32_t));
    L.qstart = o; o += al256((C + 1) * sizeof(int32_t));
    L.qcur = o; o += al256(C * sizeof(int32_t));
    L.qperm = o; o += al256((size_t)(Mmax > 0 ? Mmax : 1) * sizeof(int32_t));
    L.x64c = o; o += al256((size_t)N * p * sizeof(double));
    L.rest = o;
    return L;
}
size_t nn_ws_bytes(int grid, int64_t N, int p, int Nprime, bool sorted, int64_t Mmax) {
    const size_t bc = (size_t)nn_bufcap(Nprime, sorted);
    return nn_layout(N, p, Mmax, Nprime).rest + (size_t)grid * NN_Q * bc * (sizeof(uint64_t) + 2 * sizeof(int32_t)) + 256;
}

template <int P, bool MMA>
static cudaError_t launch_nn_t(const double *X, const float *X32, const float *rn2f, const unsigned long long *mx,
                               const unsigned long long *kmin, const unsigned long long *kmax, int64_t N, int p,
                               const double *XX, int64_t M, int Nprime, int n0, int sorted, int32_t *pool, double *d2,
                               char *w, int grid, int *fb, cudaStream_t st, NNGrid cg, const int32_t *cstart,
                               const int32_t *perm, const int32_t *qperm, int qg, const double *X64c,
                               unsigned long long *pairc) {
    size_t smem = sizeof(NNSmem);
    cudaError_t e = cudaFuncSetAttribute(nn_pool_kernel<P, MMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int bc = nn_bufcap(Nprime, sorted != 0);
    int32_t *bcmp = (int32_t *)w;
    w += (size_t)grid * NN_Q * bc * sizeof(int32_t);
    uint64_t *bk = (uint64_t *)w;
    w += (size_t)grid * NN_Q * bc * sizeof(uint64_t);
    int32_t *bi = (int32_t *)w;
    nn_pool_kernel<P, MMA><<<grid, NN_THREADS, smem, st>>>(X, X32, rn2f, mx, kmin, kmax, N, p, XX, M, Nprime, n0, bc, sorted,
                                                      pool, d2, bcmp, bk, bi, fb, cg, cstart, perm, qperm, qg, X64c, pairc);
    return cudaGetLastError();
}

// Query locations per group: 16 or 8. The tensor-core filter always takes 16 (its
// MMAs cover 2 x 8 queries; one 8-query group would idle half of them: C4 909 vs
// 776 ms). The FFMA2 filter takes 8 when p <= 4 (measured C3: 62.6 vs 67.0 ms) or
// when 8-groups fill the last round of the grid better (C2: 625 16-groups on 296
// CTAs = 2.1 rounds, 1250 8-groups = 4.2 rounds; 2.71 vs 3.02 ms).
// LAGP_NN_Q=8|16 overrides.
static int nn_group_size(int64_t M, int grid, int p, bool mma) {
    const char *ev = getenv("LAGP_NN_Q");
    if (ev) {  // A/B: 4, 8 or 16 (the tensor-core filter needs 16)
        const int v = atoi(ev);
        if ((v == 4 || v == 8 || v == 16) && !(mma && v != 16)) return v;
    }
    if (mma) return 16;
    if (p <= 4) return 8;
    const double g16 = (double)((M + 15) / 16) / grid, g8 = (double)((M + 7) / 8) / grid;
    const double eff16 = g16 / ceil(g16), eff8 = g8 / ceil(g8);
    return eff8 > 1.05 * eff16 ? 8 : 16;
}

int nn_grid(int64_t M, int num_sms, int Nprime) {
    int64_t groups = (M + 7) / 8;  // 8-query groups at the smallest (nn_group_size)
    int64_t g = 2LL * num_sms;  // 2 CTAs/SM fit (~110 KB smem each)
    // keep the survivor buffers under ~2 GiB for large pools
    const int64_t per_cta = (int64_t)NN_Q * nn_bufcap(Nprime, false) * 16;
    const int64_t gmax = ((int64_t)2 << 30) / per_cta;
    if (g > gmax) g = gmax > 1 ? gmax : 1;
    return (int)(groups < g ? (groups > 0 ? groups : 1) : g);
}

// Launches: rows (first chunk only) = bounds, cell histogram, scan, FP32 copy in cell
// order; queries (every chunk) = cell histogram, scan, scatter; then the pool kernel.
// With prepared = true the row results already in `ws` are reused (chunked calls;
// the layout is the same for every chunk: Mmax fixed by the caller).
cudaError_t launch_nn(const double *X, int64_t N, int p, const double *XX, int64_t M, int64_t Mmax, int Nprime, int n0,
                      bool sorted, int32_t *pool, double *d2, void *ws, int grid, int *fb, cudaStream_t st, bool prepared,
                      int *launches) {
    if (M > Mmax) return cudaErrorInvalidValue;
    char *w = (char *)ws;
    const NNLayout L = nn_layout(N, p, Mmax, Nprime);
    const int C = L.g.ncell;
    unsigned long long *mx = (unsigned long long *)w;
    unsigned long long *kmin = mx + 1, *kmax = mx + 1 + LAGP_PMAX;  // 8 + 2*16*8 = 264 <= 512 B
    unsigned long long *pairc = nn_pair_counters(ws);                 // bytes 384..407
    float *X32 = (float *)(w + L.x32);
    float *rn2f = (float *)(w + L.rn2f);
    int32_t *perm = (int32_t *)(w + L.perm), *rcnt = (int32_t *)(w + L.rcnt), *rstart = (int32_t *)(w + L.rstart),
            *rcur = (int32_t *)(w + L.rcur), *qcnt = (int32_t *)(w + L.qcnt), *qstart = (int32_t *)(w + L.qstart),
            *qcur = (int32_t *)(w + L.qcur), *qperm = (int32_t *)(w + L.qperm);
    char *rest = w + L.rest;
    double *X64c = (double *)(w + L.x64c);
    cudaError_t e;
    if (!prepared) {
        e = cudaMemsetAsync(mx, 0, sizeof(unsigned long long) * (1 + LAGP_PMAX), st);  // maxn2, kmin
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(kmin, 0xff, sizeof(unsigned long long) * LAGP_PMAX, st);
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(kmax, 0, sizeof(unsigned long long) * LAGP_PMAX, st);
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(pairc, 0, 3 * sizeof(unsigned long long), st);  // summed over the chunks
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(rcnt, 0, sizeof(int32_t) * C, st);
        if (e != cudaSuccess) return e;
        int blocks = (int)((N + 255) / 256);
        if (blocks > 4096) blocks = 4096;
        // few blocks: every block ends in 2p same-address global atomics (592 blocks: 32 us)
        nn_bounds_kernel<<<blocks < 148 ? blocks : 148, 256, 0, st>>>(X, N, p, kmin, kmax);
        nn_cell_hist_kernel<<<blocks, 256, 0, st>>>(X, N, p, kmin, kmax, L.g, rcnt);
        nn_cell_scan_kernel<<<1, 1024, 0, st>>>(rcnt, C, rstart, rcur);
        nn_prep_kernel<<<blocks, 256, 0, st>>>(X, N, p, X32, rn2f, mx, kmin, kmax, L.g, rcur, perm, X64c);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        if (launches) (*launches) += 4;
    }
    {
        e = cudaMemsetAsync(qcnt, 0, sizeof(int32_t) * C, st);
        if (e != cudaSuccess) return e;
        int blocks = (int)((M + 255) / 256);
        if (blocks > 4096) blocks = 4096;
        if (blocks < 1) blocks = 1;
        nn_cell_hist_kernel<<<blocks, 256, 0, st>>>(XX, M, p, kmin, kmax, L.g, qcnt);
        nn_cell_scan_kernel<<<1, 1024, 0, st>>>(qcnt, C, qstart, qcur);
        nn_cell_scatter_kernel<<<blocks, 256, 0, st>>>(XX, M, p, kmin, kmax, L.g, qcur, qperm);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        if (launches) (*launches) += 3;
    }
    if (launches) (*launches)++;
    const bool mma = L.mma;
    const int qg = nn_group_size(M, grid, p, mma);
#define NN_ARGS X, X32, rn2f, mx, kmin, kmax, N, p, XX, M, Nprime, n0, sorted ? 1 : 0, pool, d2, rest, grid, fb, st, L.g, rstart, perm, qperm, qg, X64c, pairc
    switch (p) {
        case 1: return launch_nn_t<1, false>(NN_ARGS);
        case 2: return launch_nn_t<2, false>(NN_ARGS);
        case 3: return launch_nn_t<3, false>(NN_ARGS);
        case 4: return launch_nn_t<4, false>(NN_ARGS);
        case 8: {
            // tensor-core filter when survivors are rare (~1.5 N'/N of the pairs pass)
            if (mma) return launch_nn_t<8, true>(NN_ARGS);
            return launch_nn_t<8, false>(NN_ARGS);
        }
        default: return launch_nn_t<0, false>(NN_ARGS);
    }
#undef NN_ARGS
}

}  // namespace lagp

#ifdef LAGP_NN_PROF
extern "C" int lagp_nn_prof(long long *out, int reset) {
    if (reset) {
        static long long z[1024][12];
        return (int)cudaMemcpyToSymbol(lagp::g_nn_ph, z, sizeof(z));
    }
    return (int)cudaMemcpyFromSymbol(out, lagp::g_nn_ph, sizeof(lagp::g_nn_ph));
}
#endif
