// alc_incremental_v2.cu — LAGP_ALC_INCREMENTAL for pools of
// N' <= 1024 candidates and p <= 8: the greedy ALC local design of Fig 1 step 2
// (Eq (5)-(6)) by per-candidate Schur-complement
// downdates, with ONE block barrier per greedy step.
//
// Arithmetic (same as alc_incremental.cu, restated): with K_j = L_j L_j^T every
// pool candidate c carries
//   w_c   = L_j^{-1} k_j(x_c)                   (j entries)
//   s_c   = 1 + eta - ||w_c||^2 = m_j^{-1}(x_c)  (Eq 6)
//   cov_c = kappa_c - z^T w_c,   z = L_j^{-1} h (kappa_c = K(x_c, x))
//   t_c   = y_c - y~^T w_c,      y~ = L_j^{-1} Y_j
// so Delta_c = cov_c^2 / s_c is Eq (5) (App A.1). Appending the winner c*
// (rho = sqrt(s_{c*})) is the partitioned-inverse step (a4) on the
// factor, L_{j+1} = [[L_j, 0], [w_{c*}^T, rho]], and every candidate downdates
//   e_c = K(x_c, x*) - w_{c*}^T w_c,  w_c[j] = e_c / rho,
//   s_c -= w_c[j]^2,  cov_c -= z_j w_c[j],  t_c -= y~_j w_c[j],
// with z_j = cov_{c*}/rho and y~_j = t_{c*}/rho. a5 (Eq 1-2) then
// needs only three running sums: mean = z^T y~, psi = ||y~||^2,
// s2 = psi (1 + eta - ||z||^2) / n.
//
// B200 mapping (differences from alc_incremental.cu):
//  * One persistent CTA per SM (the register file allows exactly one): 512 threads
//    with CPT = 2 candidates per thread (N' <= 512: CPT = 1; A/B shapes 256 x 4 and
//    1024 x 1), candidate c = tid + q*TH. The per-step broadcast reads of the
//    winner's data are shared by a thread's CPT candidates.
//  * Storage tiers of w_c: R entries in registers (R = 4 at p = 8, CPT = 2), then
//    shared memory in PAIRS (entry-major pairs of rows, double2 per (pair,
//    candidate): one LDS.128 per two entries, compile-time row stride), then tensor
//    memory (tcgen05.ld/st on the thread's own lane row: 32 entries per candidate),
//    then an L2-resident slab (pair layout) — n <= ~62 is on chip at N' = 1000.
//  * One barrier per step: each warp's best candidate posts its whole record
//    (key, x_c, s, cov, t, register and TMEM entries) before the barrier; after it
//    every warp reduces the 16 warp keys itself (redux.sync), reads the winner's
//    record and forms 1/rho = s^{-1/2} — no second barrier, no publish phase.
//  * Warps w and w+4 (same SMSP) run the FP64-bound K(x_c, x*) and the
//    shared-memory-bound dot in opposite orders; exp by a 16-entry table.
//  * y~ is maintained per candidate (t_c) instead of a warp-0 dot per step.
//  * Flags are accumulated per thread and reduced once per location.
#include <cuda_runtime.h>
#include <stdlib.h>

#include <type_traits>

#include "block_ops.cuh"
#include "launch.h"

namespace lagp {

// CTA shapes (threads TH x candidates per thread CPT): N' <= 512: 512 x 1; N' <= 1024:
// 512 x 2 (default), 256 x 4 or 1024 x 1 (A/B, LAGP_V2_CPT=4|1)

// register entries per candidate for (P, CPT, TH)
#ifndef LAGP_V2_STAG_EXPR
#define LAGP_V2_STAG_EXPR ((mode & 2) ? false : ((wid >> 2) & 1))
#endif
#ifndef LAGP_V2R_C2
#define LAGP_V2R_C2 2
#endif
#ifndef LAGP_V2R_C4
#define LAGP_V2R_C4 6
#endif
template <int P, int CPT, int TH>
struct V2R {
    static constexpr int value =
        (TH == 1024) ? 2 : (CPT == 1) ? 16 : (CPT == 2 ? (P <= 4 ? 8 : LAGP_V2R_C2) : (P <= 4 ? 8 : LAGP_V2R_C4));
};

// TMEM entries per candidate: each thread owns 256 KB / TH of tensor memory (its warp's
// 65536/TH columns of its lane quarter), shared by its CPT candidates
template <int CPT, int TH>
struct V2T {
    static constexpr int value = (65536 / TH) / 2 / CPT;
};

// warp post record (doubles): key | gidx,pos | key2 | - | x-x_ref[8] | s cov t |x-x_ref|^2/theta | w[R]
enum { RK = 0, RI = 1, RK2 = 2, RX = 4, RRHO = 12, RZN = 13, RYN = 14, RAC = 15, RW = 16 };
__host__ __device__ constexpr int v2_rec(int R) { return RW + R; }

// ---- tensor memory as per-thread storage (tcgen05; thread-private lane rows)
// 2E columns (E doubles) of this thread's row; tm_wait_ld() before using r
template <int E>
__device__ __forceinline__ void tm_ld(uint32_t taddr, uint32_t (&r)[2 * E]);
template <>
__device__ __forceinline__ void tm_ld<4>(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
template <>
__device__ __forceinline__ void tm_ld<8>(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
template <int N2>
__device__ __forceinline__ double tm_d(const uint32_t (&r)[N2], int k) {
    return __hiloint2double((int)r[2 * k + 1], (int)r[2 * k]);
}
__device__ __forceinline__ void tm_st1(uint32_t taddr, double v) {
    const uint32_t lo = (uint32_t)__double2loint(v), hi = (uint32_t)__double2hiint(v);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(taddr), "r"(lo), "r"(hi) : "memory");
}
// 16 zero columns (8 entries) of this thread's row
__device__ __forceinline__ void tm_zero16(uint32_t taddr) {
    const uint32_t z = 0;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
        "%1};\n" ::"r"(taddr),
        "r"(z)
        : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ double fast_div_pos(double a, double b) {
    // a / b for finite b > 0 (not tiny): reciprocal seed, one Newton step, then
    // one residual correction of the quotient (no special-case path)
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
    const double e = fma(-b, r, 1.0);
    r = fma(r, e, r);
    const double q = a * r;
    const double res = fma(-b, q, a);
    return fma(res, r, q);
}

#ifdef LAGP_V2_PROF
// clock probes (profiling builds only): lane 0 of every warp of CTA 0 on its first
// location, event k of step j: g_v2_ev[j][warp][k]
#define V2_NEV 12
__device__ long long g_v2_ev[128][32][V2_NEV];
#define V2_EV(k)                                                                    \
    do {                                                                            \
        if (lane == 0 && xi == blockIdx.x && blockIdx.x == 0 && j < 128) {          \
            long long t_;                                                           \
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_)::"memory");            \
            g_v2_ev[j][wid][k] = t_;                                                \
        }                                                                           \
    } while (0)
#else
#define V2_EV(k) \
    do {         \
    } while (0)
#endif

// mode bits: 1 = shared memory before tensor memory (A/B), 2 = no phase stagger (A/B)
template <int P, int CPT, int TH>
__global__ void __launch_bounds__(TH, 1)
alc_incremental_v2_kernel(AlcArgs A, int S, int mode) {
    constexpr int R = V2R<P, CPT, TH>::value;
    constexpr int NW = TH / 32;
    constexpr int NPC = TH * CPT;           // columns (candidates) per pair row
    constexpr int T = V2T<CPT, TH>::value;  // entries per candidate in tensor memory (multiple of 8)
    constexpr int REC = v2_rec(R);
    constexpr int TMC = CPT >= 2 ? 4 : 8;  // tensor-memory entries per load in the dot
    static_assert(T % 8 == 0 && REC % 2 == 0, "tier sizes");
    extern __shared__ __align__(16) double sm[];
    double2 *wsm2 = reinterpret_cast<double2 *>(sm);  // [S/2][NPC] pairs of shared-memory entries
    double *post = sm + (size_t)S * NPC;              // [2][NW][REC]
    double *wtm = post + 2 * NW * REC;                // [T] the winner's tensor-memory entries (this step)
    // [n][NW + 1] per greedy step: every warp's best key and the winner warp's second
    // best (top-2 gaps and the near-tie flag, formed once per location)
    unsigned long long *glog = reinterpret_cast<unsigned long long *>(wtm + T);
    const int n = A.n, Np = A.Nprime, n0 = A.n0;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // entry tiers of w_c: registers [0, R), tensor memory [T0, T1), shared memory
    // [S0, S1), L2 slab [G0, n); mode bit 1 puts shared memory first
    const int T0 = (mode & 1) ? R + S : R, T1 = T0 + T;
    const int S0 = (mode & 1) ? R : R + T, S1 = S0 + S;
    const int G0 = R + S + T;
    const int G = n - n0;
    const double eta = A.eta;
    double2 *gw2 = reinterpret_cast<double2 *>(A.cache + (size_t)blockIdx.x * A.cache_stride);  // [(a-G0)/2][NPC]
    __shared__ double xq[8];
    __shared__ uint32_t s_taddr;
    __shared__ volatile int s_pub;  // sequence number of the last winner-TMEM publication
    // all 512 TMEM columns (one CTA per SM); warp w owns lanes 32(w%4).. and columns
    // (65536/TH)(w/4).. : candidate slot q's entry e at column 2(qT + e)
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&s_taddr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 32) s_pub = -1;
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tbase = s_taddr + ((uint32_t)(32 * (wid & 3)) << 16) + (uint32_t)((65536 / TH) * (wid >> 2));
    __shared__ double zyv[2][LAGP_NMAX];  // z_j, y~_j of every append (a5)
    __shared__ double s_exptab[16];        // 2^(k/16) for exp_nonpos_tab
    if (threadIdx.x < 16) s_exptab[threadIdx.x] = c_exp2_16[threadIdx.x];
    int pubseq = 0;  // sequence number of the next winner-TMEM publication (uniform)

    for (int64_t xi = blockIdx.x; xi < A.M; xi += gridDim.x) {
        const double rth = A.theta_vec ? 1.0 / A.theta_vec[xi] : A.rtheta;  // per-location theta (Fig 1 step 4)
        const int32_t *pool = A.pool + xi * (int64_t)Np;
        int32_t *idx = A.idx_out + xi * (int64_t)n;
        if (tid < P) xq[tid] = A.XX[xi * P + tid];
        for (int t = tid; t < n; t += TH) idx[t] = (t < n0) ? pool[t] : -1;
        __syncthreads();

        // ---- per-candidate state
        double xc[CPT][P];  // x_c - x (offsets from the reference location)
        double ac[CPT];     // |x_c - x|^2 / theta
        double s[CPT], cov[CPT], tc[CPT];
        double wr[CPT][R];
        bool chosen[CPT];
        int gidx[CPT];
        uint32_t fl = 0;
        bool in_range = true;  // every pool d^2 to x finite and d^2/theta <= 175
#pragma unroll
        for (int q = 0; q < CPT; q++) {
            const int c = tid + q * TH;
            const bool valid = c < Np;
            chosen[q] = !valid;  // padding columns never compete
            gidx[q] = valid ? pool[c] : 0x7fffffff - c;  // unique keys for the warp argmax
            double d2 = 0.0;
#pragma unroll
            for (int k = 0; k < P; k++) {
                const double diff = __dsub_rn(valid ? A.X[(int64_t)gidx[q] * P + k] : xq[k], xq[k]);
                xc[q][k] = diff;
                d2 = __fma_rn(diff, diff, d2);
            }
            ac[q] = d2 * rth;
            if (valid && !(ac[q] <= 175.0)) in_range = false;
            s[q] = 1.0 + eta;
            cov[q] = valid ? exp_nonpos_tab(-ac[q], s_exptab) : 0.0;  // kappa_c (z is empty at j = 0)
            tc[q] = valid ? A.Z[gidx[q]] : 0.0;             // y_c (y~ is empty at j = 0)
#pragma unroll
            for (int a = 0; a < R; a++) wr[q][a] = 0.0;
#pragma unroll
            for (int e = 0; e < T; e += 8) tm_zero16(tbase + 2 * (q * T + e));  // unwritten entries read as 0
        }
        tm_wait_st();
        // pairwise: d^2(x_c, x*) <= 2 d^2(x_c, x) + 2 d^2(x*, x), so every K(x_c, x*) of
        // this location has argument >= -700: the exp needs no range or NaN guard
        const bool fast = __syncthreads_and(in_range);
        bool exhausted = false;

        int j = 0;
        for (; j < n; j++) {
            V2_EV(0);
            const int par = j & 1;
            double *pst = post + par * (NW * REC);
            const double *rec;
            unsigned long long sk2 = ~0ull;  // the winner warp's per-lane second-best candidates
            if (j < n0) {
                // forced NN append (a2): pool position j (thread j, q = 0; j < n <= LAGP_NMAX <= TH)
                if (tid == j) {
                    double *r = pst;
#pragma unroll
                    for (int k = 0; k < P; k++) r[RX + k] = xc[0][k];
                    r[RRHO] = s[0];  // raw s, cov, t: the readers scale by 1/sqrt(s)
                    r[RZN] = cov[0];
                    r[RYN] = tc[0];
                    r[RAC] = ac[0];
#pragma unroll
                    for (int a = 0; a < R; a += 2)
                        *reinterpret_cast<double2 *>(r + RW + a) = make_double2(wr[0][a], wr[0][a + 1]);
                    reinterpret_cast<unsigned long long *>(r)[RI] =
                        ((unsigned long long)(unsigned)j << 32) | (unsigned)gidx[0];
                    chosen[0] = true;
                    if (!(s[0] > 0.0)) fl |= LAGP_FLAG_NONFINITE;
                }
                __syncthreads();
                rec = pst;
            } else {
                // ---- a3: keys of Delta_c = cov_c^2 / s_c (0 = not a candidate)
                unsigned long long key[CPT];
#pragma unroll
                for (int q = 0; q < CPT; q++) {
                    bool ok = !chosen[q];
                    if (ok && !(s[q] > kSMin)) {
                        fl |= LAGP_FLAG_SENTINEL;
                        ok = false;
                    }
                    const double dl = fast_div_pos(cov[q] * cov[q], s[q]);
                    if (ok && !(dl < INFINITY)) {  // NaN or inf
                        fl |= LAGP_FLAG_NONFINITE;
                        ok = false;
                    }
                    key[q] = ok ? (unsigned long long)__double_as_longlong(dl) + 1ull : 0ull;
                }
                unsigned long long kb = key[0], k2 = 0;
                int gb = gidx[0], qb = 0;
#pragma unroll
                for (int q = 1; q < CPT; q++) {
                    const bool b = key[q] > kb || (key[q] == kb && gidx[q] < gb);
                    k2 = b ? kb : (key[q] > k2 ? key[q] : k2);
                    kb = b ? key[q] : kb;
                    gb = b ? gidx[q] : gb;
                    qb = b ? q : qb;
                }
                V2_EV(1);
                // warp argmax on (key desc, gidx asc) with 32-bit redux
                const unsigned hi = (unsigned)(kb >> 32), lo = (unsigned)kb;
                const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
                const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
                const bool tie = hi == mh && lo == ml;
                const unsigned mi = __reduce_min_sync(0xffffffffu, tie ? (unsigned)gb : 0xffffffffu);
                const bool wl = tie && (unsigned)gb == mi;  // unique: gidx are distinct
                V2_EV(2);
                if (wl) {
                    double *r = pst + wid * REC;
                    reinterpret_cast<ulonglong2 *>(r)[0] =
                        make_ulonglong2(kb, ((unsigned long long)(unsigned)(tid + qb * TH) << 32) | (unsigned)gb);
#pragma unroll
                    for (int q = 0; q < CPT; q++) {
                        if (q == qb) {
#pragma unroll
                            for (int k = 0; k < P; k++) r[RX + k] = xc[q][k];
                            *reinterpret_cast<double2 *>(r + RRHO) = make_double2(s[q], cov[q]);
                            *reinterpret_cast<double2 *>(r + RYN) = make_double2(tc[q], ac[q]);  // raw s, cov, t
#pragma unroll
                            for (int a = 0; a < R; a += 2)
                                *reinterpret_cast<double2 *>(r + RW + a) = make_double2(wr[q][a], wr[q][a + 1]);
                        }
                    }
                }
                V2_EV(3);
                __syncthreads();
                // every warp: argmax over the warp posts
                unsigned long long pk = 0;
                unsigned pg = 0xffffffffu;
                if (lane < NW) {
                    const ulonglong2 kv = reinterpret_cast<const ulonglong2 *>(pst + lane * REC)[0];
                    pk = kv.x;
                    pg = (unsigned)kv.y;
                }
                const unsigned ph = (unsigned)(pk >> 32), pl = (unsigned)pk;
                const unsigned qh = __reduce_max_sync(0xffffffffu, ph);
                const unsigned ql = __reduce_max_sync(0xffffffffu, ph == qh ? pl : 0u);
                if ((qh | ql) == 0u) {  // no valid candidate left (uniform)
                    exhausted = true;
                    break;
                }
                const bool ptie = ph == qh && pl == ql;
                const unsigned qi = __reduce_min_sync(0xffffffffu, ptie ? pg : 0xffffffffu);
                const int W = __ffs(__ballot_sync(0xffffffffu, ptie && pg == qi)) - 1;
                rec = pst + W * REC;
                V2_EV(4);
                if (wid == NW - 1) {  // log every warp's best key (the gaps are formed at the end)
                    if (lane < NW) glog[(j - n0) * (NW + 1) + lane] = pk;
                    if (lane == 0) idx[j] = (int)qi;
                }
                if (wid == W) sk2 = wl ? k2 : kb;  // reduced at the end of the step (off the path)
            }
            // ---- a4 on the factor: every candidate takes its new entry and downdates
            const unsigned long long ri = reinterpret_cast<const unsigned long long *>(rec)[RI];
            const int cstar = (int)(ri >> 32);
#pragma unroll
            for (int q = 0; q < CPT; q++)
                if (cstar == tid + q * TH) chosen[q] = true;
            // the winner's tensor-memory entries [T0, j), published in wtm by its warp (a
            // warp-collective load of its lane row; entries of a chunk beyond j are 0 on both
            // sides); the other warps wait on s_pub only when they reach their TMEM dot
            const int mt = j <= T0 ? 0 : (j < T1 ? j : T1) - T0;
            if (mt > 0 && wid == ((cstar & (TH - 1)) >> 5)) {
                const int qs = cstar / TH, wlane = cstar & 31;
                tm_wait_st();  // the previous steps' TMEM stores (off the key/argmax path)
                for (int e = 0; e < mt; e += 8) {
                    uint32_t r[16];
                    tm_ld<8>(tbase + 2 * (qs * T + e), r);
                    tm_wait_ld();
                    if (lane == wlane) {
#pragma unroll
                        for (int k = 0; k < 8; k += 2)
                            *reinterpret_cast<double2 *>(wtm + e + k) = make_double2(tm_d(r, k), tm_d(r, k + 1));
                    }
                }
                if (lane == wlane) {
                    __threadfence_block();
                    s_pub = pubseq;
                }
                V2_EV(5);
            }
            // 1/rho = s*^{-1/2} (off the posting lanes' path: every thread forms it)
            const double rrho = rsqrt_nr(rec[RRHO]), znew = rec[RZN] * rrho, ynew = rec[RYN] * rrho;
            V2_EV(6);
            if (tid == TH - 1) {  // a5 state (summed once at the end)
                zyv[0][j] = znew;
                zyv[1][j] = ynew;
            }

            // Two phases per candidate: K(x_c, x*) (FP64 pipe) and the dot w_{c*}^T w_c
            // (shared / tensor memory). Warps w and w+4 (same SMSP) run them in opposite
            // orders, so the two units are busy at the same time.
            double kx[CPT];
            double acc[CPT][2];
#pragma unroll
            for (int q = 0; q < CPT; q++) acc[q][0] = acc[q][1] = 0.0;
            auto kx_phase = [&](auto fastc) {
                // -|x_c - x*|^2 / theta = 2 (x_c - x).(x* - x) / theta - (a_c + a*), offsets from
                // the reference location x (the pool lies in a ball around it)
                double dt[CPT][2];  // two partial sums: half the dependent-chain depth
#pragma unroll
                for (int q = 0; q < CPT; q++) dt[q][0] = dt[q][1] = 0.0;
#pragma unroll
                for (int k = 0; k < P; k++) {
                    const double xs = rec[RX + k];
#pragma unroll
                    for (int q = 0; q < CPT; q++) dt[q][k & 1] = fma(xc[q][k], xs, dt[q][k & 1]);
                }
                const double as = rec[RAC], r2 = 2.0 * rth;
#pragma unroll
                for (int q = 0; q < CPT; q++) {
                    const double xa = fma(dt[q][0] + dt[q][1], r2, -(ac[q] + as));
                    if constexpr (decltype(fastc)::value)
                        kx[q] = exp_nonpos_tab_inrange(xa, s_exptab);
                    else
                        kx[q] = exp_nonpos_tab(fmin(xa, 0.0), s_exptab);
                }
            };
            auto kx_any = [&]() {
                if (fast)
                    kx_phase(std::true_type{});
                else
                    kx_phase(std::false_type{});
                V2_EV(7);
            };
            auto dot_phase = [&]() {
                // register entries (entries >= j are 0 on both sides)
#pragma unroll
                for (int a = 0; a < R; a += 2) {
                    const double2 wv = *reinterpret_cast<const double2 *>(rec + RW + a);
#pragma unroll
                    for (int q = 0; q < CPT; q++) {
                        acc[q][0] = fma(wv.x, wr[q][a], acc[q][0]);
                        acc[q][1] = fma(wv.y, wr[q][a + 1], acc[q][1]);
                    }
                }
                // shared entries [S0, min(j, S1)): one LDS.128 per two entries of a column
                if (j > S0) {
                    const int m = (j < S1 ? j : S1) - S0;
                    const double2 *swin = wsm2 + cstar;
                    const double2 *sown = wsm2 + tid;
                    const int np = m >> 1;
#pragma unroll 2
                    for (int pr = 0; pr < np; pr++) {
                        const double2 wv = *swin;
#pragma unroll
                        for (int q = 0; q < CPT; q++) {
                            const double2 o = sown[q * TH];
                            acc[q][0] = fma(wv.x, o.x, acc[q][0]);
                            acc[q][1] = fma(wv.y, o.y, acc[q][1]);
                        }
                        swin += NPC;
                        sown += NPC;
                    }
                    if (m & 1) {
                        const double wv = reinterpret_cast<const double *>(swin)[0];
#pragma unroll
                        for (int q = 0; q < CPT; q++)
                            acc[q][0] = fma(wv, reinterpret_cast<const double *>(sown + q * TH)[0], acc[q][0]);
                    }
                }
                // slab entries [G0, j) (L2-resident), two pairs per iteration
                if (j > G0) {
                    const int m = j - G0;
                    const double2 *gwin = gw2 + cstar;
                    const double2 *gown = gw2 + tid;
                    const int np = m >> 1;
#pragma unroll 2
                    for (int pr = 0; pr < np; pr++) {
                        const double2 wv = *gwin;
#pragma unroll
                        for (int q = 0; q < CPT; q++) {
                            const double2 o = gown[q * TH];
                            acc[q][0] = fma(wv.x, o.x, acc[q][0]);
                            acc[q][1] = fma(wv.y, o.y, acc[q][1]);
                        }
                        gwin += NPC;
                        gown += NPC;
                    }
                    if (m & 1) {
                        const double wv = reinterpret_cast<const double *>(gwin)[0];
#pragma unroll
                        for (int q = 0; q < CPT; q++)
                            acc[q][0] = fma(wv, reinterpret_cast<const double *>(gown + q * TH)[0], acc[q][0]);
                    }
                }
                // tensor-memory entries [T0, T0 + mt): own rows by tcgen05.ld, TMC entries per
                // load (the first chunk's loads issued before the publication wait); the
                // winner's entries from wtm once its warp has published them
                if (mt > 0) {
                    uint32_t ra[CPT][2 * TMC];
                    tm_wait_st();  // this thread's TMEM stores of the previous steps
#pragma unroll
                    for (int q = 0; q < CPT; q++) tm_ld<TMC>(tbase + 2 * (q * T), ra[q]);
                    V2_EV(9);
                    while (s_pub != pubseq) {
                    }
                    __threadfence_block();
                    V2_EV(10);
                    for (int e = 0; e < mt; e += TMC) {
                        if (e > 0)
#pragma unroll
                            for (int q = 0; q < CPT; q++) tm_ld<TMC>(tbase + 2 * (q * T + e), ra[q]);
                        tm_wait_ld();
#pragma unroll
                        for (int k = 0; k < TMC; k += 2) {
                            const double2 wv = *reinterpret_cast<const double2 *>(wtm + e + k);
#pragma unroll
                            for (int q = 0; q < CPT; q++) {
                                acc[q][0] = fma(wv.x, tm_d(ra[q], k), acc[q][0]);
                                acc[q][1] = fma(wv.y, tm_d(ra[q], k + 1), acc[q][1]);
                            }
                        }
                    }
                }
            };
            if (LAGP_V2_STAG_EXPR) {  // warps w and w+4 share an SMSP: opposite orders
                dot_phase();
                kx_any();
            } else {
                kx_any();
                dot_phase();
            }
            V2_EV(8);
            if (mt > 0) pubseq++;
            double wn[CPT];
#pragma unroll
            for (int q = 0; q < CPT; q++) wn[q] = (kx[q] - (acc[q][0] + acc[q][1])) * rrho;
            // store entry j of every column in its tier (the tier is uniform per step)
            if (j < R) {
#pragma unroll
                for (int q = 0; q < CPT; q++)
#pragma unroll
                    for (int b = 0; b < R; b++)
                        if (b == j) wr[q][b] = wn[q];
            } else if (j >= T0 && j < T1) {
#pragma unroll
                for (int q = 0; q < CPT; q++) tm_st1(tbase + 2 * (q * T + (j - T0)), wn[q]);
            } else if (j >= S0 && j < S1) {
                double *dst = reinterpret_cast<double *>(wsm2 + ((j - S0) >> 1) * NPC + tid) + ((j - S0) & 1);
#pragma unroll
                for (int q = 0; q < CPT; q++) dst[2 * q * TH] = wn[q];
            } else {
                double *dst = reinterpret_cast<double *>(gw2 + ((j - G0) >> 1) * NPC + tid) + ((j - G0) & 1);
#pragma unroll
                for (int q = 0; q < CPT; q++) dst[2 * q * TH] = wn[q];
            }
#pragma unroll
            for (int q = 0; q < CPT; q++) {
                s[q] = fma(-wn[q], wn[q], s[q]);
                cov[q] = fma(-znew, wn[q], cov[q]);
                tc[q] = fma(-ynew, wn[q], tc[q]);
            }
            V2_EV(11);
            if (sk2 != ~0ull) {  // (warp-uniform) the winner warp's second-best key, for the top-2 gap
                const unsigned sh = __reduce_max_sync(0xffffffffu, (unsigned)(sk2 >> 32));
                const unsigned sl = __reduce_max_sync(0xffffffffu, (unsigned)(sk2 >> 32) == sh ? (unsigned)sk2 : 0u);
                if (lane == 0) glog[(j - n0) * (NW + 1) + NW] = ((unsigned long long)sh << 32) | sl;
            }
        }

        // ---- flags and a5: mean = z^T y~, psi = ||y~||^2, s2 = psi (1 + eta - ||z||^2) / j
        const bool any_sent = __syncthreads_or((fl & LAGP_FLAG_SENTINEL) != 0);
        const bool any_nonf = __syncthreads_or((fl & LAGP_FLAG_NONFINITE) != 0);
        if (wid == NW - 1) {
            // top-2 gap of every step: d1 = the best warp key, d2 = max(the winner warp's
            // second best, the other warps' best keys); equal best keys give gap 0
            const int ns = (j > n0 ? j : n0) - n0;  // greedy steps taken
            bool tie_any = false;
            for (int t = lane; t < ns; t += 32) {
                const unsigned long long *lg = glog + t * (NW + 1);
                unsigned long long k1 = 0, k2b = lg[NW];
                int wb = 0;
#pragma unroll
                for (int w = 0; w < NW; w++) {
                    const unsigned long long v = lg[w];
                    if (v > k1) {
                        k1 = v;
                        wb = w;
                    }
                }
#pragma unroll
                for (int w = 0; w < NW; w++)
                    if (w != wb && lg[w] > k2b) k2b = lg[w];
                const double d1 = __longlong_as_double((long long)(k1 - 1ull));
                const double d2 = k2b ? __longlong_as_double((long long)(k2b - 1ull)) : 0.0;
                const double gap = top2_gap(d1, d2);
                if (!(d1 > 0.0) || gap < kTieGap) tie_any = true;
                if (A.gap_out) A.gap_out[xi * G + t] = gap;
            }
            const bool near_tie = __any_sync(0xffffffffu, tie_any);
            double mu = 0.0, psi = 0.0, zz = 0.0;
            for (int a = lane; a < j; a += 32) {
                mu = fma(zyv[0][a], zyv[1][a], mu);
                psi = fma(zyv[1][a], zyv[1][a], psi);
                zz = fma(zyv[0][a], zyv[0][a], zz);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                mu += __shfl_xor_sync(0xffffffffu, mu, off);
                psi += __shfl_xor_sync(0xffffffffu, psi, off);
                zz += __shfl_xor_sync(0xffffffffu, zz, off);
            }
            if (lane == 0) {
            uint32_t f = (any_sent ? LAGP_FLAG_SENTINEL : 0u) | (any_nonf ? LAGP_FLAG_NONFINITE : 0u) |
                         (near_tie ? LAGP_FLAG_NEAR_TIE : 0u) | (exhausted ? LAGP_FLAG_EXHAUSTED : 0u);
            const double sc = psi * (1.0 + eta - zz) / (double)j;
            const double vr = j > 2 ? sc * (double)j / (double)(j - 2) : __longlong_as_double(0x7ff8000000000000LL);
            if (!isfinite(mu) || !isfinite(sc)) f |= LAGP_FLAG_NONFINITE;
            A.mean[xi] = mu;
            A.s2[xi] = sc;
            if (A.var) A.var[xi] = vr;
            if (A.flags) A.flags[xi] = f;
            if (f & (LAGP_FLAG_EXHAUSTED | LAGP_FLAG_NONFINITE)) atomicAdd(A.n_partial, 1);
            }
            if (A.gap_out)
                for (int t = ns + lane; t < G; t += 32) A.gap_out[xi * G + t] = __longlong_as_double(0x7ff8000000000000LL);
        }
        __syncthreads();
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(s_taddr));
}

// ---------------------------------------------------------------- host side
template <int P, int CPT, int TH>
static cudaError_t v2_launch_t(const AlcArgs &a, int S, int mode, int grid, size_t smem, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(alc_incremental_v2_kernel<P, CPT, TH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    alc_incremental_v2_kernel<P, CPT, TH><<<grid, TH, smem, st>>>(a, S, mode);
    return cudaGetLastError();
}

template <int CPT, int TH>
static int v2_R_t(int p) {
    switch (p) {
        case 1: return V2R<1, CPT, TH>::value;
        case 2: return V2R<2, CPT, TH>::value;
        case 3: return V2R<3, CPT, TH>::value;
        case 4: return V2R<4, CPT, TH>::value;
        case 8: return V2R<8, CPT, TH>::value;
        default: return -1;
    }
}

static int v2_R(int p, int cpt, int th) {
    if (th == 1024) return v2_R_t<1, 1024>(p);
    return cpt == 1 ? v2_R_t<1, 512>(p) : cpt == 2 ? v2_R_t<2, 512>(p) : v2_R_t<4, 256>(p);
}

bool inc_v2_plan(int n, int p, int Nprime, size_t smem_optin, IncPlan &pl) {
    if (Nprime > 1024) return false;
    int cpt = Nprime <= 512 ? 1 : 4, th = Nprime <= 512 ? 512 : 256;
    const char *ev = getenv("LAGP_V2_CPT");  // A/B experiments for N' in (512, 1024]: 2 (512 thr) or 1 (1024 thr)
    if (ev && Nprime > 512 && ev[0] == '2') { cpt = 2; th = 512; }
    if (ev && Nprime > 512 && ev[0] == '1') { cpt = 1; th = 1024; }
    const int R = v2_R(p, cpt, th);
    if (R < 0) return false;
    const int npc = th * cpt;
    const int T = (65536 / th) / 2 / cpt;
    int mode = 0;
    const char *sf = getenv("LAGP_V2_SFIRST");  // A/B: 1 = shared memory before tensor memory
    if (sf && sf[0] == '1') mode |= 1;
    const char *ns = getenv("LAGP_V2_NOSTAGGER");  // A/B: every warp runs K(x_c,x*) before the dot
    if (ns && ns[0] == '1') mode |= 2;
    const size_t fixed = ((size_t)2 * (th / 32) * v2_rec(R) + T + (size_t)n * (th / 32 + 1)) * sizeof(double);
    if (smem_optin < fixed + 2048) return false;
    const size_t pair_bytes = (size_t)npc * 2 * sizeof(double);
    int S = 2 * (int)((smem_optin - fixed - 2048) / pair_bytes);
    const int need = n - R - ((mode & 1) ? 0 : T) > 0 ? n - R - ((mode & 1) ? 0 : T) : 0;
    const int need2 = (need + 1) & ~1;
    if (S > need2) S = need2;
    pl = IncPlan{};
    pl.ok = true;
    pl.v2 = true;
    pl.tfirst = mode;
    pl.cpt = cpt;
    pl.threads = th;
    pl.R = R;
    pl.S = S;
    pl.global_entries = n - R - S - T > 0 ? n - R - S - T : 0;
    pl.smem = (size_t)S * npc * sizeof(double) + fixed;
    pl.wsz = S * npc;
    pl.cache_doubles = (int64_t)((pl.global_entries + 1) & ~1) * npc + 16;
    return true;
}

cudaError_t launch_alc_incremental_v2(const AlcArgs &a, const IncPlan &pl, int grid, cudaStream_t st) {
#define V2_DISPATCH(CPT_, TH_)                                                                 \
    switch (a.p) {                                                                             \
        case 1: return v2_launch_t<1, CPT_, TH_>(a, pl.S, pl.tfirst, grid, pl.smem, st);       \
        case 2: return v2_launch_t<2, CPT_, TH_>(a, pl.S, pl.tfirst, grid, pl.smem, st);       \
        case 3: return v2_launch_t<3, CPT_, TH_>(a, pl.S, pl.tfirst, grid, pl.smem, st);       \
        case 4: return v2_launch_t<4, CPT_, TH_>(a, pl.S, pl.tfirst, grid, pl.smem, st);       \
        case 8: return v2_launch_t<8, CPT_, TH_>(a, pl.S, pl.tfirst, grid, pl.smem, st);       \
        default: return cudaErrorInvalidValue;                                                 \
    }
    if (pl.threads == 1024) { V2_DISPATCH(1, 1024) }
    if (pl.cpt == 1) { V2_DISPATCH(1, 512) }
    if (pl.cpt == 2) { V2_DISPATCH(2, 512) }
    V2_DISPATCH(4, 256)
#undef V2_DISPATCH
}

}  // namespace lagp

#ifdef LAGP_V2_PROF
extern "C" int lagp_v2_prof(long long *out) {
    return (int)cudaMemcpyFromSymbol(out, lagp::g_v2_ev, sizeof(lagp::g_v2_ev));
}
#endif
