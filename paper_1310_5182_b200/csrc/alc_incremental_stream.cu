// alc_incremental_stream.cu — LAGP_ALC_INCREMENTAL for large
// candidate pools, 1024 < N' <= 65,536 (the paper's LGBB N' = 10,000 variant,
// P:1029-1032; the C5 sweep up to N' = 60,000): the greedy ALC local design of Fig 1
// step 2 (Eq (5)-(6)) by the per-candidate Schur-complement
// downdates of alc_incremental_v2.cu (arithmetic restated there), with the whole
// per-candidate state in HBM.
//
// Every candidate c of the pool carries x_c - x (offsets from the reference location),
// s_c = m_j^{-1}(x_c), cov_c, t_c and w_c = L_j^{-1} k_j(x_c) (j entries). A pool of
// N' = 60,000 with n = 128 is 60 MB per location: it cannot live on chip, so the state
// is a per-CTA slab in HBM, entry-major (w[a][c] contiguous in c: coalesced), and each
// greedy step is ONE streaming pass over it:
//   for every unchosen c:  K(x_c, x*) - w_{c*}^T w_c -> w_c[j]; s_c, cov_c, t_c downdated
//                          and stored; the key Delta_c = cov_c^2 / s_c of the next step.
// Per step the CTA then reduces the keys (warp redux, one barrier), gathers the winner's
// column (j scattered loads by j threads) and its scalars into shared memory (second
// barrier), and streams again. The pass reads (p + j + 4) and writes 4 doubles per
// candidate: HBM-bound by design (bench roofline "hbm"). Two CTAs per SM, so one
// location's argmax/gather latency overlaps the other's stream.
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "launch.h"

namespace lagp {

constexpr int STR_TH = 512;
constexpr int STR_NW = STR_TH / 32;

// slab (doubles) per CTA: gid [Npad/2 (int32)] | x - x_ref [p][Npad] | s, cov, t [3][Npad] | w [n][Npad]
__host__ __device__ inline int64_t str_slab_doubles(int n, int p, int Npad) {
    return (int64_t)Npad / 2 + (int64_t)(p + 3 + n) * Npad + 64;
}

template <int P>
__global__ void __launch_bounds__(STR_TH, 2) alc_incremental_stream_kernel(AlcArgs A) {
    const int n = A.n, Np = A.Nprime, n0 = A.n0, G = n - n0;
    const int p = P ? P : A.p;
    const int64_t Npad = (Np + 31) & ~31;  // slab stride (inc_stream_npad)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    double *slab = A.cache + (size_t)blockIdx.x * A.cache_stride;
    int32_t *gid = reinterpret_cast<int32_t *>(slab);
    double *xs = slab + Npad / 2;
    double *sv = xs + (int64_t)p * Npad, *cv = sv + Npad, *tv = cv + Npad;
    double *w = tv + Npad;
    const double eta = A.eta;
    __shared__ double ws[LAGP_NMAX];          // the winner's w entries
    __shared__ double xst[LAGP_PMAX + 4];     // the winner's x - x_ref, s, cov, t
    __shared__ double xq[LAGP_PMAX];
    __shared__ double zyv[2][LAGP_NMAX];
    __shared__ unsigned long long pk[STR_NW], pk2[STR_NW];
    __shared__ unsigned pg[STR_NW];
    __shared__ int pc[STR_NW];
    __shared__ double s_exptab[16];
    if (tid < 16) s_exptab[tid] = c_exp2_16[tid];

    for (int64_t xi = blockIdx.x; xi < A.M; xi += gridDim.x) {
        const double rth = A.theta_vec ? 1.0 / A.theta_vec[xi] : A.rtheta;
        const int32_t *pool = A.pool + xi * (int64_t)Np;
        int32_t *idx = A.idx_out + xi * (int64_t)n;
        if (tid < p) xq[tid] = A.XX[xi * p + tid];
        for (int t = tid; t < n; t += STR_TH) idx[t] = (t < n0) ? pool[t] : -1;
        __syncthreads();
        // ---- initial state: offsets, s = 1 + eta, cov = kappa_c, t = y_c (z, y~ empty)
        for (int c = tid; c < Npad; c += STR_TH) {
            const int g = c < Np ? pool[c] : -1;
            gid[c] = g;
            if (g < 0) continue;
            double d2 = 0.0;
            for (int k = 0; k < p; k++) {
                const double diff = __dsub_rn(A.X[(int64_t)g * p + k], xq[k]);
                xs[k * Npad + c] = diff;
                d2 = __fma_rn(diff, diff, d2);
            }
            sv[c] = 1.0 + eta;
            cv[c] = exp_nonpos_tab(-d2 * rth, s_exptab);
            tv[c] = A.Z[g];
        }
        uint32_t fl = 0;
        bool near_tie = false, exhausted = false;
        int j = 0;
        // thread best of the current keys: (key, gidx, position), second-best key
        unsigned long long kb = 0, k2 = 0;
        int gb = 0x7fffffff, cb = -1;
        __syncthreads();
        for (; j < n; j++) {
            int cstar;
            if (j < n0) {
                cstar = j;  // the forced NN append (pool position j)
                __syncthreads();  // the last pass's stores (its column, s, cov, t) before the gather
            } else {
                // ---- argmax of the keys formed in the last pass (ties -> lowest global row)
                const unsigned hi = (unsigned)(kb >> 32), lo = (unsigned)kb;
                const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
                const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
                const bool tie = hi == mh && lo == ml;
                const unsigned mi = __reduce_min_sync(0xffffffffu, tie ? (unsigned)gb : 0xffffffffu);
                const bool wl = tie && (unsigned)gb == mi;
                const unsigned long long sk = wl ? k2 : kb;
                const unsigned sh = __reduce_max_sync(0xffffffffu, (unsigned)(sk >> 32));
                const unsigned sl = __reduce_max_sync(0xffffffffu, (unsigned)(sk >> 32) == sh ? (unsigned)sk : 0u);
                if (wl) {
                    pk[wid] = kb;
                    pg[wid] = (unsigned)gb;
                    pc[wid] = cb;
                    pk2[wid] = ((unsigned long long)sh << 32) | sl;
                }
                __syncthreads();
                unsigned long long qk = 0;
                unsigned qg = 0xffffffffu;
                if (lane < STR_NW) {
                    qk = pk[lane];
                    qg = pg[lane];
                }
                const unsigned qh = __reduce_max_sync(0xffffffffu, (unsigned)(qk >> 32));
                const unsigned ql = __reduce_max_sync(0xffffffffu, (unsigned)(qk >> 32) == qh ? (unsigned)qk : 0u);
                if ((qh | ql) == 0u) {  // no valid candidate left (uniform)
                    exhausted = true;
                    break;
                }
                const bool qt = (unsigned)(qk >> 32) == qh && (unsigned)qk == ql;
                const unsigned qi = __reduce_min_sync(0xffffffffu, qt ? qg : 0xffffffffu);
                const int W = __ffs(__ballot_sync(0xffffffffu, qt && qg == qi)) - 1;
                cstar = pc[W];
                if (tid == 0) {  // top-2 gap: max(winner warp's second, other warps' best)
                    unsigned long long k2b = pk2[W];
                    for (int w2 = 0; w2 < STR_NW; w2++)
                        if (w2 != W && pk[w2] > k2b) k2b = pk[w2];
                    const unsigned long long k1 = ((unsigned long long)qh << 32) | ql;
                    const double d1 = __longlong_as_double((long long)(k1 - 1ull));
                    const double d2 = k2b ? __longlong_as_double((long long)(k2b - 1ull)) : 0.0;
                    const double gap = top2_gap(d1, d2);
                    if (!(d1 > 0.0) || gap < kTieGap) near_tie = true;
                    if (A.gap_out) A.gap_out[xi * G + (j - n0)] = gap;
                    idx[j] = (int)qi;
                }
            }
            // ---- the winner's column and scalars into shared memory; mark it chosen
            for (int a = tid; a < j; a += STR_TH) ws[a] = w[(int64_t)a * Npad + cstar];
            if (tid >= STR_TH - 32) {
                const int k = tid - (STR_TH - 32);
                if (k < p) xst[k] = xs[(int64_t)k * Npad + cstar];
                if (k == 16) xst[LAGP_PMAX] = sv[cstar];
                if (k == 17) xst[LAGP_PMAX + 1] = cv[cstar];
                if (k == 18) xst[LAGP_PMAX + 2] = tv[cstar];
            }
            __syncthreads();
            if (tid == 0) gid[cstar] = -1;  // chosen (read again only after the next barrier)
            const double sst = xst[LAGP_PMAX];
            if (tid == 0 && !(sst > 0.0)) fl |= LAGP_FLAG_NONFINITE;
            const double rrho = rsqrt_nr(sst), znew = xst[LAGP_PMAX + 1] * rrho, ynew = xst[LAGP_PMAX + 2] * rrho;
            if (tid == 0) {
                zyv[0][j] = znew;
                zyv[1][j] = ynew;
            }
            if (j + 1 >= n) continue;  // the last append needs no candidate update
            // ---- the streaming pass: new entry j of every w_c, downdates, next keys
            const bool keys = j + 1 >= n0 && j + 1 < n;
            kb = 0;
            k2 = 0;
            gb = 0x7fffffff;
            cb = -1;
            for (int c = tid; c < Np; c += STR_TH) {
                const int g = gid[c];
                if (g < 0 || c == cstar) continue;
                double d2a = 0.0, d2b = 0.0;
#pragma unroll
                for (int k = 0; k < (P ? P : LAGP_PMAX); k++) {
                    if (!P && k >= p) break;
                    const double df = xs[(int64_t)k * Npad + c] - xst[k];
                    if (k & 1)
                        d2b = fma(df, df, d2b);
                    else
                        d2a = fma(df, df, d2a);
                }
                const double kx = exp_nonpos_tab(-(d2a + d2b) * rth, s_exptab);
                double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
                const double *wc = w + c;
                int a = 0;
                for (; a + 4 <= j; a += 4) {
                    a0 = fma(ws[a], wc[(int64_t)a * Npad], a0);
                    a1 = fma(ws[a + 1], wc[(int64_t)(a + 1) * Npad], a1);
                    a2 = fma(ws[a + 2], wc[(int64_t)(a + 2) * Npad], a2);
                    a3 = fma(ws[a + 3], wc[(int64_t)(a + 3) * Npad], a3);
                }
                for (; a < j; a++) a0 = fma(ws[a], wc[(int64_t)a * Npad], a0);
                const double wn = (kx - ((a0 + a1) + (a2 + a3))) * rrho;
                w[(int64_t)j * Npad + c] = wn;
                const double s = fma(-wn, wn, sv[c]);
                const double cov = fma(-znew, wn, cv[c]);
                sv[c] = s;
                cv[c] = cov;
                tv[c] = fma(-ynew, wn, tv[c]);
                if (keys) {
                    bool ok = true;
                    if (!(s > kSMin)) {
                        fl |= LAGP_FLAG_SENTINEL;
                        ok = false;
                    }
                    const double dl = cov * cov / s;
                    if (ok && !(dl < INFINITY)) {
                        fl |= LAGP_FLAG_NONFINITE;
                        ok = false;
                    }
                    if (ok) {
                        const unsigned long long key = (unsigned long long)__double_as_longlong(dl) + 1ull;
                        if (key > kb || (key == kb && g < gb)) {
                            k2 = kb;
                            kb = key;
                            gb = g;
                            cb = c;
                        } else if (key > k2) {
                            k2 = key;
                        }
                    }
                }
            }
        }
        // ---- flags and a5: mean = z^T y~, psi = ||y~||^2, s2 = psi (1 + eta - ||z||^2) / j
        const bool any_sent = __syncthreads_or((fl & LAGP_FLAG_SENTINEL) != 0);
        const bool any_nonf = __syncthreads_or((fl & LAGP_FLAG_NONFINITE) != 0);
        const bool any_tie = __syncthreads_or(near_tie);
        if (wid == 0) {
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
                             (any_tie ? LAGP_FLAG_NEAR_TIE : 0u) | (exhausted ? LAGP_FLAG_EXHAUSTED : 0u);
                const double sc = psi * (1.0 + eta - zz) / (double)j;
                const double vr =
                    j > 2 ? sc * (double)j / (double)(j - 2) : __longlong_as_double(0x7ff8000000000000LL);
                if (!isfinite(mu) || !isfinite(sc)) f |= LAGP_FLAG_NONFINITE;
                A.mean[xi] = mu;
                A.s2[xi] = sc;
                if (A.var) A.var[xi] = vr;
                if (A.flags) A.flags[xi] = f;
                if (f & (LAGP_FLAG_EXHAUSTED | LAGP_FLAG_NONFINITE)) atomicAdd(A.n_partial, 1);
            }
            if (A.gap_out) {
                const int ns = (j > n0 ? j : n0) - n0;
                for (int t = ns + lane; t < G; t += 32) A.gap_out[xi * G + t] = __longlong_as_double(0x7ff8000000000000LL);
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- host side
bool inc_stream_plan(int n, int p, int Nprime, IncPlan &pl) {
    if (Nprime > 65536 || p > LAGP_PMAX || n > LAGP_NMAX) return false;
    const int Npad = (Nprime + 31) & ~31;
    pl = IncPlan{};
    pl.ok = true;
    pl.stream = true;
    pl.threads = STR_TH;
    pl.cpt = 0;
    pl.R = 0;
    pl.S = 0;
    pl.global_entries = n;
    pl.smem = 0;
    pl.cache_doubles = str_slab_doubles(n, p, Npad);
    return true;
}

int inc_stream_npad(int Nprime) { return (Nprime + 31) & ~31; }

template <int P>
static cudaError_t str_launch_t(const AlcArgs &a, int grid, cudaStream_t st) {
    alc_incremental_stream_kernel<P><<<grid, STR_TH, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_alc_incremental_stream(const AlcArgs &a, int grid, cudaStream_t st) {
    switch (a.p) {
        case 1: return str_launch_t<1>(a, grid, st);
        case 2: return str_launch_t<2>(a, grid, st);
        case 3: return str_launch_t<3>(a, grid, st);
        case 4: return str_launch_t<4>(a, grid, st);
        case 8: return str_launch_t<8>(a, grid, st);
        default: return str_launch_t<0>(a, grid, st);
    }
}

}  // namespace lagp
