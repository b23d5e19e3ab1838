// alc_scores_gemm.cu — row a3 alone at the paper's Fig 4 scale (SURVEY §8f row
// f4; one reference location, N' = 60,000 candidates, local design
// size n = 16..512, K_n^{-1} given): the ALC scores of Eq (5)-(6) for every
// candidate, as a dense FP64 contraction on the tensor path.
//
// For a location with design X_j (j rows), explicit K_j^{-1} and candidates x_c:
//   h = k_j(x), w = K_j^{-1} h                       (prep kernel, once per location)
//   Kc = [k_j(x_c1) .. k_j(x_cT)]                    (j × T tile, built in shared memory)
//   U  = K_j^{-1} Kc                                 (DMMA: mma.sync m8n8k4 f64)
//   q_c = sum_a Kc[a][c] U[a][c],  s_c = 1 + eta - q_c  (= m_j^{-1}(x_c), Eq 6)
//   cov_c = kappa_c - w^T k_c,     Delta_c = cov_c^2 / s_c (Eq 5, reading R1)
// With T = 32-64 candidates per CTA the j × j by j × T product is a genuinely dense
// GEMM (j up to 768), unlike the greedy loop's per-location matvecs: this is the
// one place of the path where the FP64 tensor instruction is the right tool.
// Per-CTA (Delta, row) top-2 go to a workspace; a second kernel merges them per
// location (argmax ties to the lowest candidate row id, R7; gap R19).
//
// Fragment layouts (PTX ISA, mma.m8n8k4 .f64): A a0 = A[g][k], B b0 = B[k][g],
// C {c0,c1} = C[g][2k], C[g][2k+1] with g = lane>>2, k = lane&3. The tile row
// stride T + 4 ≡ 4 (mod 16) doubles makes every B fragment load conflict-free
// (64-bit loads are served per half-warp).
#include <cuda_runtime.h>

#include "block_ops.cuh"
#include "launch.h"

namespace lagp {

constexpr int SG_THREADS = 256;  // 8 warps
// candidates per CTA: T = 32 or 64 (4 or 8 column blocks of 8); tile row stride
// TL = T + 4 (≡ 4 mod 16 doubles: conflict-free B fragments). Every A fragment of
// K^{-1} (streamed from L2) feeds T/8 DMMAs, so T = 64 halves the K^{-1} traffic
// per flop, but measured slower (occupancy): T = 32 is used.
__host__ __device__ constexpr int sg_tl(int T) { return T + 4; }

__device__ __forceinline__ void sg_cp16(void *smem, const void *gmem) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(gmem));
}
__device__ __forceinline__ void sg_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void sg_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
constexpr int SG_AL = 36;              // staged K^{-1} chunk row stride (≡ 4 mod 16: conflict-free A fragments)
constexpr int SG_ABUF = 2 * 8 * SG_AL;  // per warp: two 8 × 32 chunks

__device__ __forceinline__ void sg_dmma(double &c0, double &c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

// prep: h = k_j(x), w = K^{-1} h for location b (one CTA per location).
__global__ void __launch_bounds__(SG_THREADS)
alc_scores_prep_kernel(int j, int p, const double *__restrict__ Xj, const double *__restrict__ Kinv,
                       const double *__restrict__ xref, double rtheta, double *__restrict__ wout, int wl) {
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    double *h = sm;  // j
    __shared__ double xq[LAGP_PMAX];
    if (tid < p) xq[tid] = xref[(size_t)b * p + tid];
    __syncthreads();
    const double *Xb = Xj + (size_t)b * j * p;
    for (int a = tid; a < j; a += SG_THREADS) h[a] = corr_from_d2(sqdist_fma(Xb + (size_t)a * p, xq, p), rtheta);
    __syncthreads();
    const double *K = Kinv + (size_t)b * j * j;
    for (int a = wid; a < j; a += SG_THREADS / 32) {
        double acc = 0.0;
        for (int t = lane; t < j; t += 32) acc = fma(K[(size_t)a * j + t], h[t], acc);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) wout[(size_t)b * wl + a] = acc;
    }
}

// scores: grid (ceil(nc / T), B)
template <int SG_T, bool STAGE>
__global__ void __launch_bounds__(SG_THREADS)
alc_scores_gemm_kernel(int j, int p, int nc, const double *__restrict__ Xj, const double *__restrict__ Kinv,
                       const double *__restrict__ cands, const int32_t *__restrict__ cand_idx,
                       const double *__restrict__ xref, double rtheta, double eta, const double *__restrict__ wvec,
                       int wl, double *__restrict__ delta_out, double *__restrict__ part) {
    extern __shared__ __align__(16) double sm[];
    const int b = blockIdx.y, c0 = blockIdx.x * SG_T;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int g = lane >> 2, kq = lane & 3;
    constexpr int SG_TL = sg_tl(SG_T);
    constexpr int CB = SG_T / 8;                 // column blocks
    const int jr = (j + 7) & ~7;                 // rows padded to the 8-row blocks
    double *Kc = sm;                             // jr × SG_TL
    double *xcs = Kc + (size_t)jr * SG_TL;       // T × p candidate coordinates
    double *qred = xcs + SG_T * LAGP_PMAX;       // 8 warps × T partial q
    double *cvred = qred + 8 * SG_T;             // T: w^T k_c
    double *Abuf = cvred + SG_T + wid * SG_ABUF; // this warp's staged K^{-1} chunks
    __shared__ double xq[LAGP_PMAX];
    const double *Xb = Xj + (size_t)b * j * p;
    if (tid < p) xq[tid] = xref[(size_t)b * p + tid];
    for (int e = tid; e < SG_T * p; e += SG_THREADS) {
        const int c = e / p, k = e - c * p;
        xcs[e] = (c0 + c < nc) ? cands[((size_t)b * nc + c0 + c) * p + k] : 0.0;
    }
    __syncthreads();
    // Kc tile: entry (a, c) = K(X_a, x_c); rows >= j and columns >= nc are 0
    for (int e = tid; e < jr * SG_T; e += SG_THREADS) {
        const int a = e / SG_T, c = e - a * SG_T;
        double v = 0.0;
        if (a < j && c0 + c < nc) v = corr_from_d2(sqdist_fma(Xb + (size_t)a * p, xcs + c * p, p), rtheta);
        Kc[a * SG_TL + c] = v;
    }
    __syncthreads();
    // cov part: w^T k_c (warp w: columns CB*w .. CB*w + CB - 1)
    {
        const double *wb = wvec + (size_t)b * wl;
        for (int cc = 0; cc < CB; cc++) {
            const int c = CB * wid + cc;
            double acc = 0.0;
            for (int a = lane; a < j; a += 32) acc = fma(wb[a], Kc[a * SG_TL + c], acc);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) cvred[c] = acc;
        }
    }
    // U = K^{-1} Kc by 8-row blocks (warp w: row blocks w, w+8, ...), q partials
    const double *K = Kinv + (size_t)b * j * j;
    double qp[CB][2];
#pragma unroll
    for (int cb = 0; cb < CB; cb++) qp[cb][0] = qp[cb][1] = 0.0;
    const int nrb = jr >> 3;
    for (int rb = wid; rb < nrb; rb += 8) {
        const int row = 8 * rb + g;
        const bool rok = row < j;
        const double *Krow = K + (size_t)(rok ? row : 0) * j;
        double acc[CB][2];
#pragma unroll
        for (int cb = 0; cb < CB; cb++) acc[cb][0] = acc[cb][1] = 0.0;
        int t = 0;
        // main loop: 8 × 32 chunks of the warp's K^{-1} row block staged into shared
        // memory by cp.async (double-buffered: chunk c+1 in flight while chunk c feeds
        // 8 k-steps × T/8 DMMAs); j even keeps every 16-byte copy aligned
        const int nfull = (STAGE && j % 2 == 0) ? j / 32 : 0;
        if (nfull > 0) {
            auto issue = [&](int ch) {
                double *dst = Abuf + (ch & 1) * (8 * SG_AL);
                for (int sg = lane; sg < 128; sg += 32) {
                    const int r = sg >> 4, cs = (sg & 15) * 2;
                    const int rr = (8 * rb + r < j) ? 8 * rb + r : 0;  // rows >= j: masked at use
                    sg_cp16(dst + r * SG_AL + cs, K + (size_t)rr * j + ch * 32 + cs);
                }
                sg_commit();
            };
            issue(0);
            for (int ch = 0; ch < nfull; ch++) {
                if (ch + 1 < nfull)
                    issue(ch + 1);
                else
                    sg_commit();  // empty group: the wait below always means "chunk ch landed"
                sg_wait1();
                __syncwarp();
                const double *Ab = Abuf + (ch & 1) * (8 * SG_AL) + g * SG_AL;
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const double a = rok ? Ab[4 * u + kq] : 0.0;
                    const double *Brow = Kc + (ch * 32 + 4 * u + kq) * SG_TL + g;
#pragma unroll
                    for (int cb = 0; cb < CB; cb++) sg_dmma(acc[cb][0], acc[cb][1], a, Brow[8 * cb]);
                }
                __syncwarp();
            }
            t = nfull * 32;
        }
        for (; t + 32 <= j; t += 32) {  // odd j: A fragments straight from L2
            double av[8];
#pragma unroll
            for (int u = 0; u < 8; u++) av[u] = rok ? __ldg(Krow + t + 4 * u + kq) : 0.0;
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const double *Brow = Kc + (t + 4 * u + kq) * SG_TL + g;
#pragma unroll
                for (int cb = 0; cb < CB; cb++) sg_dmma(acc[cb][0], acc[cb][1], av[u], Brow[8 * cb]);
            }
        }
        for (; t < j; t += 4) {
            const int col = t + kq;
            const double a = (rok && col < j) ? __ldg(Krow + col) : 0.0;
            const double *Brow = Kc + (size_t)col * SG_TL + g;  // rows >= j are 0 in the tile
#pragma unroll
            for (int cb = 0; cb < CB; cb++) sg_dmma(acc[cb][0], acc[cb][1], a, col < jr ? Brow[8 * cb] : 0.0);
        }
        // q partial: sum over this row block of Kc[a][c] U[a][c]
        const double *Krw = Kc + (size_t)row * SG_TL;
#pragma unroll
        for (int cb = 0; cb < CB; cb++) {
            qp[cb][0] = fma(Krw[8 * cb + 2 * kq], acc[cb][0], qp[cb][0]);
            qp[cb][1] = fma(Krw[8 * cb + 2 * kq + 1], acc[cb][1], qp[cb][1]);
        }
    }
    // reduce over g (lane bits 2..4), then across warps
#pragma unroll
    for (int cb = 0; cb < CB; cb++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
            double v = qp[cb][h];
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            if (g == 0) qred[wid * SG_T + 8 * cb + 2 * kq + h] = v;
        }
    __syncthreads();
    // scores and the CTA's top-2 (warp 0; lane takes columns lane, lane + 32)
    if (wid == 0) {
        Top2 t2;
        t2.init();
#pragma unroll
        for (int h = 0; h < SG_T / 32; h++) {
            const int c = lane + 32 * h;
            double q = 0.0;
#pragma unroll
            for (int w = 0; w < 8; w++) q += qred[w * SG_T + c];
            double dl = -INFINITY;
            int gi = 0x7fffffff;
            const bool valid = c0 + c < nc;
            if (valid) {
                const double s = 1.0 + eta - q;
                gi = cand_idx[(size_t)b * nc + c0 + c];
                if (s > kSMin) {
                    const double kap = corr_from_d2(sqdist_fma(xcs + c * p, xq, p), rtheta);
                    const double cov = kap - cvred[c];
                    dl = cov * cov / s;
                }
                if (delta_out) delta_out[(size_t)b * nc + c0 + c] = dl;
            }
            if (valid && dl > -INFINITY) t2.push(dl, gi, c0 + c);
        }
        warp_merge_top2(t2);
        if (lane == 0) {
            double *pp = part + ((size_t)b * gridDim.x + blockIdx.x) * 4;
            pp[0] = t2.d1;
            pp[1] = t2.d2;
            pp[2] = int_bits_to_double(t2.i1);
            pp[3] = int_bits_to_double(t2.pos);
        }
    }
}

// per location: merge the per-CTA top-2 records
__global__ void __launch_bounds__(SG_THREADS)
alc_scores_merge_kernel(int nblk, const double *__restrict__ part, int32_t *__restrict__ best_out,
                        double *__restrict__ gap_out) {
    __shared__ double red[160];
    const int b = blockIdx.x;
    Top2 t;
    t.init();
    for (int k = threadIdx.x; k < nblk; k += SG_THREADS) {
        const double *pp = part + ((size_t)b * nblk + k) * 4;
        if (pp[0] > -INFINITY) t.merge(pp[0], double_bits_to_int(pp[2]), double_bits_to_int(pp[3]), pp[1]);
    }
    t = block_top2(t, red);
    if (threadIdx.x == 0) {
        best_out[b] = t.pos;
        if (gap_out) gap_out[b] = (t.pos >= 0) ? top2_gap(t.d1, t.d2) : __longlong_as_double(0x7ff8000000000000LL);
    }
}

static int sg_tile(int j) {
    (void)j;
    return 32;  // measured: T = 64 (fewer CTAs per SM, 95 registers) is 1.3-1.6x slower at n = 208-336
}

static size_t sg_smem(int j, int T, bool stage) {
    const int jr = (j + 7) & ~7;
    return ((size_t)jr * sg_tl(T) + (size_t)T * LAGP_PMAX + 8 * (size_t)T + T + (stage ? 8 * (size_t)SG_ABUF : 0)) *
           sizeof(double);
}
// K^{-1} staging for j >= 384 (one CTA per SM either way: the copies hide the L2
// latency) while the tile plus the chunk buffers fit (j <= 640 at T = 32); below 384
// the 37 KB of buffers would cost resident CTAs (measured 8-15 % slower at 208-336)
static bool sg_stage(int j) { return j >= 384 && sg_smem(j, 32, true) <= 227 * 1024; }

size_t alc_scores_gemm_smem(int j, int p) {
    (void)p;
    return sg_smem(j, sg_tile(j), sg_stage(j));
}

size_t alc_scores_gemm_ws_bytes(int B, int j, int nc) {
    const int wl = (j + 3) & ~3;
    const int T = sg_tile(j);
    const int nblk = (nc + T - 1) / T;
    return ((size_t)B * wl + (size_t)B * nblk * 4) * sizeof(double);
}

template <int T, bool STAGE>
static cudaError_t sg_launch(int B, int j, int p, int nc, const double *Xj, const double *Kinv, const double *cands,
                             const int32_t *cand_idx, const double *x, double rtheta, double eta, const double *wv,
                             int wl, double *delta, double *part, cudaStream_t st) {
    const size_t smem = sg_smem(j, T, STAGE);
    cudaError_t e =
        cudaFuncSetAttribute(alc_scores_gemm_kernel<T, STAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int nblk = (nc + T - 1) / T;
    alc_scores_gemm_kernel<T, STAGE><<<dim3(nblk, B), SG_THREADS, smem, st>>>(j, p, nc, Xj, Kinv, cands, cand_idx, x, rtheta,
                                                                       eta, wv, wl, delta, part);
    return cudaGetLastError();
}

cudaError_t launch_alc_scores_gemm(int B, int j, int p, int nc, const double *Xj, const double *Kinv,
                                   const double *cands, const int32_t *cand_idx, const double *x, double rtheta,
                                   double eta, double *delta, int32_t *best, double *gap, void *ws, cudaStream_t st,
                                   int *launches) {
    const int wl = (j + 3) & ~3;
    const int T = sg_tile(j);
    const int nblk = (nc + T - 1) / T;
    double *wv = static_cast<double *>(ws);
    double *part = wv + (size_t)B * wl;
    const size_t sp = (size_t)j * sizeof(double);
    alc_scores_prep_kernel<<<B, SG_THREADS, sp, st>>>(j, p, Xj, Kinv, x, rtheta, wv, wl);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (T == 64)
        e = sg_launch<64, false>(B, j, p, nc, Xj, Kinv, cands, cand_idx, x, rtheta, eta, wv, wl, delta, part, st);
    else if (sg_stage(j))
        e = sg_launch<32, true>(B, j, p, nc, Xj, Kinv, cands, cand_idx, x, rtheta, eta, wv, wl, delta, part, st);
    else
        e = sg_launch<32, false>(B, j, p, nc, Xj, Kinv, cands, cand_idx, x, rtheta, eta, wv, wl, delta, part, st);
    if (e != cudaSuccess) return e;
    alc_scores_merge_kernel<<<B, SG_THREADS, 0, st>>>(nblk, part, best, gap);
    if (launches) *launches += 3;
    return cudaGetLastError();
}

}  // namespace lagp
