// TMEM -> register bandwidth and latency with tcgen05.ld.32x32b (thread-private
// lane rows), alone and concurrently with shared-memory LDS.128 streaming: can
// TMEM serve as extra per-thread storage for the incremental kernel's w_c entries?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tmem_bw scripts/tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

template <int NX, bool WITH_SMEM, bool WITH_TMEM>
__global__ void __launch_bounds__(512, 1) tmem_bw(unsigned *out, long long *cyc) {
    __shared__ uint32_t taddr;
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, wid = tid >> 5;
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&taddr)),
                     "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    for (int i = tid; i < 96 * 1024 / 8; i += 512) sm[i] = i;
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t base = taddr;
    // warp w: lanes 32*(w%4).., columns (w/4)*128 ..
    const uint32_t a0 = base + ((uint32_t)(32 * (wid & 3)) << 16) + (uint32_t)((wid >> 2) * 128);
    unsigned acc = 0;
    double dacc = 0;
    const double2 *s2 = reinterpret_cast<const double2 *>(sm);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
        if (WITH_TMEM) {
            const uint32_t a = a0 + (uint32_t)((it * NX) & 127);
            uint32_t r[NX];
            if (NX == 4) {
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                             : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                             : "r"(a));
            } else {
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                      "=r"(r[7])
                    : "r"(a));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < NX; k++) acc += r[k];
        }
        if (WITH_SMEM) {
            const double2 v = s2[((it * 512 + tid) & (96 * 1024 / 16 - 1))];
            dacc += v.x + v.y;
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * 512 + tid] = acc + (unsigned)dacc;
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    __syncthreads();
    if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "n"(512));
}

template <int NX, bool S, bool T>
void run(const char *name) {
    unsigned *out;
    long long *cyc, h;
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&cyc, 148 * 8);
    cudaFuncSetAttribute(tmem_bw<NX, S, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    tmem_bw<NX, S, T><<<148, 512, 96 * 1024>>>(out, cyc);
    tmem_bw<NX, S, T><<<148, 512, 96 * 1024>>>(out, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double tb = T ? 512.0 * NX * 4 * ITERS : 0, sb = S ? 512.0 * 16 * ITERS : 0;
    printf("{\"case\": \"%s\", \"err\": \"%s\", \"cycles\": %lld, \"tmem_B_per_clk\": %.1f, \"smem_B_per_clk\": %.1f}\n",
           name, cudaGetErrorString(e), h, tb / h, sb / h);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run<4, false, true>("tmem x4 (16 B/thread per ld)");
    run<8, false, true>("tmem x8 (32 B/thread per ld)");
    run<4, true, false>("smem LDS.128 alone");
    run<4, true, true>("tmem x4 + smem LDS.128");
    run<8, true, true>("tmem x8 + smem LDS.128");
    return 0;
}
