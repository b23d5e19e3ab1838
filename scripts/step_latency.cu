// Latencies of the operations on the incremental kernel's per-step critical path:
// MUFU.RCP64H / RSQ64H (+ the Newton DFMAs), redux.sync (CREDUX), a dependent LDS
// chain, bar.sync with 8 / 16 warps, tcgen05.ld + wait::ld, a shared-memory flag
// handoff between two warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/step_latency scripts/step_latency.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int IT = 2048;

__global__ void k_rcp(double *out, long long *cyc, double s) {
    double v = s + threadIdx.x * 1e-12;
    long long t0 = clock64();
    for (int i = 0; i < IT; i++) {
        double r;
        asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v));
        v = r + 1.0;
    }
    long long t1 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_rsq(double *out, long long *cyc, double s) {
    double v = s + threadIdx.x * 1e-12;
    long long t0 = clock64();
    for (int i = 0; i < IT; i++) {
        double r;
        asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v));
        v = r + 1.0;
    }
    long long t1 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dadd(double *out, long long *cyc, double s) {
    double v = s + threadIdx.x * 1e-12;
    long long t0 = clock64();
    for (int i = 0; i < IT; i++) {
        asm volatile("add.rn.f64 %0, %0, 1.0;" : "+d"(v));
        asm volatile("add.rn.f64 %0, %0, 1.0;" : "+d"(v));
    }
    long long t1 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_redux(double *out, long long *cyc, unsigned s) {
    unsigned v = s + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < IT; i++) v = __reduce_max_sync(0xffffffffu, v ^ threadIdx.x) + 1u;
    long long t1 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds(double *out, long long *cyc, int s) {
    __shared__ int buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i + 1 + s) & 1023;
    __syncthreads();
    int p = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < IT; i++) p = buf[p];
    long long t1 = clock64();
    out[threadIdx.x] = p;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_bar(double *out, long long *cyc, int s) {
    long long t0 = clock64();
    for (int i = 0; i < IT; i++) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_tmem(double *out, long long *cyc, int s) {
    __shared__ uint32_t taddr;
    const int wid = threadIdx.x >> 5;
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&taddr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tb = taddr + ((uint32_t)(32 * (wid & 3)) << 16);
    uint32_t acc = s;
    long long t0 = clock64();
    for (int i = 0; i < IT; i++) {
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(tb + (acc & 8)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        acc += r[0] + r[7];
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(taddr));
}
// warp 0 and warp 1 hand a token back and forth through a volatile shared flag
__global__ void k_flag(double *out, long long *cyc, int s) {
    __shared__ volatile int flag;
    if (threadIdx.x == 0) flag = 0;
    __syncthreads();
    const int wid = threadIdx.x >> 5;
    long long t0 = clock64();
    for (int i = 0; i < IT; i++) {
        if (wid == (i & 1)) {
            while (flag != i) {
            }
            __threadfence_block();
            if ((threadIdx.x & 31) == 0) flag = i + 1;
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <typename K>
void run(const char *name, K k, int threads, int per) {
    double *out;
    long long *cyc, h;
    cudaMalloc(&out, 1 << 16);
    cudaMalloc(&cyc, 8);
    k<<<1, threads>>>(out, cyc, 1);
    k<<<1, threads>>>(out, cyc, 1);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"op\": \"%s\", \"threads\": %d, \"cycles_per_op\": %.1f, \"err\": \"%s\"}\n", name, threads,
           (double)h / IT / per, cudaGetErrorString(e));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run("rcp.approx.f64 + DADD (dependent)", k_rcp, 32, 1);
    run("rcp.approx.f64 + DADD, 16 warps", k_rcp, 512, 1);
    run("rsqrt.approx.f64 + DADD (dependent)", k_rsq, 32, 1);
    run("DADD (dependent)", k_dadd, 32, 2);
    run("redux.sync.max + IADD (dependent)", k_redux, 32, 1);
    run("redux.sync.max, 16 warps", k_redux, 512, 1);
    run("LDS (dependent)", k_lds, 32, 1);
    run("bar.sync, 8 warps", k_bar, 256, 1);
    run("bar.sync, 16 warps", k_bar, 512, 1);
    run("tcgen05.ld.x8 + wait::ld (dependent)", k_tmem, 32, 1);
    run("tcgen05.ld.x8 + wait::ld, 8 warps", k_tmem, 256, 1);
    run("shared flag handoff (per handoff)", k_flag, 64, 1);
    return 0;
}
