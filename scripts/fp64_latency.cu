// Dependent-chain latency and single-warp throughput of the FP64 instructions the
// local-design kernels use (DFMA, DADD, DMUL, FRND.F64, F2I.F64, MUFU.RCP64H, LDS).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/fp64_latency scripts/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int OP, int CHAINS>
__global__ void chain(double *out, long long *cyc, double seed) {
    double v[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; c++) v[c] = seed + threadIdx.x * 1e-9 + c * 1e-7;
    __syncwarp();
    long long t0 = clock64();
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int c = 0; c < CHAINS; c++) {
            if (OP == 0) v[c] = fma(v[c], 0.999999, 1e-9);
            if (OP == 1) v[c] = v[c] + 1e-9;
            if (OP == 2) v[c] = v[c] * 0.9999999;
            if (OP == 3) v[c] = rint(v[c]) + 0.25;
            if (OP == 4) v[c] = (double)(int)v[c] + 0.25;
            if (OP == 5) {
                double r;
                asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v[c]));
                v[c] = r;
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) s += v[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP, int CHAINS>
void run(const char *name, int warps) {
    double *out;
    long long *cyc, h;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&cyc, 8);
    chain<OP, CHAINS><<<1, 32 * warps>>>(out, cyc, 1.5);
    chain<OP, CHAINS><<<1, 32 * warps>>>(out, cyc, 1.5);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double per = (double)h / ITERS;
    printf("{\"op\": \"%s\", \"chains\": %d, \"warps_per_cta\": %d, \"cycles_per_iter\": %.2f, "
           "\"cycles_per_op_per_chain\": %.2f}\n",
           name, CHAINS, warps, per, per / 1.0);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    // latency: 1 chain, 1 warp; throughput: 8 chains x 4 warps (one SMSP each) / 16 warps
    run<0, 1>("DFMA", 1);
    run<1, 1>("DADD", 1);
    run<2, 1>("DMUL", 1);
    run<3, 1>("FRND.F64+DADD", 1);
    run<4, 1>("F2I.F64+I2F.F64+DADD", 1);
    run<5, 1>("MUFU.RCP64H", 1);
    run<0, 8>("DFMA", 1);
    run<0, 8>("DFMA", 4);
    run<0, 8>("DFMA", 16);
    run<3, 8>("FRND.F64+DADD", 4);
    run<4, 8>("F2I.F64+I2F.F64+DADD", 4);
    run<5, 8>("MUFU.RCP64H", 4);
    return 0;
}
