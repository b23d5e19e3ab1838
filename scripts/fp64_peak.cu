// fp64_peak.cu — measured FP64 ceilings on this B200 (the ALU roofline
// denominator for the ALC kernels, which are FP64-pipe bound):
//   dfma : independent DFMA chains, 148 SMs × full occupancy
//   dmma : mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 (legacy FP64 tensor path, SASS DMMA)
//   exp  : double exp() throughput (evaluations/s)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 16; u++) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma_kernel(double *out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-3, b = 0.5;
    double c[4][2] = {};
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 4; u++) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[u][0]), "+d"(c[u][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0;
    for (int u = 0; u < 4; u++) s += c[u][0] + c[u][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void exp_kernel(double *out, int iters) {
    double x = -1e-3 * threadIdx.x, acc = 0.0;
    for (int i = 0; i < iters; i++) {
        acc += exp(x);
        x -= 1e-7;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double *out;
    const int threads = 256, blocks = sms * 8;
    cudaMalloc(&out, (size_t)blocks * threads * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    // warm
    dfma_kernel<<<blocks, threads>>>(out, 100, 0.999, 1e-3);
    cudaDeviceSynchronize();
    int it = 20000;
    double best_dfma = 0;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, it, 0.999, 1e-3);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 8 * 16 * (double)it * blocks * threads;
        if (fl / (ms * 1e-3) > best_dfma) best_dfma = fl / (ms * 1e-3);
    }
    double best_dmma = 0;
    int itm = 20000;
    dmma_kernel<<<blocks, threads>>>(out, 100);
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        dmma_kernel<<<blocks, threads>>>(out, itm);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        // each warp-level mma = 8*8*4 FMA = 512 flop; 4 per iter per warp
        double fl = 512.0 * 4 * (double)itm * blocks * (threads / 32);
        if (fl / (ms * 1e-3) > best_dmma) best_dmma = fl / (ms * 1e-3);
    }
    double best_exp = 0;
    int ite = 4000;
    exp_kernel<<<blocks, threads>>>(out, 10);
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        exp_kernel<<<blocks, threads>>>(out, ite);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double ev = (double)ite * blocks * threads;
        if (ev / (ms * 1e-3) > best_exp) best_exp = ev / (ms * 1e-3);
    }
    printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"exp_geval_s\": %.3f}\n",
           sms, clk, best_dfma / 1e12, best_dmma / 1e12, best_exp / 1e9);
    return 0;
}
