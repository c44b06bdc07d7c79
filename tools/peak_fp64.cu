// peak_fp64.cu -- microbenchmark of the FP64 pipes on this GPU (the roofline
// denominators the resident kernels are judged against; MEASURED_PEAKS.json has
// no FP64 entry).  DFMA: 8 independent chains per thread; DMMA m8n8k4: 4
// independent accumulators per warp.  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma_kernel(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0;
    for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out; cudaMalloc(&out, sizeof(double) * sms * 16 * 1024);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = sms * 4, threads = 512, iters = 4096;
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (r) best = ms < best ? ms : best;
    }
    double dfma_tf = 2.0 * blocks * threads * (double)iters * 16 * 8 / (best * 1e-3) / 1e12;
    float bestm = 1e30f;
    const int iters2 = 2048;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        dmma_kernel<<<blocks, threads>>>(out, iters2);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (r) bestm = ms < bestm ? ms : bestm;
    }
    double warps = blocks * threads / 32.0;
    double dmma_tf = 2.0 * 256.0 * warps * (double)iters2 * 16 / (bestm * 1e-3) / 1e12;
    printf("{\"fp64_fma_tflops\": %.3f, \"fp64_dmma_tflops\": %.3f, \"sms\": %d, \"clock_mhz_attr\": %d, \"dfma_ms\": %.3f, \"dmma_ms\": %.3f}\n",
           dfma_tf, dmma_tf, sms, clk / 1000, best, bestm);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    return 0;
}
