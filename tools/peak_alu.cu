// peak_alu.cu -- microbenchmark of the ALU pipes the resident kernels are bound by
// (MEASURED_PEAKS.json holds only HBM copy and bf16 GEMM figures).  Measures, on
// all SMs, with CUDA events (best of 5 after one warm-up launch, each ~10-50 ms):
//   DFMA   fp64 FMA, 8 independent chains per thread       -> fp64_fma_tflops   (K3, K3m: FP64 ALU)
//   DMMA   mma.sync m8n8k4 f64, 4 accumulators per warp    -> fp64_dmma_tflops  (K1 field synthesis)
//   FFMA   fp32 FMA, 8 independent chains per thread       -> fp32_fma_tflops   (K4 fp32/E4M3 factor)
//   HFMA2  packed fp16 FMA, 8 chains per thread            -> fp16x2_fma_tflops (K4 fp16 arithmetic)
// plus a "sustained" DFMA figure: back-to-back launches for ~2 s.  Prints one JSON line;
// tools/gpu_peaks.sh records the SM clocks while it runs.
#include <cstdio>
#include <cuda_fp16.h>
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

__global__ void ffma_kernel(double* out, int iters, float a, float b) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void hfma2_kernel(double* out, int iters, float af, float bf) {
    __half2 a = __float2half2_rn(af), b = __float2half2_rn(bf);
    __half2 x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = __float2half2_rn(1e-3f * (threadIdx.x + q));
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int q = 0; q < 8; ++q) x[q] = __hfma2(x[q], a, b);
        }
    }
    float s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += __low2float(x[q]) + __high2float(x[q]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
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

template <class F>
static float best_ms(F launch, int reps = 5) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    launch();  // warm-up
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    return best;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out; cudaMalloc(&out, sizeof(double) * sms * 16 * 1024);
    const int blocks = sms * 4, threads = 512;
    const double thr = (double)blocks * threads;
    const int it_d = 4096, it_f = 8192, it_h = 8192, it_m = 2048;
    float t_d = best_ms([&] { dfma_kernel<<<blocks, threads>>>(out, it_d, 0.999999, 1e-7); });
    float t_f = best_ms([&] { ffma_kernel<<<blocks, threads>>>(out, it_f, 0.999999f, 1e-7f); });
    float t_h = best_ms([&] { hfma2_kernel<<<blocks, threads>>>(out, it_h, 0.999f, 1e-4f); });
    float t_m = best_ms([&] { dmma_kernel<<<blocks, threads>>>(out, it_m); });
    double dfma = 2.0 * thr * it_d * 16 * 8 / (t_d * 1e-3) / 1e12;
    double ffma = 2.0 * thr * it_f * 16 * 8 / (t_f * 1e-3) / 1e12;
    double hfma2 = 4.0 * thr * it_h * 16 * 8 / (t_h * 1e-3) / 1e12;   // 2 lanes x 2 flops
    double dmma = 2.0 * 256.0 * (thr / 32.0) * it_m * 16 / (t_m * 1e-3) / 1e12;
    // sustained DFMA: back-to-back launches for ~2 s, mean per launch
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    int reps = (int)(2000.0f / t_d) + 1;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) dfma_kernel<<<blocks, threads>>>(out, it_d, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float tot; cudaEventElapsedTime(&tot, e0, e1);
    double dfma_sus = 2.0 * thr * it_d * 16 * 8 * reps / (tot * 1e-3) / 1e12;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; }
    printf("{\"fp64_fma_tflops\": %.3f, \"fp64_fma_tflops_sustained\": %.3f, \"fp64_dmma_tflops\": %.3f, "
           "\"fp32_fma_tflops\": %.3f, \"fp16x2_fma_tflops\": %.3f, \"sms\": %d, \"clock_mhz_attr\": %d, "
           "\"ms\": {\"dfma\": %.3f, \"dmma\": %.3f, \"ffma\": %.3f, \"hfma2\": %.3f, \"dfma_sustained_total\": %.1f}}\n",
           dfma, dfma_sus, dmma, ffma, hfma2, sms, clk / 1000, t_d, t_m, t_f, t_h, tot);
    return 0;
}
