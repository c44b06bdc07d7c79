// k_reduce.cu -- K5: per-level accumulators of Algorithm 2 (steps 5-6).
//
// From the per-sample records (Q_f, Q_c, iterations, residuals, status) form
// Y = Q_f - Q_c (Y = Q_f on level 0) and accumulate sum Y, sum Y^2
// (for hat Y_l and s_l^2 of Eq. (3)/(4)), sum Q_f, sum Q_c, the deterministic
// cost model C_l (R5), counts, failures and iteration statistics.
// Deterministic: fixed 4096-sample chunks, a fixed per-thread stride and xor
// butterflies inside a chunk, then the chunk partials added in chunk order.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "internal.h"

namespace mlmc {

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double wmax(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

constexpr int RT = 256;

__global__ void __launch_bounds__(RT) chunk_sums_kernel(const double* __restrict__ rec, uint64_t nb, int level,
                                                        double n_f, double n_c, double cff, double cfs,
                                                        double ccf, double ccs, double* __restrict__ partial) {
    const uint64_t c0 = blockIdx.x * kChunk;
    double v[kSumsLen];
#pragma unroll
    for (int k = 0; k < kSumsLen; ++k) v[k] = 0.0;
    for (uint64_t s = c0 + threadIdx.x; s < c0 + kChunk && s < nb; s += RT) {
        const double* r = rec + s * kRecLen;
        const double qf = r[0], qc = level > 0 ? r[1] : 0.0;
        const double y = qf - qc;
        const double itf = r[2], itc = level > 0 ? r[3] : 0.0;
        // status 4 = converged after escalation (a failed MINRES solve re-solved by MG-PCG): a success
        const bool fail = (r[6] != 0.0 && r[6] != 4.0) || (level > 0 && r[7] != 0.0 && r[7] != 4.0);
        const bool esc = r[6] == 4.0 || (level > 0 && r[7] == 4.0);
        v[0] += y;
        v[1] = fma(y, y, v[1]);
        v[2] += qf;
        v[3] += qc;
        v[4] += (cff + cfs * itf) + (level > 0 ? (ccf + ccs * itc) : 0.0);
        v[5] += 1.0;
        v[6] += fail ? 1.0 : 0.0;
        v[7] += itf;
        v[8] += itc;
        v[9] = fmax(v[9], itf);
        v[10] = fmax(v[10], itc);
        v[11] += esc ? 1.0 : 0.0;
    }
    __shared__ double sh[RT / 32][kSumsLen];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < kSumsLen; ++k) {
        double t = (k == 9 || k == 10) ? wmax(v[k]) : wsum(v[k]);
        if (lane == 0) sh[wid][k] = t;
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int k = 0; k < kSumsLen; ++k) {
            double t = lane < RT / 32 ? sh[lane][k] : 0.0;
            t = (k == 9 || k == 10) ? wmax(t) : wsum(t);
            if (lane == 0) partial[blockIdx.x * kSumsLen + k] = t;
        }
    }
}

// escalation (R15 / SURVEY A15): the indices of the samples whose solve of record slot `slot` failed
// (status 1-3), appended to list (order irrelevant: every listed system is re-solved independently)
__global__ void escalate_collect_kernel(const double* __restrict__ rec, uint64_t nb, int slot, int* __restrict__ list,
                                        int* __restrict__ count) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < nb; s += (uint64_t)gridDim.x * blockDim.x) {
        const double st = rec[s * kRecLen + 6 + slot];
        if (st != 0.0 && st != 4.0) list[atomicAdd(count, 1)] = (int)s;
    }
}

cudaError_t launch_escalate_collect(const double* rec, uint64_t nb, int slot, int* list, int* count, cudaStream_t s) {
    if (nb == 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<uint64_t>((nb + 255) / 256, 148ull * 8);
    escalate_collect_kernel<<<grid, 256, 0, s>>>(rec, nb, slot, list, count);
    return cudaGetLastError();
}

__global__ void combine_chunks_kernel(const double* __restrict__ partial, int nchunks, double* __restrict__ sums,
                                      int accumulate) {
    const int k = threadIdx.x;
    if (k >= kSumsLen) return;
    const bool isMax = (k == 9 || k == 10);
    double t = accumulate ? sums[k] : 0.0;
    for (int c = 0; c < nchunks; ++c) {
        double p = partial[c * kSumsLen + k];
        t = isMax ? fmax(t, p) : t + p;
    }
    sums[k] = t;
}

cudaError_t launch_level_sums(const double* rec, uint64_t nb, int level, double n_f, double n_c,
                              double cost_f_fixed, double cost_f_step, double cost_c_fixed, double cost_c_step,
                              double* chunk_scratch, double* sums, bool accumulate, cudaStream_t s) {
    const int nchunks = (int)((nb + kChunk - 1) / kChunk);
    if (nchunks > 0)
        chunk_sums_kernel<<<nchunks, RT, 0, s>>>(rec, nb, level, n_f, n_c, cost_f_fixed, cost_f_step,
                                                  cost_c_fixed, cost_c_step, chunk_scratch);
    combine_chunks_kernel<<<1, 32, 0, s>>>(chunk_scratch, nchunks, sums, accumulate ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace mlmc
