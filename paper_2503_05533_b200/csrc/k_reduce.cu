// k_reduce.cu -- K5: per-level accumulators of Algorithm 2 (steps 5-6).
//
// From the per-sample records (Q_f, Q_c, iterations, residuals, status) form
// Y = Q_f - Q_c (Y = Q_f on level 0) and accumulate sum Y, sum Y^2
// (for hat Y_l and s_l^2 of Eq. (3)/(4)), sum Q_f, sum Q_c, the deterministic
// cost model C_l (R5), counts, failures and iteration statistics.
// Deterministic: fixed 4096-sample chunks, a fixed per-thread stride and xor
// butterflies inside a chunk, then the chunk partials added in chunk order.  The
// five real-valued sums are also formed exactly in 256-bit fixed point (internal.h
// kX*), which the adaptive controller exchanges across ranks so that its sums and
// decisions are bit-identical for any number of ranks.
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

constexpr int RT = 512;   // threads per chunk CTA (8 samples each): 8.3 vs 10.9 us per launch with 256 on configs[1]
using u64 = unsigned long long;

// ---- exact fixed-point sums (internal.h kX*): 256-bit two's-complement integers in units of 2^-kXScale
struct X256 {
    u64 w[4];
};
__device__ __forceinline__ void x_add(X256& a, const X256& b) {
    asm("add.cc.u64 %0, %0, %4;\n\taddc.cc.u64 %1, %1, %5;\n\taddc.cc.u64 %2, %2, %6;\n\taddc.u64 %3, %3, %7;"
        : "+l"(a.w[0]), "+l"(a.w[1]), "+l"(a.w[2]), "+l"(a.w[3])
        : "l"(b.w[0]), "l"(b.w[1]), "l"(b.w[2]), "l"(b.w[3]));
}
// x rounded once (to nearest even) to a multiple of 2^-kXScale, added to a; |x| >= 2^62 and non-finite
// values are counted in ovf instead
__device__ __forceinline__ void x_acc(X256& a, u64& ovf, double x) {
    if (x == 0.0) return;
    if (!(fabs(x) < 0x1p62)) { ++ovf; return; }
    const double X = scalbn(x, kXScale);   // exact: a power-of-two scaling without overflow
    X256 v;
    if (fabs(X) < 0x1p62) {
        const long long i = __double2ll_rn(X);
        v.w[0] = (u64)i;
        v.w[1] = v.w[2] = v.w[3] = i < 0 ? ~0ull : 0ull;
    } else {   // |X| = m 2^k with a 53-bit integer m and k >= 10: already an integer
        int e;
        const double f = frexp(fabs(X), &e);
        const u64 m = (u64)(f * 0x1p53);
        const int k = e - 53, q = k >> 6, r = k & 63;
        const u64 lo = m << r, hi = r ? m >> (64 - r) : 0ull;
#pragma unroll
        for (int i = 0; i < 4; ++i) v.w[i] = q == i ? lo : (q + 1 == i ? hi : 0ull);
        if (x < 0.0) {   // two's complement
            X256 one{{1ull, 0ull, 0ull, 0ull}};
#pragma unroll
            for (int i = 0; i < 4; ++i) v.w[i] = ~v.w[i];
            x_add(v, one);
        }
    }
    x_add(a, v);
}
__device__ __forceinline__ void x_warp(X256& a, u64& ovf) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        X256 b;
#pragma unroll
        for (int i = 0; i < 4; ++i) b.w[i] = __shfl_xor_sync(0xffffffffu, a.w[i], o);
        ovf += __shfl_xor_sync(0xffffffffu, ovf, o);
        x_add(a, b);
    }
}

__global__ void __launch_bounds__(RT) chunk_sums_kernel(const double* __restrict__ rec, uint64_t nb, int level,
                                                        const CostParams cp, double* __restrict__ partial,
                                                        u64* __restrict__ xpart) {
    const uint64_t c0 = blockIdx.x * kChunk;
    double v[kSumsLen];
#pragma unroll
    for (int k = 0; k < kSumsLen; ++k) v[k] = 0.0;
    X256 xs[kXFields];
    u64 xo[kXFields];
#pragma unroll
    for (int f = 0; f < kXFields; ++f) {
        xs[f] = X256{{0ull, 0ull, 0ull, 0ull}};
        xo[f] = 0ull;
    }
    for (uint64_t s = c0 + threadIdx.x; s < c0 + kChunk && s < nb; s += RT) {
        const double* r = rec + s * kRecLen;
        const double qf = r[0], qc = level > 0 ? r[1] : 0.0;
        const double y = qf - qc;
        const double itf = r[2], itc = level > 0 ? r[3] : 0.0;
        // status 4 = converged after escalation (a failed MINRES solve re-solved by MG-PCG): a success
        const bool fail = (r[6] != 0.0 && r[6] != 4.0) || (level > 0 && r[7] != 0.0 && r[7] != 4.0);
        const bool esc = r[6] == 4.0 || (level > 0 && r[7] == 4.0);
        // cost model (R5): fixed + step x iterations; an escalated half (status 4) is charged the failed first
        // attempt plus the MG-PCG re-solve, whose steps the record holds
        const double cf = r[6] == 4.0 ? cp.f_esc + cp.f_esc_step * itf : cp.f_fixed + cp.f_step * itf;
        const double cc = level > 0 ? (r[7] == 4.0 ? cp.c_esc + cp.c_esc_step * itc : cp.c_fixed + cp.c_step * itc) : 0.0;
        const double cost = cf + cc;
        v[0] += y;
        v[1] = fma(y, y, v[1]);
        v[2] += qf;
        v[3] += qc;
        v[4] += cost;
        if (xpart) {
            x_acc(xs[0], xo[0], y);
            x_acc(xs[1], xo[1], y * y);
            x_acc(xs[2], xo[2], qf);
            x_acc(xs[3], xo[3], qc);
            x_acc(xs[4], xo[4], cost);
        }
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
    if (!xpart) return;   // uniform
    __shared__ u64 shx[RT / 32][kXLen];
#pragma unroll
    for (int f = 0; f < kXFields; ++f) {
        x_warp(xs[f], xo[f]);
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) shx[wid][f * kXWords + i] = xs[f].w[i];
            shx[wid][f * kXWords + 4] = xo[f];
        }
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int f = 0; f < kXFields; ++f) {
            X256 a{{0ull, 0ull, 0ull, 0ull}};
            u64 o = 0ull;
            if (lane < RT / 32) {
#pragma unroll
                for (int i = 0; i < 4; ++i) a.w[i] = shx[lane][f * kXWords + i];
                o = shx[lane][f * kXWords + 4];
            }
            x_warp(a, o);
            if (lane == 0) {
#pragma unroll
                for (int i = 0; i < 4; ++i) xpart[(size_t)blockIdx.x * kXLen + f * kXWords + i] = a.w[i];
                xpart[(size_t)blockIdx.x * kXLen + f * kXWords + 4] = o;
            }
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
                                      int accumulate, const u64* __restrict__ xpart, u64* __restrict__ xsums) {
    const int k = threadIdx.x;
    if (xsums && k < kXFields) {
        X256 a{{0ull, 0ull, 0ull, 0ull}};
        u64 o = 0ull;
        if (accumulate) {
#pragma unroll
            for (int i = 0; i < 4; ++i) a.w[i] = xsums[k * kXWords + i];
            o = xsums[k * kXWords + 4];
        }
        for (int c = 0; c < nchunks; ++c) {
            X256 b;
#pragma unroll
            for (int i = 0; i < 4; ++i) b.w[i] = xpart[(size_t)c * kXLen + k * kXWords + i];
            o += xpart[(size_t)c * kXLen + k * kXWords + 4];
            x_add(a, b);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) xsums[k * kXWords + i] = a.w[i];
        xsums[k * kXWords + 4] = o;
    }
    if (k >= kSumsLen) return;
    const bool isMax = (k == 9 || k == 10);
    double t = accumulate ? sums[k] : 0.0;
    for (int c = 0; c < nchunks; ++c) {
        double p = partial[c * kSumsLen + k];
        t = isMax ? fmax(t, p) : t + p;
    }
    sums[k] = t;
}

cudaError_t launch_level_sums(const double* rec, uint64_t nb, int level, const CostParams& cp, double* chunk_scratch,
                              double* sums, bool accumulate, cudaStream_t s, u64* xsums) {
    const int nchunks = (int)((nb + kChunk - 1) / kChunk);
    u64* xpart = xsums ? reinterpret_cast<u64*>(chunk_scratch + (size_t)kSumsLen * nchunks) : nullptr;
    if (nchunks > 0)
        chunk_sums_kernel<<<nchunks, RT, 0, s>>>(rec, nb, level, cp, chunk_scratch, xpart);
    combine_chunks_kernel<<<1, 32, 0, s>>>(chunk_scratch, nchunks, sums, accumulate ? 1 : 0, xpart, xsums);
    return cudaGetLastError();
}

}  // namespace mlmc
