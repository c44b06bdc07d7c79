// k_field.cu -- K0 (counter-based normals) and K1+K2 (KL synthesis + exp).
//
// K0: xi ~ N(0,1)^m per sample from Philox4x32-10 keyed by the seed, counter
//     (t, index_lo, index_hi, level), Box-Muller on 53-bit uniforms (R12).
//     The paper draws omega_j ~ N(0, sigma^2); the variance is folded
//     into the synthesis matrix Phi.
// K1+K2: log a at the 2N^2 triangle centroids is the dense contraction
//     G[b][p] = sum_k xi[b][k] Phi[p][k]   (truncated KL)
//     followed by a = exp(G) (lognormal coefficient).  All binary64
//     ("apart from the linear solver, all calculations ... in double").
//     Register-tiled FFMA64: a 64(b) x 64(p) output tile per 256-thread CTA,
//     4x4 outputs per thread, k staged through shared memory in chunks of 16.
#include <cuda_runtime.h>
#include <algorithm>
#include <cfloat>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace mlmc {

__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                             uint32_t k0, uint32_t k1) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
    uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
}

__device__ __forceinline__ void philox10(uint32_t ctr[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        philox_round(ctr[0], ctr[1], ctr[2], ctr[3], k0, k1);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

__global__ void rng_kernel(double* __restrict__ xi, int m, uint64_t nb, uint64_t seed, int level,
                           uint64_t first_index) {
    const int pairs = (m + 1) / 2;
    const uint64_t total = nb * (uint64_t)pairs;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
         g += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t b = g / pairs;
        int t = (int)(g - b * pairs);
        uint64_t idx = first_index + b;
        uint32_t ctr[4] = {(uint32_t)t, (uint32_t)idx, (uint32_t)(idx >> 32), (uint32_t)level};
        philox10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32));
        const double two53inv = 1.0 / 9007199254740992.0;
        double u1 = (fma((double)(ctr[0] >> 5), 67108864.0, (double)(ctr[1] >> 6)) + 0.5) * two53inv;
        double u2 = (fma((double)(ctr[2] >> 5), 67108864.0, (double)(ctr[3] >> 6)) + 0.5) * two53inv;
        double rad = sqrt(-2.0 * log(u1));
        double s, c;
        sincospi(2.0 * u2, &s, &c);
        double* o = xi + b * (uint64_t)m;
        o[2 * t] = rad * c;
        if (2 * t + 1 < m) o[2 * t + 1] = rad * s;
    }
}

cudaError_t launch_rng(double* xi, int m, uint64_t nb, uint64_t seed, int level, uint64_t first_index,
                       cudaStream_t s) {
    if (nb == 0) return cudaSuccess;
    uint64_t total = nb * (uint64_t)((m + 1) / 2);
    unsigned grid = (unsigned)std::min<uint64_t>((total + 255) / 256, 148ull * 16);
    rng_kernel<<<grid, 256, 0, s>>>(xi, m, nb, seed, level, first_index);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------- K1 + K2
constexpr int FT_B = 64, FT_P = 64, FT_K = 16;

// Per-sample contrast keys (optional): keys[2b] = max a, keys[2b+1] = ~min a as u64 bit patterns
// (order-preserving for positive doubles), combined with atomicMax.
__device__ __forceinline__ void key_update(unsigned long long* keys, int b, double mx, double mn) {
    atomicMax(keys + 2 * b, (unsigned long long)__double_as_longlong(mx));
    atomicMax(keys + 2 * b + 1, ~(unsigned long long)__double_as_longlong(mn));
}

__global__ void __launch_bounds__(256) field_kernel(const double* __restrict__ phi, const double* __restrict__ xi,
                                                    double* __restrict__ a, int P, int m, int nb,
                                                    unsigned long long* __restrict__ keys) {
    __shared__ double sX[FT_K][FT_B + 1];
    __shared__ double sP[FT_K][FT_P + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;   // tx -> p, ty -> b
    const int b0 = blockIdx.y * FT_B, p0 = blockIdx.x * FT_P;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k0 = 0; k0 < m; k0 += FT_K) {
        // stage xi[b0.., k0..] and phi[p0.., k0..] transposed to [k][row]
        for (int e = threadIdx.x; e < FT_K * FT_B; e += 256) {
            int r = e / FT_K, k = e % FT_K;
            int b = b0 + r, kk = k0 + k;
            sX[k][r] = (b < nb && kk < m) ? xi[(size_t)b * m + kk] : 0.0;
            int p = p0 + r;
            sP[k][r] = (p < P && kk < m) ? phi[(size_t)p * m + kk] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < FT_K; ++k) {
            double xb[4], pp[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) { xb[i] = sX[k][ty + 16 * i]; pp[i] = sP[k][tx + 16 * i]; }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(xb[i], pp[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int b = b0 + ty + 16 * i;
        if (b >= nb) continue;
        double mx = 0.0, mn = DBL_MAX;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int p = p0 + tx + 16 * j;
            if (p < P) {
                const double v = exp(acc[i][j]);
                a[(size_t)b * P + p] = v;
                mx = fmax(mx, v);
                mn = fmin(mn, v);
            }
        }
        if (keys) key_update(keys, b, mx, mn);
    }
}

// K1 on the FP64 tensor cores: DMMA (mma.sync m8n8k4 f64; tcgen05 has no f64 kind).
// A CTA computes a 64-sample x 64-centroid tile of G = Xi Phi^T with 8 warps (2 along the
// samples x 4 along the centroids, 32 x 16 each = 4 x 2 MMA tiles), K staged through shared
// memory 16 at a time with a pitch of 68 doubles (= 4 mod 16: conflict-free fragment loads);
// the epilogue applies exp (K2) and stores a[b * P + p].
constexpr int FD_B = 64, FD_P = 64, FD_K = 16, FD_PITCH = 68;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) field_dmma_kernel(const double* __restrict__ phi, const double* __restrict__ xi,
                                                         double* __restrict__ a, int P, int m, int nb,
                                                         unsigned long long* __restrict__ keys) {
    __shared__ double sX[FD_K][FD_PITCH];
    __shared__ double sP[FD_K][FD_PITCH];
    __shared__ double kmx[4][FD_B], kmn[4][FD_B];      // per-warp-column contrast partials
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wb = warp >> 2, wp = warp & 3;            // warp tile: samples 32*wb.., centroids 16*wp..
    const int gq = lane >> 2, tq = lane & 3;            // fragment row group / thread in group
    const int b0 = blockIdx.y * FD_B, p0 = blockIdx.x * FD_P;
    double acc[4][2][2];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int u = 0; u < 2; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
    for (int k0 = 0; k0 < m; k0 += FD_K) {
        for (int e = threadIdx.x; e < FD_K * FD_B; e += 256) {
            const int r = e / FD_K, k = e % FD_K;
            const int kk = k0 + k, b = b0 + r, pp = p0 + r;
            sX[k][r] = (b < nb && kk < m) ? xi[(size_t)b * m + kk] : 0.0;
            sP[k][r] = (pp < P && kk < m) ? phi[(size_t)pp * m + kk] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int k4 = 0; k4 < FD_K; k4 += 4) {
            double fa[4], fb[2];
#pragma unroll
            for (int t = 0; t < 4; ++t) fa[t] = sX[k4 + tq][32 * wb + 8 * t + gq];   // A[row = b][col = k]
#pragma unroll
            for (int u = 0; u < 2; ++u) fb[u] = sP[k4 + tq][16 * wp + 8 * u + gq];   // B[row = k][col = p]
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
                for (int u = 0; u < 2; ++u) dmma(acc[t][u][0], acc[t][u][1], fa[t], fb[u]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int b = b0 + 32 * wb + 8 * t + gq;
        double mx = 0.0, mn = DBL_MAX;
        if (b < nb) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int p = p0 + 16 * wp + 8 * u + 2 * tq;
                double* dst = a + (size_t)b * P + p;
                if (p + 1 < P) {
                    const double v0 = exp(acc[t][u][0]), v1 = exp(acc[t][u][1]);
                    *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
                    mx = fmax(mx, fmax(v0, v1));
                    mn = fmin(mn, fmin(v0, v1));
                } else if (p < P) {
                    const double v0 = exp(acc[t][u][0]);
                    dst[0] = v0;
                    mx = fmax(mx, v0);
                    mn = fmin(mn, v0);
                }
            }
        }
        if (keys) {                                   // reduce over the 4 lanes of the row group
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, 1));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, 2));
            if (tq == 0) {
                kmx[wp][32 * wb + 8 * t + gq] = mx;
                kmn[wp][32 * wb + 8 * t + gq] = mn;
            }
        }
    }
    if (keys) {                                       // one atomic pair per sample and CTA
        __syncthreads();
        if (threadIdx.x < FD_B && b0 + threadIdx.x < nb) {
            const int r = threadIdx.x;
            const double mx = fmax(fmax(kmx[0][r], kmx[1][r]), fmax(kmx[2][r], kmx[3][r]));
            const double mn = fmin(fmin(kmn[0][r], kmn[1][r]), fmin(kmn[2][r], kmn[3][r]));
            key_update(keys, b0 + r, mx, mn);
        }
    }
}

// Longest-first order: one CTA of 1024 threads buckets the nb <= kOrderMax systems by log contrast
// (256 buckets between the batch's extremes, highest contrast first) -- a counting sort, four barriers,
// instead of a comparison sort: the schedule only needs the long solves early, and the order within
// a bucket (atomic placement) does not change any result (every system is solved independently).
__global__ void __launch_bounds__(1024) order_kernel(const unsigned long long* __restrict__ keys, int nb,
                                                     int* __restrict__ order) {
    constexpr int NBK = 256;
    __shared__ float lk[kOrderMax];
    __shared__ int cnt[NBK], pos[NBK];
    __shared__ float red_lo[32], red_hi[32];
    float lo = FLT_MAX, hi = -FLT_MAX;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        const double mx = __longlong_as_double((long long)keys[2 * i]);
        const double mn = __longlong_as_double((long long)~keys[2 * i + 1]);
        const float v = (mn > 0.0 && mx >= mn) ? (float)log(mx / mn) : 1e30f;
        lk[i] = v;
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
    }
    if (threadIdx.x < NBK) cnt[threadIdx.x] = 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) { red_lo[threadIdx.x >> 5] = lo; red_hi[threadIdx.x >> 5] = hi; }
    __syncthreads();
    lo = red_lo[0];
    hi = red_hi[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { lo = fminf(lo, red_lo[w]); hi = fmaxf(hi, red_hi[w]); }
    const float scale = hi > lo ? (NBK - 1) / (hi - lo) : 0.0f;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        const int bk = (NBK - 1) - min(NBK - 1, max(0, (int)((lk[i] - lo) * scale)));   // 0 = highest contrast
        lk[i] = __int_as_float(bk);
        atomicAdd(&cnt[bk], 1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {                            // exclusive prefix sum of the 256 counts (one warp)
        int v[NBK / 32], run = 0;
#pragma unroll
        for (int j = 0; j < NBK / 32; ++j) { v[j] = cnt[threadIdx.x * (NBK / 32) + j]; run += v[j]; }
        int incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)threadIdx.x >= o) incl += t;
        }
        int base = incl - run;
#pragma unroll
        for (int j = 0; j < NBK / 32; ++j) { pos[threadIdx.x * (NBK / 32) + j] = base; base += v[j]; }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += blockDim.x) order[atomicAdd(&pos[__float_as_int(lk[i])], 1)] = i;
}

cudaError_t launch_order(const unsigned long long* keys, int nb, int* order, cudaStream_t s) {
    if (nb <= 0) return cudaSuccess;
    if (nb > kOrderMax) return cudaErrorInvalidValue;
    order_kernel<<<1, 1024, 0, s>>>(keys, nb, order);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- K1s: separable synthesis
// Both fields are sums of products: g(x1, x2) = sum_k c_k xi_k f_{a_k}(x1) g_{b_k}(x2) (the 2D KL modes of
// the separable covariance, R11; Eq. (20)'s sin x cos terms).  With f, g tabulated at the N centroid
// abscissae (i + 1/3) h, (i + 2/3) h of each axis, a lower triangle (centroid ((i+2/3)h, (j+1/3)h)) gets
//     g_L(i, j) = sum_a f23[i][a] W_L[a][j],   W_L[a][j] = sum_{k: a_k = a} c_k xi_k g13[j][b_k],
// an upper one the same with f13 and g23.  Per sample: 2 m N + 4 K N^2 flops instead of 4 m N^2 (K = the
// number of 1D functions: 16 for configs[1], 30 for configs[4]); the same values as the P x m synthesis
// up to the order of the binary64 sums.  A CTA takes SB samples x a TJ-row x TI-column tile of the mesh:
// u = c xi (gathered in the CSR order), W_L / W_U for its rows, then the outputs (i fastest, so the
// (lower, upper) pairs of a row are stored as contiguous double2), exp, and the contrast keys.
__global__ void __launch_bounds__(256) field_sep_kernel(const double* __restrict__ tab, const int* __restrict__ aoff,
                                                        const int* __restrict__ mk, const int* __restrict__ mb,
                                                        const double* __restrict__ mc, int K,
                                                        const double* __restrict__ xi, double* __restrict__ a, int N,
                                                        int m, int nb, int SB, int TJ, int TI,
                                                        unsigned long long* __restrict__ keys) {
    extern __shared__ __align__(16) double fsm[];
    double* u = fsm;                               // [SB][m] in CSR order
    double* W0 = u + SB * m;                       // [SB][K][TJ]
    double* W1 = W0 + SB * K * TJ;
    double* F23 = W1 + SB * K * TJ;                // [K][TI]
    double* F13 = F23 + K * TI;
    double* G13 = F13 + K * TI;                    // [K][TJ]
    double* G23 = G13 + K * TJ;
    unsigned long long* kk = reinterpret_cast<unsigned long long*>(G23 + K * TJ);   // [SB][2]
    const int tid = threadIdx.x;
    const int b0 = blockIdx.x * SB, j0 = blockIdx.y * TJ, i0 = blockIdx.z * TI;
    const int ns = min(SB, nb - b0), nj = min(TJ, N - j0), ni = min(TI, N - i0);
    const size_t NK = (size_t)N * K;
    for (int e = tid; e < SB * m; e += blockDim.x) {
        const int sm = e / m, q = e % m;
        u[e] = sm < ns ? __ldg(mc + q) * __ldg(xi + (size_t)(b0 + sm) * m + __ldg(mk + q)) : 0.0;
    }
    for (int e = tid; e < K * TI; e += blockDim.x) {
        const int q = e / TI, ii = e % TI;
        const bool in = ii < ni;
        F13[e] = in ? __ldg(tab + (size_t)(i0 + ii) * K + q) : 0.0;
        F23[e] = in ? __ldg(tab + NK + (size_t)(i0 + ii) * K + q) : 0.0;
    }
    for (int e = tid; e < K * TJ; e += blockDim.x) {
        const int q = e / TJ, jj = e % TJ;
        const bool in = jj < nj;
        G13[e] = in ? __ldg(tab + 2 * NK + (size_t)(j0 + jj) * K + q) : 0.0;
        G23[e] = in ? __ldg(tab + 3 * NK + (size_t)(j0 + jj) * K + q) : 0.0;
    }
    if (tid < 2 * SB) kk[tid] = 0ull;
    __syncthreads();
    for (int e = tid; e < SB * K * TJ; e += blockDim.x) {
        const int sm = e / (K * TJ), r = e % (K * TJ), q = r / TJ, jj = r % TJ;
        const double* us = u + sm * m;
        double w0 = 0.0, w1 = 0.0;
        const int e1 = __ldg(aoff + q + 1);
        for (int c = __ldg(aoff + q); c < e1; ++c) {
            const double uc = us[c];
            const int bq = __ldg(mb + c);
            w0 = fma(uc, G13[bq * TJ + jj], w0);
            w1 = fma(uc, G23[bq * TJ + jj], w1);
        }
        W0[e] = w0;
        W1[e] = w1;
    }
    __syncthreads();
    const int P = 2 * N * N;
    for (int e = tid; e < SB * TJ * TI; e += blockDim.x) {
        const int sm = e / (TJ * TI), r = e % (TJ * TI), jj = r / TI, ii = r % TI;
        const bool live = sm < ns && jj < nj && ii < ni;
        double v0 = 0.0, v1 = 0.0;
        if (live) {
            const double* w0 = W0 + sm * K * TJ + jj;
            const double* w1 = W1 + sm * K * TJ + jj;
            double g0 = 0.0, g1 = 0.0;
            for (int q = 0; q < K; ++q) {
                g0 = fma(F23[q * TI + ii], w0[q * TJ], g0);
                g1 = fma(F13[q * TI + ii], w1[q * TJ], g1);
            }
            v0 = exp(g0);
            v1 = exp(g1);
            *reinterpret_cast<double2*>(a + (size_t)(b0 + sm) * P + 2 * ((size_t)(j0 + jj) * N + i0 + ii)) =
                make_double2(v0, v1);
        }
        if (keys) {
            // contrast partials: a warp's outputs belong to one sample when TJ * TI is a multiple of 32
            double mx = live ? fmax(v0, v1) : 0.0, mn = live ? fmin(v0, v1) : DBL_MAX;
            const int s0 = __shfl_sync(0xffffffffu, sm, 0);
            if (__all_sync(0xffffffffu, sm == s0)) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                }
                if ((tid & 31) == 0 && s0 < ns) {
                    atomicMax(kk + 2 * s0, (unsigned long long)__double_as_longlong(mx));
                    atomicMax(kk + 2 * s0 + 1, ~(unsigned long long)__double_as_longlong(mn));
                }
            } else if (live) {
                atomicMax(kk + 2 * sm, (unsigned long long)__double_as_longlong(mx));
                atomicMax(kk + 2 * sm + 1, ~(unsigned long long)__double_as_longlong(mn));
            }
        }
    }
    if (keys) {
        __syncthreads();
        if (tid < ns) {
            atomicMax(keys + 2 * (b0 + tid), kk[2 * tid]);
            atomicMax(keys + 2 * (b0 + tid) + 1, kk[2 * tid + 1]);
        }
    }
}

cudaError_t launch_field_sep(const double* tab, const int* aoff, const int* mk, const int* mb, const double* mc,
                             int K, const double* xi, double* a, int N, int m, uint64_t nb, unsigned long long* keys,
                             cudaStream_t s) {
    if (nb == 0) return cudaSuccess;
    // tile: all of a small mesh per CTA with several samples, else 16 rows x 64 columns of one sample
    int SB, TJ, TI;
    if (N <= 8) { SB = 16; TJ = N; TI = N; }
    else if (N <= 16) { SB = 4; TJ = N; TI = N; }
    else if (N <= 32) { SB = 1; TJ = N; TI = N; }
    else { SB = 1; TJ = 16; TI = 64; }
    auto bytes = [&](int sb) {
        return (size_t)8 * ((size_t)sb * m + 2 * (size_t)sb * K * TJ + 2 * (size_t)K * TI + 2 * (size_t)K * TJ) +
               16 * (size_t)sb;
    };
    while (SB > 1 && bytes(SB) > 200 * 1024) SB /= 2;
    const size_t smem = bytes(SB);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
        cudaError_t e = cudaFuncSetAttribute(field_sep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = smem;
    }
    const dim3 grid((unsigned)((nb + SB - 1) / SB), (unsigned)((N + TJ - 1) / TJ), (unsigned)((N + TI - 1) / TI));
    field_sep_kernel<<<grid, 256, smem, s>>>(tab, aoff, mk, mb, mc, K, xi, a, N, m, (int)nb, SB, TJ, TI, keys);
    return cudaGetLastError();
}

static bool field_use_ffma() {
#ifndef MLMC_TUNING
    return false;      // production build: DMMA (the FFMA64 kernel is an A/B variant, tools only)
#endif
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("MLMC_FIELD_KERNEL");
        v = (e && std::strcmp(e, "ffma") == 0) ? 1 : 0;
    }
    return v == 1;
}

bool field_use_dense() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("MLMC_FIELD_KERNEL");
        v = (e && (std::strcmp(e, "ffma") == 0 || std::strcmp(e, "dense") == 0)) ? 1 : 0;
    }
    return v == 1;
}

bool field_force_sep() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("MLMC_FIELD_KERNEL");
        v = (e && std::strcmp(e, "sep") == 0) ? 1 : 0;
    }
    return v == 1;
}

cudaError_t launch_field(const double* phi, const double* xi, double* a, int P, int m, uint64_t nb,
                         unsigned long long* keys, cudaStream_t s) {
    if (nb == 0) return cudaSuccess;
    // grid.y (sample blocks) is capped at 65535: larger batches go in slices of whole sample blocks
    if (P & 1) return cudaErrorInvalidValue;          // P = 2 N^2 is always even (DMMA tiles pairs of centroids)
    const bool ffma = field_use_ffma();
    const uint64_t per = 65535ull * (ffma ? FT_B : FD_B);
    for (uint64_t b0 = 0; b0 < nb; b0 += per) {
        const uint64_t nbs = std::min<uint64_t>(per, nb - b0);
        const double* xs = xi + b0 * m;
        double* as = a + b0 * (uint64_t)P;
        unsigned long long* ks = keys ? keys + 2 * b0 : nullptr;
        if (ffma) {
#ifdef MLMC_TUNING
            dim3 grid((P + FT_P - 1) / FT_P, (unsigned)((nbs + FT_B - 1) / FT_B));
            field_kernel<<<grid, 256, 0, s>>>(phi, xs, as, P, m, (int)nbs, ks);
#endif
        } else {
            dim3 grid((P + FD_P - 1) / FD_P, (unsigned)((nbs + FD_B - 1) / FD_B));
            field_dmma_kernel<<<grid, 256, 0, s>>>(phi, xs, as, P, m, (int)nbs, ks);
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace mlmc
