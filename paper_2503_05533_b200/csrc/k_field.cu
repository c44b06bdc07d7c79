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

// Longest-first order: one CTA buckets the nb <= kOrderMax systems by log contrast (256 buckets between the
// batch's extremes, highest contrast first) -- a counting sort, four barriers, instead of a comparison sort:
// the schedule only needs the long solves early, and the order within a bucket (atomic placement) does not
// change any result (every system is solved independently).  Run by order_kernel (1024 threads) or by the
// last CTA of the separable field kernel (256 threads) over `scratch` (kOrderScratch bytes of shared memory).
__device__ void lpt_order_block(const unsigned long long* __restrict__ keys, int nb, int* __restrict__ order,
                                unsigned char* scratch) {
    constexpr int NBK = 256;
    float* lk = reinterpret_cast<float*>(scratch);            // [kOrderMax]
    int* cnt = reinterpret_cast<int*>(lk + kOrderMax);       // [NBK]
    int* pos = cnt + NBK;                                     // [NBK]
    float* red_lo = reinterpret_cast<float*>(pos + NBK);      // [32]
    float* red_hi = red_lo + 32;                              // [32]
    const int tid = threadIdx.x, nt = blockDim.x;
    float lo = FLT_MAX, hi = -FLT_MAX;
    for (int i = tid; i < nb; i += nt) {
        const double mx = __longlong_as_double((long long)__ldcg(keys + 2 * i));
        const double mn = __longlong_as_double((long long)~__ldcg(keys + 2 * i + 1));
        const float v = (mn > 0.0 && mx >= mn) ? (float)log(mx / mn) : 1e30f;
        lk[i] = v;
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
    }
    for (int i = tid; i < NBK; i += nt) cnt[i] = 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((tid & 31) == 0) { red_lo[tid >> 5] = lo; red_hi[tid >> 5] = hi; }
    __syncthreads();
    lo = red_lo[0];
    hi = red_hi[0];
    for (int w = 1; w < (nt >> 5); ++w) { lo = fminf(lo, red_lo[w]); hi = fmaxf(hi, red_hi[w]); }
    const float scale = hi > lo ? (NBK - 1) / (hi - lo) : 0.0f;
    for (int i = tid; i < nb; i += nt) {
        const int bk = (NBK - 1) - min(NBK - 1, max(0, (int)((lk[i] - lo) * scale)));   // 0 = highest contrast
        lk[i] = __int_as_float(bk);
        atomicAdd(&cnt[bk], 1);
    }
    __syncthreads();
    if (tid < 32) {                                   // exclusive prefix sum of the 256 counts (one warp)
        int v[NBK / 32], run = 0;
#pragma unroll
        for (int j = 0; j < NBK / 32; ++j) { v[j] = cnt[tid * (NBK / 32) + j]; run += v[j]; }
        int incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (tid >= o) incl += t;
        }
        int base = incl - run;
#pragma unroll
        for (int j = 0; j < NBK / 32; ++j) { pos[tid * (NBK / 32) + j] = base; base += v[j]; }
    }
    __syncthreads();
    for (int i = tid; i < nb; i += nt) order[atomicAdd(&pos[__float_as_int(lk[i])], 1)] = i;
}

__global__ void __launch_bounds__(1024) order_kernel(const unsigned long long* __restrict__ keys, int nb,
                                                     int* __restrict__ order) {
    __shared__ __align__(16) unsigned char scratch[kOrderScratch];
    lpt_order_block(keys, nb, order, scratch);
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
//     g_L(i, j) = sum_a F23[i][a] W_L[a][j],   W_L[a][j] = sum_{k: a_k = a} c_k xi_k G13[j][b_k],
// an upper one the same with F13 and G23.  Per sample 4 m N + 4 K N^2 flops instead of 4 m N^2 (K = the
// number of 1D functions: 16 for configs[1], 30 for configs[4]); the same values as the P x m synthesis
// up to the order of the binary64 sums.
//
// Per sample both stages are small matrix products on the FP64 tensor cores (DMMA m8n8k4):
//     W_t = C_xi G_t^T     (Kp x Kp) (Kp x N):  C_xi[a][b] = c_k xi_k for the mode k = (a, b), else 0
//     g_t = F_t W_t        (N x Kp) (Kp x N):   t = lower (F23, G13) / upper (F13, G23)
// with K zero-padded to KP in {8, 16, 32}; C_xi is gathered through the K x K mode map (kmap, cmap:
// every (a, b) pair belongs to at most one mode).  A CTA owns a TJ x TJ tile of the mesh (TJ = min(N,
// 32)), stages its F and G tables and the mode map once, and loops over groups of SB samples
// (SB (TJ/8)^2 >= 8 output blocks; see launch_sep_t): gather C_xi, W for its rows, then the 8 x 8 output blocks -- the
// lower and upper triangles of a block in one warp, so that a thread holds (L, U) at two adjacent
// cells and stores 2 x double2 = the 32 contiguous bytes a[2(jN+i) .. 2(jN+i)+3].  Warp w always takes
// column block w mod (TJ/8), so its F fragments stay in registers; all trip counts are compile-time
// (unrolled: the loads and DMMA chains of a thread's blocks are independent).  Every sum runs over b,
// resp. a, in ascending order whatever the tiling.  Shared-memory pitches are 4 mod 16 doubles: the
// fragment loads (row tq, column gq) are conflict-free.
namespace {
__host__ __device__ constexpr int sep_pitch(int w) { return ((w + 15) / 16) * 16 + 4; }
template <int TJ, int KP, int SB>
__host__ __device__ constexpr size_t sep_smem() {
    return (size_t)8 * (2 * (size_t)KP * sep_pitch(SB * TJ)              // W_t[a][s TJ + jj]
                        + 2 * (size_t)KP * sep_pitch(TJ)                  // F_t[a][ii]
                        + 2 * (size_t)KP * sep_pitch(TJ)                  // G_t[b][jj]
                        + (size_t)SB * KP * sep_pitch(KP)                 // C_xi[s][a][b]
                        + (size_t)KP * KP) +                              // c of the mode map
           4 * (size_t)KP * KP +                                          // k of the mode map
           16 * (size_t)SB;                                               // contrast keys
}
}  // namespace

template <int TJ, int KP, int SB>
__global__ void __launch_bounds__(256, KP == 32 ? (TJ == 8 ? 2 : 3) : 4) field_sep_kernel(const double* __restrict__ tab, const int* __restrict__ kmap,
                                                        const double* __restrict__ cmap, int K,
                                                        const double* __restrict__ xi, double* __restrict__ a, int N,
                                                        int m, int nb, unsigned long long* __restrict__ keys,
                                                        int* __restrict__ order, unsigned* __restrict__ done) {
    constexpr int TI = TJ, SJ = SB * TJ;
    constexpr int PW = sep_pitch(SJ), PF = sep_pitch(TI), PG = sep_pitch(TJ), PC = sep_pitch(KP);
    constexpr int NT = 256, NW = 8, NBJ = TJ / 8, NBI = TI / 8, PER = NBJ * NBI, NK4 = KP / 4;
    constexpr int NAB = KP / 8, WPER = 2 * NAB * NBJ;
    static_assert(NW % NBI == 0 && (SB * PER) % NW == 0 && (SB * WPER) % NW == 0, "even warp split");
    extern __shared__ __align__(16) double fsm[];
    double* W = fsm;                               // [2][KP][PW]
    double* F = W + 2 * KP * PW;                   // [2][KP][PF]   t = 0: F23, t = 1: F13
    double* G = F + 2 * KP * PF;                   // [2][KP][PG]   t = 0: G13, t = 1: G23
    double* Cx = G + 2 * KP * PG;                  // [SB][KP][PC]
    double* Cm = Cx + SB * KP * PC;                // [KP * KP]  c_k of the pair (a, b), 0 if none
    int* Km = reinterpret_cast<int*>(Cm + KP * KP);                                // [KP * KP]  k, or -1
    unsigned long long* kk = reinterpret_cast<unsigned long long*>(Km + KP * KP);  // [SB][2]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const int nti = N / TI;
    const int j0 = (blockIdx.y / nti) * TJ, i0 = (blockIdx.y % nti) * TI;
    const size_t NK = (size_t)N * K, P = 2 * (size_t)N * N;
    {   // the tile's 1D tables, [t][x][q] -> [t][q][x], zero-padded q >= K (q fastest: coalesced reads)
        constexpr int R = (2 * TI * KP + NT - 1) / NT;
        double fv[R], gv[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int e = tid + NT * r, t = e / (TI * KP), ii = (e / KP) % TI, q = e % KP;
            const bool in = e < 2 * TI * KP && q < K;
            fv[r] = in ? __ldg(tab + (t == 0 ? NK : 0) + (size_t)(i0 + ii) * K + q) : 0.0;
            gv[r] = in ? __ldg(tab + (2 + t) * NK + (size_t)(j0 + ii) * K + q) : 0.0;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int e = tid + NT * r, t = e / (TI * KP), ii = (e / KP) % TI, q = e % KP;
            if (e < 2 * TI * KP) {
                F[(t * KP + q) * PF + ii] = fv[r];
                G[(t * KP + q) * PG + ii] = gv[r];
            }
        }
        for (int e = tid; e < KP * KP; e += NT) {
            const int ra = e / KP, rb = e % KP;
            const bool in = ra < K && rb < K;
            const int k = in ? __ldg(kmap + ra * K + rb) : -1;
            Km[e] = k;
            Cm[e] = k >= 0 ? __ldg(cmap + ra * K + rb) : 0.0;
        }
    }
    __syncthreads();
    const int ib = warp % NBI;                     // this warp's column block (fixed)
    double fL[NK4], fU[NK4];
#pragma unroll
    for (int k = 0; k < NK4; ++k) {
        fL[k] = F[(4 * k + tq) * PF + 8 * ib + gq];
        fU[k] = F[(KP + 4 * k + tq) * PF + 8 * ib + gq];
    }
    const int ngroups = (nb + SB - 1) / SB;
    for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        const int b0 = grp * SB, ns = min(SB, nb - b0);
        {   // C_xi[s][a][b] = c xi_k (gathered)
            constexpr int R = (SB * KP * KP + NT - 1) / NT;
            double v[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int e = tid + NT * r, sm = e / (KP * KP), me = e % (KP * KP);
                const int k = e < SB * KP * KP ? Km[me] : -1;
                v[r] = (k >= 0 && sm < ns) ? Cm[me] * __ldg(xi + (size_t)(b0 + sm) * m + k) : 0.0;
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int e = tid + NT * r, sm = e / (KP * KP), me = e % (KP * KP);
                if (e < SB * KP * KP) Cx[(sm * KP + me / KP) * PC + me % KP] = v[r];
            }
        }
        if (keys && tid < 2 * SB) kk[tid] = tid & 1 ? ~0ull : 0ull;   // per sample: bits(max) up, bits(min) down
        __syncthreads();
        // W_t[a][s TJ + jj] = sum_b C_xi[s][a][b] G_t[b][jj]  (8 x 8 blocks, KP / 4 DMMA each)
#pragma unroll
        for (int n = 0; n < SB * WPER / NW; ++n) {
            const int task = warp + NW * n;
            const int sm = task / WPER, r = task % WPER, t = r / (NAB * NBJ), ab = (r / NBJ) % NAB, jb = r % NBJ;
            double d0 = 0.0, d1 = 0.0;
            const double* ca = Cx + (sm * KP + 8 * ab + gq) * PC + tq;          // A[row a][col b]
            const double* gb = G + (t * KP + tq) * PG + 8 * jb + gq;            // B[row b][col jj]
#pragma unroll
            for (int k = 0; k < NK4; ++k) dmma(d0, d1, ca[4 * k], gb[4 * k * PG]);
            *reinterpret_cast<double2*>(W + (t * KP + 8 * ab + gq) * PW + sm * TJ + 8 * jb + 2 * tq) =
                make_double2(d0, d1);
        }
        __syncthreads();
        // g_t[jj][ii] = sum_a W_t[a][jj] F_t[a][ii], exp, store; contrast keys per sample
        constexpr int NB = SB * PER / NW;          // blocks per warp; a warp's blocks of one sample are adjacent
        double mx = 0.0, mn = DBL_MAX;
#pragma unroll
        for (int n = 0; n < NB; ++n) {
            const int blk = warp + NW * n, sm = blk / PER, jb = (blk % PER) / NBI;
            if (sm < ns) {
                double dL0 = 0.0, dL1 = 0.0, dU0 = 0.0, dU1 = 0.0;
                const double* wL = W + tq * PW + sm * TJ + 8 * jb + gq;         // A[row jj][col a]
#pragma unroll
                for (int k = 0; k < NK4; ++k) {
                    dmma(dL0, dL1, wL[4 * k * PW], fL[k]);
                    dmma(dU0, dU1, wL[(KP + 4 * k) * PW], fU[k]);
                }
                const int j = j0 + 8 * jb + gq, i = i0 + 8 * ib + 2 * tq;
                const double l0 = exp(dL0), u0 = exp(dU0), l1 = exp(dL1), u1 = exp(dU1);
                double* dst = a + (size_t)(b0 + sm) * P + 2 * ((size_t)j * N + i);
                *reinterpret_cast<double2*>(dst) = make_double2(l0, u0);
                *reinterpret_cast<double2*>(dst + 2) = make_double2(l1, u1);
                mx = fmax(mx, fmax(fmax(l0, u0), fmax(l1, u1)));
                mn = fmin(mn, fmin(fmin(l0, u0), fmin(l1, u1)));
            }
            const bool last = n + 1 == NB || (warp + NW * (n + 1)) / PER != sm;
            if (keys && last) {                                   // warp-uniform
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                }
                if (lane == 0 && sm < ns) {
                    atomicMax(kk + 2 * sm, (unsigned long long)__double_as_longlong(mx));
                    atomicMin(kk + 2 * sm + 1, (unsigned long long)__double_as_longlong(mn));
                }
                mx = 0.0;
                mn = DBL_MAX;
            }
        }
        if (keys) {
            __syncthreads();
            if (tid < ns) {                                       // the global keys hold ~bits(min): max of ~
                atomicMax(keys + 2 * (b0 + tid), kk[2 * tid]);
                atomicMax(keys + 2 * (b0 + tid) + 1, ~kk[2 * tid + 1]);
            }
        }
        __syncthreads();                                          // Cx, W and kk are rewritten next group
    }
    if (order) {   // the last CTA to finish forms the longest-first order from the completed contrast keys
        __shared__ int last;
        __threadfence();                                      // every thread's key atomics before the count
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            last = atomicAdd(done, 1u) == gridDim.x * gridDim.y - 1;
        }
        __syncthreads();
        if (last) {
            __threadfence();
            lpt_order_block(keys, nb, order, reinterpret_cast<unsigned char*>(fsm));
        }
    }
}

namespace {
// SB samples per group: 8 at N = 8, 4 at N = 16 (8 output blocks per group), 1 at N >= 32 (two per group
// measured 7% slower at configs[1] level 3: fewer CTAs to hide the latency of the phases).
template <int TJ, int KP, int SB>
cudaError_t launch_sep_t(const double* tab, const int* kmap, const double* cmap, int K, const double* xi, double* a,
                         int N, int m, uint64_t nb, unsigned long long* keys, int* order, unsigned* done,
                         cudaStream_t s) {
    // (the tile's shared memory doubles as the order's scratch in the last CTA)
    constexpr size_t smem = sep_smem<TJ, KP, SB>() > kOrderScratch ? sep_smem<TJ, KP, SB>() : kOrderScratch;
    static_assert(smem <= 227 * 1024, "separable synthesis tile exceeds shared memory");
    static PerDevice<KernelOcc> cache;
    const KernelOcc occ = occ_of(cache, field_sep_kernel<TJ, KP, SB>, 256, smem);
    if (occ.err != cudaSuccess) return occ.err;
    const uint64_t tiles = (uint64_t)(N / TJ) * (N / TJ);
    if (tiles > 65535) return cudaErrorInvalidValue;
    const uint64_t groups = (nb + SB - 1) / SB;
    const uint64_t all = (uint64_t)occ.per_sm * occ.sms;
    const uint64_t gx = std::min<uint64_t>(groups, std::max<uint64_t>(1, all / tiles));
    if (order && (!keys || !done || nb > (uint64_t)kOrderMax)) return cudaErrorInvalidValue;
    field_sep_kernel<TJ, KP, SB><<<dim3((unsigned)gx, (unsigned)tiles), 256, smem, s>>>(tab, kmap, cmap, K, xi, a, N,
                                                                                       m, (int)nb, keys, order, done);
    return cudaGetLastError();
}
template <int TJ, int KP>
cudaError_t launch_sep_sb(const double* tab, const int* kmap, const double* cmap, int K, const double* xi, double* a,
                          int N, int m, uint64_t nb, unsigned long long* keys, int* order, unsigned* done,
                          cudaStream_t s) {
    if constexpr (TJ == 8) {
        return launch_sep_t<TJ, KP, 8>(tab, kmap, cmap, K, xi, a, N, m, nb, keys, order, done, s);
    } else if constexpr (TJ == 16) {
        return launch_sep_t<TJ, KP, 4>(tab, kmap, cmap, K, xi, a, N, m, nb, keys, order, done, s);
    } else {
        return launch_sep_t<TJ, KP, 1>(tab, kmap, cmap, K, xi, a, N, m, nb, keys, order, done, s);
    }
}
template <int TJ>
cudaError_t launch_sep_k(const double* tab, const int* kmap, const double* cmap, int K, const double* xi, double* a,
                         int N, int m, uint64_t nb, unsigned long long* keys, int* order, unsigned* done,
                         cudaStream_t s) {
    if (K <= 8) return launch_sep_sb<TJ, 8>(tab, kmap, cmap, K, xi, a, N, m, nb, keys, order, done, s);
    if (K <= 16) return launch_sep_sb<TJ, 16>(tab, kmap, cmap, K, xi, a, N, m, nb, keys, order, done, s);
    return launch_sep_sb<TJ, 32>(tab, kmap, cmap, K, xi, a, N, m, nb, keys, order, done, s);
}
}  // namespace

bool field_sep_supported(int N, int K) { return N >= 8 && (N < 32 ? (N & (N - 1)) == 0 : N % 32 == 0) && K >= 1 && K <= 32; }

cudaError_t launch_field_sep(const double* tab, const int* kmap, const double* cmap, int K, const double* xi,
                             double* a, int N, int m, uint64_t nb, unsigned long long* keys, cudaStream_t s,
                             int* order, unsigned* done) {
    if (nb == 0) return cudaSuccess;
    if (!field_sep_supported(N, K) || nb > 0x7fffffffull) return cudaErrorInvalidValue;
    if (N >= 32) return launch_sep_k<32>(tab, kmap, cmap, K, xi, a, N, m, nb, keys, order, done, s);
    if (N == 16) return launch_sep_k<16>(tab, kmap, cmap, K, xi, a, N, m, nb, keys, order, done, s);
    return launch_sep_k<8>(tab, kmap, cmap, K, xi, a, N, m, nb, keys, order, done, s);
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
