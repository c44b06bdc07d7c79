// k_chol.cu -- K4: batched banded Cholesky in a low precision u_f + iterative refinement.
//
// Algorithm 1 for the P1 system A x = b of one sample:
//   1. factorise A = L L^T in precision u_f
//   2. solve A x0 = b by substitution, store x0 in u    (substitutions in u_s, R24)
//   3. for i = 0..i_max:
//   4.   r_i = b - A x_i in u_r (binary64), rounded to u (binary64)   (R13)
//   5.   if ||r_i|| / ||b|| < tol: exit
//   7.   solve A d_i = r_i with the retained factor in u_s
//   8.   x_{i+1} = x_i + d_i in u (binary64)
// The matrix is the 5-point P1 operator (R10): natural ordering gives band
// width bw = N - 1 and the factor fills the band completely, so L is kept as
// a dense n x (bw+1) band, Lb[r*(bw+1) + d] = L(r, r-d), in shared memory in
// the factor format (fp16 / fp32 / fp64) -- mixed precision is what makes the
// factor of the h = 1/32 level fit on chip (61.5 KB fp16, 123 KB fp32).
//
// B200 mapping: one warp per sample, lanes = band offsets (bw + 1 <= 32).
//  * factorisation, right-looking in place: step k computes column k
//    (lane i: L(k+i,k)) and applies the rank-1 update to the (bw x bw) window,
//    lane i owning row k+i; every arithmetic op in the factor type.
//  * substitutions, column-oriented with a sliding register window: lane d
//    holds the pending right-hand side entry k+d; one broadcast and one
//    shift per row.
//  * residual in binary64 with the stencil from the conductances (kept in
//    shared memory), reductions by xor butterflies.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cfloat>
#include <cstdint>

#include "internal.h"

namespace mlmc {

template <typename T> struct FT;
template <> struct FT<double> {
    static __device__ __forceinline__ double from(double v) { return v; }
    static __device__ __forceinline__ double to_d(double v) { return v; }
    static __device__ __forceinline__ double fnma(double a, double b, double c) { return fma(-a, b, c); }
    static __device__ __forceinline__ double div(double a, double b) { return a / b; }
    static __device__ __forceinline__ double sqrt_(double a) { return sqrt(a); }
    static __device__ __forceinline__ bool pos_finite(double a) { return a > 0.0 && a <= DBL_MAX; }
};
template <> struct FT<float> {
    static __device__ __forceinline__ float from(double v) { return __double2float_rn(v); }
    static __device__ __forceinline__ double to_d(float v) { return (double)v; }
    static __device__ __forceinline__ float fnma(float a, float b, float c) { return __fmaf_rn(-a, b, c); }
    static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
    static __device__ __forceinline__ float sqrt_(float a) { return __fsqrt_rn(a); }
    static __device__ __forceinline__ bool pos_finite(float a) { return a > 0.0f && a <= FLT_MAX; }
};
template <> struct FT<__half> {
    static __device__ __forceinline__ __half from(double v) { return __double2half(v); }
    static __device__ __forceinline__ double to_d(__half v) { return (double)__half2float(v); }
    static __device__ __forceinline__ __half fnma(__half a, __half b, __half c) { return __hfma(__hneg(a), b, c); }
    static __device__ __forceinline__ __half div(__half a, __half b) { return __hdiv(a, b); }
    static __device__ __forceinline__ __half sqrt_(__half a) { return __float2half_rn(sqrtf(__half2float(a))); }
    static __device__ __forceinline__ bool pos_finite(__half a) {
        float f = __half2float(a);
        return f > 0.0f && f <= 65504.0f;
    }
};

__device__ __forceinline__ double wsum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int N, typename F>
struct CholCfg {
    static constexpr int n = (N - 1) * (N - 1);
    static constexpr int BW = N - 1;
    static constexpr int W = BW + 1;   // band row length (<= 32)
    static constexpr size_t band_bytes = ((sizeof(F) * (size_t)n * W + 15) / 16) * 16;
    // per warp: band, cE, cN (N^2 doubles each), x, r (n doubles each), 2 ints
    static constexpr size_t per_warp = band_bytes + sizeof(double) * (2 * N * N + 2 * n) + 16;
    static constexpr int WARPS = (int)((200 * 1024) / per_warp) < 1 ? 1
                                 : ((int)((200 * 1024) / per_warp) > 8 ? 8 : (int)((200 * 1024) / per_warp));
    static constexpr size_t SMEM = per_warp * WARPS;
    static_assert(W <= 32, "band must fit a warp");
};

// forward (L y = r) and backward (L^T z = y) substitution in precision S, in place on v (binary64 storage).
template <int N, typename F, typename S>
__device__ __forceinline__ void band_solve(const F* __restrict__ Lb, double* __restrict__ v, int lane) {
    using C = CholCfg<N, F>;
    constexpr int n = C::n, W = C::W, BW = C::BW;
    // forward: lane d holds the pending entry k + d
    S cur = (lane < W && lane < n) ? (S)v[lane] : (S)0;
    for (int k = 0; k < n; ++k) {
        S yk = (S)0;
        if (lane == 0) yk = cur / (S)FT<F>::to_d(Lb[(size_t)k * W]);
        yk = __shfl_sync(0xffffffffu, yk, 0);
        if (lane >= 1 && lane <= BW && k + lane < n) cur = cur - (S)FT<F>::to_d(Lb[(size_t)(k + lane) * W + lane]) * yk;
        if (lane == 0) v[k] = (double)yk;
        S nxt = __shfl_down_sync(0xffffffffu, cur, 1);
        if (lane == BW) nxt = (k + W < n) ? (S)v[k + W] : (S)0;
        cur = nxt;
    }
    __syncwarp();
    // backward: lane d holds the pending entry k - d
    cur = (lane < W && n - 1 - lane >= 0) ? (S)v[n - 1 - lane] : (S)0;
    for (int k = n - 1; k >= 0; --k) {
        S xk = (S)0;
        if (lane == 0) xk = cur / (S)FT<F>::to_d(Lb[(size_t)k * W]);
        xk = __shfl_sync(0xffffffffu, xk, 0);
        if (lane >= 1 && lane <= BW && k - lane >= 0) cur = cur - (S)FT<F>::to_d(Lb[(size_t)k * W + lane]) * xk;
        if (lane == 0) v[k] = (double)xk;
        S nxt = __shfl_down_sync(0xffffffffu, cur, 1);
        if (lane == BW) nxt = (k - W >= 0) ? (S)v[k - W] : (S)0;
        cur = nxt;
    }
    __syncwarp();
}

template <int N, typename F, typename S>
__global__ void __launch_bounds__(32 * CholCfg<N, F>::WARPS)
chol_ir_kernel(const double* __restrict__ a_all, int nb, double tol, int i_max, double* __restrict__ out, int slot,
               unsigned* __restrict__ job_counter) {
    using C = CholCfg<N, F>;
    constexpr int n = C::n, W = C::W, BW = C::BW, P = 2 * N * N;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* base = smem_raw + C::per_warp * warp;
    F* Lb = reinterpret_cast<F*>(base);
    double* cE = reinterpret_cast<double*>(base + C::band_bytes);
    double* cN = cE + N * N;
    double* xv = cN + N * N;
    double* rv = xv + n;
    const double h = 1.0 / N, h2 = h * h;
    const double bnorm = h2 * sqrt((double)n);

    for (;;) {
        int job = 0;
        if (lane == 0) job = (int)atomicAdd(job_counter, 1u);
        job = __shfl_sync(0xffffffffu, job, 0);
        if (job >= nb) break;
        const double* a = a_all + (size_t)job * P;
        // conductances (binary64, the assembled operator of P:178)
        for (int e = lane; e < N * N; e += 32) {
            int i = e % N, j = e / N;
            cE[e] = (j >= 1) ? 0.5 * (__ldg(a + 2 * (j * N + i)) + __ldg(a + 2 * ((j - 1) * N + i) + 1)) : 0.0;
            cN[e] = (i >= 1) ? 0.5 * (__ldg(a + 2 * (j * N + i) + 1) + __ldg(a + 2 * (j * N + i - 1))) : 0.0;
        }
        __syncwarp();
        // band of A rounded to u_f: diagonal, west (d = 1) and south (d = BW) couplings
        for (int e = lane; e < n * W; e += 32) {
            int r = e / W, d = e % W;
            int i = r % (N - 1) + 1, j = r / (N - 1) + 1, c = j * N + i;
            double v = 0.0;
            if (d == 0) v = (cE[c] + cE[c - 1]) + (cN[c] + cN[c - N]);
            else if (d == 1 && i > 1) v = -cE[c - 1];
            else if (d == BW && j > 1) v = -cN[c - N];
            Lb[e] = FT<F>::from(v);
        }
        __syncwarp();
        // ---- step 1: right-looking banded Cholesky in F
        int status = 0;
        for (int k = 0; k < n; ++k) {
            F piv = Lb[(size_t)k * W];
            if (!FT<F>::pos_finite(piv)) { status = 2; break; }
            F lkk = FT<F>::sqrt_(piv);
            F li = FT<F>::from(0.0);
            const bool act = lane >= 1 && lane <= BW && k + lane < n;
            if (act) {
                li = FT<F>::div(Lb[(size_t)(k + lane) * W + lane], lkk);
                Lb[(size_t)(k + lane) * W + lane] = li;
            }
            __syncwarp();
            if (lane == 0) Lb[(size_t)k * W] = lkk;
            if (act) {
                F* row = Lb + (size_t)(k + lane) * W;
#pragma unroll 4
                for (int jj = 1; jj <= BW; ++jj) {
                    if (jj > lane) break;
                    F lj = Lb[(size_t)(k + jj) * W + jj];
                    row[lane - jj] = FT<F>::fnma(li, lj, row[lane - jj]);
                }
            }
            __syncwarp();
        }
        double rel = 1.0;
        int it = 0;
        if (status == 0) {
            // ---- step 2: x0 = (L L^T)^-1 b in u_s, stored in binary64
            for (int e = lane; e < n; e += 32) rv[e] = (double)(S)h2;
            __syncwarp();
            band_solve<N, F, S>(Lb, rv, lane);
            for (int e = lane; e < n; e += 32) xv[e] = rv[e];
            __syncwarp();
            status = 1;
            for (it = 0; it <= i_max; ++it) {
                // ---- step 4: r = b - A x in binary64
                double part = 0.0;
                for (int e = lane; e < n; e += 32) {
                    int i = e % (N - 1) + 1, j = e / (N - 1) + 1, c = j * N + i;
                    double ce = cE[c], cw = cE[c - 1], cn = cN[c], cs = cN[c - N];
                    double Ax = ((ce + cw) + (cn + cs)) * xv[e];
                    if (i < N - 1) Ax = fma(-ce, xv[e + 1], Ax);
                    if (i > 1) Ax = fma(-cw, xv[e - 1], Ax);
                    if (j < N - 1) Ax = fma(-cn, xv[e + N - 1], Ax);
                    if (j > 1) Ax = fma(-cs, xv[e - (N - 1)], Ax);
                    double r = h2 - Ax;
                    rv[e] = r;
                    part = fma(r, r, part);
                }
                rel = sqrt(wsum_d(part)) / bnorm;
                __syncwarp();
                if (!(rel == rel) || rel > DBL_MAX) { status = 3; break; }
                if (rel < tol) { status = 0; break; }          // step 5
                if (it == i_max) break;
                // ---- step 7: d = (L L^T)^-1 r in u_s;  step 8: x += d in binary64
                for (int e = lane; e < n; e += 32) rv[e] = (double)(S)rv[e];
                __syncwarp();
                band_solve<N, F, S>(Lb, rv, lane);
                for (int e = lane; e < n; e += 32) xv[e] += rv[e];
                __syncwarp();
            }
        }
        double sx = 0.0;
        for (int e = lane; e < n; e += 32) sx += xv[e];
        sx = wsum_d(sx);
        if (lane == 0) {
            double* o = out + (size_t)job * kRecLen;
            o[0 + slot] = status == 2 ? 0.0 : h2 * sx;
            o[2 + slot] = (double)it;
            o[4 + slot] = rel;
            o[6 + slot] = (double)status;
        }
        __syncwarp();
    }
}

template <int N, typename F, typename S>
static cudaError_t run_chol(const double* a, uint64_t nb, double tol, int i_max, double* out, int slot, unsigned* ctr,
                            cudaStream_t s) {
    using C = CholCfg<N, F>;
    auto kern = chol_ir_kernel<N, F, S>;
    static int bps = -1, sms = 0;
    if (bps < 0) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 32 * C::WARPS, C::SMEM);
        if (e != cudaSuccess) return e;
        int dev;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (bps < 1) return cudaErrorInvalidConfiguration;
    }
    uint64_t need = (nb + C::WARPS - 1) / C::WARPS;
    uint64_t grid = std::min<uint64_t>(need, (uint64_t)bps * sms);
    if (grid == 0) return cudaSuccess;
    kern<<<(unsigned)grid, 32 * C::WARPS, C::SMEM, s>>>(a, (int)nb, tol, i_max, out, slot, ctr);
    return cudaGetLastError();
}

bool chol_supported(int N, int u_f, int u_s) {
    if (!(N == 2 || N == 4 || N == 8 || N == 16 || N == 32)) return false;
    if (!(u_f == MLMC_FMT_F16 || u_f == MLMC_FMT_F32 || u_f == MLMC_FMT_F64)) return false;
    if (!(u_s == MLMC_FMT_F32 || u_s == MLMC_FMT_F64)) return false;
    if (u_f == MLMC_FMT_F64 && N == 32) return false;   // 240 KB band: beyond shared memory
    return true;
}

template <int N>
static cudaError_t chol_dispatch(int u_f, int u_s, const double* a, uint64_t nb, double tol, int i_max, double* out,
                                 int slot, unsigned* ctr, cudaStream_t s) {
    if (u_f == MLMC_FMT_F16) {
        if (u_s == MLMC_FMT_F32) return run_chol<N, __half, float>(a, nb, tol, i_max, out, slot, ctr, s);
        return run_chol<N, __half, double>(a, nb, tol, i_max, out, slot, ctr, s);
    }
    if (u_f == MLMC_FMT_F32) {
        if (u_s == MLMC_FMT_F32) return run_chol<N, float, float>(a, nb, tol, i_max, out, slot, ctr, s);
        return run_chol<N, float, double>(a, nb, tol, i_max, out, slot, ctr, s);
    }
    if constexpr (N <= 16) return run_chol<N, double, double>(a, nb, tol, i_max, out, slot, ctr, s);
    return cudaErrorNotSupported;
}

cudaError_t launch_chol_ir(int N, const double* a, uint64_t nb, int u_f, int u_s, double tol, int i_max, double* out,
                           int slot, unsigned* ctr, cudaStream_t s) {
    switch (N) {
        case 2: return chol_dispatch<2>(u_f, u_s, a, nb, tol, i_max, out, slot, ctr, s);
        case 4: return chol_dispatch<4>(u_f, u_s, a, nb, tol, i_max, out, slot, ctr, s);
        case 8: return chol_dispatch<8>(u_f, u_s, a, nb, tol, i_max, out, slot, ctr, s);
        case 16: return chol_dispatch<16>(u_f, u_s, a, nb, tol, i_max, out, slot, ctr, s);
        case 32: return chol_dispatch<32>(u_f, u_s, a, nb, tol, i_max, out, slot, ctr, s);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace mlmc
