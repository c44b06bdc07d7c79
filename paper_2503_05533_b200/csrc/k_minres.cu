// k_minres.cu -- K3: batched, on-chip-resident MINRES for the P1 systems of one mesh level.
//
// Method (paper): MINRES minimises ||b - A x_k||_2 over x0 + K_k(A, r0),
// all arithmetic in binary64, stopped on the relative residual
// ||b - A x_k|| / ||b|| <= tol (Eq. (2); C = 1, R9), x0 = 0,
// no preconditioner (R9).  The Lanczos/Givens recurrences are Paige-Saunders'
// (the same quantities alpha, beta, delta, gbar, epsilon, phibar as the oracle).
//
// Operator (R10): P1 stiffness on the uniform SW-NE triangulation with
// the centroid coefficient rule equals the 5-point stencil with edge
// conductances c = mean of the two triangles sharing the edge:
//   cE(i,j) = (aL(i,j) + aU(i,j-1))/2   cN(i,j) = (aU(i,j) + aL(i-1,j))/2
//   (A v)_ij = d v_ij - cE(i,j) v_{i+1,j} - cE(i-1,j) v_{i-1,j}
//                     - cN(i,j) v_{i,j+1} - cN(i,j-1) v_{i,j-1},  d = sum of the four.
// b = h^2 1 (int phi_i for f = 1) and Q = int u_h = h^2 sum_i x_i.
//
// B200 mapping: one thread group (a warp, two warps, or a whole CTA) owns one
// system at a time; every vector lives in registers, NPT nodes per thread,
// node p = t + k*T (coalesced, conflict-free shared-memory rows); only the
// Lanczos vector r2 is exchanged through a zero-padded (N+1)^2 shared grid for
// the stencil.  Two group reductions per iteration (alpha, ||r2||^2), each one
// barrier: the r2 exchange rides on the ||r2|| barrier.  Reductions are xor
// butterflies, so every thread holds bit-identical scalars and the stopping
// decision is uniform.  Groups pull systems from an atomic job counter
// (iteration counts vary by ~2x between samples).
#include <cuda_runtime.h>
#include <cfloat>
#include <cstdint>

#include "internal.h"

namespace mlmc {

__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int T, int GROUPS>
__device__ __forceinline__ void group_sync(int g) {
    if constexpr (T == 32) {
        __syncwarp();
    } else if constexpr (GROUPS == 1) {
        __syncthreads();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(T) : "memory");
    }
}

// Sum over the T threads of a group; identical bits in every thread.
template <int T, int GROUPS>
__device__ __forceinline__ double group_sum(double v, double* buf, int tg, int g) {
    v = warp_allsum(v);
    if constexpr (T == 32) {
        __syncwarp();      // memory ordering of the shared grid across lanes
        return v;
    } else {
        if ((tg & 31) == 0) buf[tg >> 5] = v;
        group_sync<T, GROUPS>(g);
        double s = ((tg & 31) < T / 32) ? buf[tg & 31] : 0.0;
        return warp_allsum(s);
    }
}

template <int N, int T, int NPT, bool CSMEM>
struct MinresCfg {
    static constexpr int n = (N - 1) * (N - 1);
    static constexpr int G = N + 1;                           // padded grid pitch
    static constexpr int GROUPS = T >= 128 ? 1 : 128 / T;     // CTA = 128 threads for small groups
    static constexpr int BLOCK = T * GROUPS;
    static constexpr int RED = T / 32 < 1 ? 1 : T / 32;
    // per-group shared doubles: grid, 2 reduction buffers (+2 spare), coefficient grids
    static constexpr int SMEM_PER_GROUP = G * G + 2 * RED + 2 + (CSMEM ? 2 * N * N : 0);
    static constexpr size_t SMEM = sizeof(double) * SMEM_PER_GROUP * GROUPS + 16 * GROUPS;
    static_assert(NPT * T >= n, "not enough node slots");
};

template <int N, int T, int NPT, bool CSMEM>
__global__ void __launch_bounds__(MinresCfg<N, T, NPT, CSMEM>::BLOCK)
minres_kernel(const double* __restrict__ a_all, int nb, double tol, int max_iter, double* __restrict__ out,
              int slot, unsigned* __restrict__ job_counter) {
    using C = MinresCfg<N, T, NPT, CSMEM>;
    constexpr int G = C::G, n = C::n, P = 2 * N * N;
    extern __shared__ double smem[];
    const int g = threadIdx.x / T, tg = threadIdx.x % T;
    double* S = smem + g * C::SMEM_PER_GROUP;        // zero-padded (N+1)^2 grid
    double* redA = S + G * G;
    double* redB = redA + C::RED;
    double* cEg = redB + C::RED + 2;                 // CSMEM: cE, cN edge grids [j*N + i]
    double* cNg = cEg + N * N;
    int* jobslot = reinterpret_cast<int*>(smem + C::SMEM_PER_GROUP * C::GROUPS) + 4 * g;

    const double h = 1.0 / N, h2 = h * h;

    // node geometry (fixed per thread)
    int cidx[NPT];
    bool own[NPT];
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
        int p = tg + q * T;
        own[q] = p < n;
        int pp = own[q] ? p : 0;
        int i = pp % (N - 1) + 1, j = pp / (N - 1) + 1;
        cidx[q] = j * G + i;
    }

    for (;;) {
        if (tg == 0) *jobslot = (int)atomicAdd(job_counter, 1u);
        group_sync<T, C::GROUPS>(g);
        const int job = *jobslot;
        if (job >= nb) break;
        const double* a = a_all + (size_t)job * P;

        // ---- prologue: zero the padded grid, build the stencil coefficients
        for (int e = tg; e < G * G; e += T) S[e] = 0.0;
        double cEo[CSMEM ? 1 : NPT], cWo[CSMEM ? 1 : NPT], cNo[CSMEM ? 1 : NPT], cSo[CSMEM ? 1 : NPT];
        if constexpr (CSMEM) {
            for (int e = tg; e < N * N; e += T) {
                int i = e % N, j = e / N;
                // edge (i,j)-(i+1,j): lower tri of cell (i,j) + upper tri of cell (i,j-1)
                cEg[e] = (j >= 1) ? 0.5 * (__ldg(a + 2 * (j * N + i)) + __ldg(a + 2 * ((j - 1) * N + i) + 1)) : 0.0;
                // edge (i,j)-(i,j+1): upper tri of cell (i,j) + lower tri of cell (i-1,j)
                cNg[e] = (i >= 1) ? 0.5 * (__ldg(a + 2 * (j * N + i) + 1) + __ldg(a + 2 * (j * N + i - 1))) : 0.0;
            }
        } else {
#pragma unroll
            for (int q = 0; q < NPT; ++q) {
                int c = cidx[q], i = c % G, j = c / G;
                auto aL = [&](int ci, int cj) { return __ldg(a + 2 * (cj * N + ci)); };
                auto aU = [&](int ci, int cj) { return __ldg(a + 2 * (cj * N + ci) + 1); };
                cEo[q] = 0.5 * (aL(i, j) + aU(i, j - 1));
                cWo[q] = 0.5 * (aL(i - 1, j) + aU(i - 1, j - 1));
                cNo[q] = 0.5 * (aU(i, j) + aL(i - 1, j));
                cSo[q] = 0.5 * (aU(i, j - 1) + aL(i - 1, j - 1));
            }
        }
        group_sync<T, C::GROUPS>(g);

        // ---- MINRES state: r1 = r2 = b, w = w2 = x = 0
        double r1[NPT], r2[NPT], w[NPT], w2[NPT], x[NPT];
        double part = 0.0;
#pragma unroll
        for (int q = 0; q < NPT; ++q) {
            double bq = own[q] ? h2 : 0.0;
            r1[q] = bq; r2[q] = bq; w[q] = 0.0; w2[q] = 0.0; x[q] = 0.0;
            if (own[q]) S[cidx[q]] = bq;
            part = fma(bq, bq, part);
        }
        const double beta1 = sqrt(group_sum<T, C::GROUPS>(part, redA, tg, g));   // barrier: S holds b
        double beta = beta1, oldb = 0.0, dbar = 0.0, epsln = 0.0, phibar = beta1, cs = -1.0, sn = 0.0;
        int k = 0, status = 1;
        if (beta1 == 0.0) status = 0;
        while (status == 1 && k < max_iter) {
            ++k;
            const double invb = 1.0 / beta;
            const double cr1 = (k >= 2) ? beta / oldb : 0.0;
            // y = A v - (beta/oldb) r1, v = r2/beta; y is parked in r1 (r1 is dead afterwards)
            part = 0.0;
#pragma unroll
            for (int q = 0; q < NPT; ++q) {
                if (!own[q]) continue;
                const int c = cidx[q];
                double cE, cW, cN, cS;
                if constexpr (CSMEM) {
                    const int i = c % G, j = c / G, e = j * N + i;
                    cE = cEg[e]; cW = cEg[e - 1]; cN = cNg[e]; cS = cNg[e - N];
                } else {
                    cE = cEo[q]; cW = cWo[q]; cN = cNo[q]; cS = cSo[q];
                }
                const double d = (cE + cW) + (cN + cS);
                double Av = d * S[c];
                Av = fma(-cE, S[c + 1], Av);
                Av = fma(-cW, S[c - 1], Av);
                Av = fma(-cN, S[c + G], Av);
                Av = fma(-cS, S[c - G], Av);
                const double v = r2[q] * invb;
                const double y = fma(-cr1, r1[q], Av * invb);
                r1[q] = y;
                part = fma(v, y, part);
            }
            const double alpha = group_sum<T, C::GROUPS>(part, redA, tg, g);   // all stencil reads done
            const double ca = alpha / beta;
            part = 0.0;
#pragma unroll
            for (int q = 0; q < NPT; ++q) {
                if (!own[q]) continue;
                const double y = fma(-ca, r2[q], r1[q]);
                r1[q] = r2[q];
                r2[q] = y;
                S[cidx[q]] = y;
                part = fma(y, y, part);
            }
            const double bb = group_sum<T, C::GROUPS>(part, redB, tg, g);      // S holds the new r2
            oldb = beta;
            beta = sqrt(bb);
            // Givens rotation (Paige-Saunders)
            const double oldeps = epsln;
            const double delta = cs * dbar + sn * alpha;
            const double gbar = sn * dbar - cs * alpha;
            epsln = sn * beta;
            dbar = -cs * beta;
            double gamma = hypot(gbar, beta);
            gamma = gamma < DBL_MIN ? DBL_MIN : gamma;
            cs = gbar / gamma;
            sn = beta / gamma;
            const double phi = cs * phibar;
            phibar = sn * phibar;
            const double invg = 1.0 / gamma;
#pragma unroll
            for (int q = 0; q < NPT; ++q) {
                const double v = r1[q] * invb;            // r1 now holds the previous r2: v_k
                const double w1 = w2[q];
                w2[q] = w[q];
                w[q] = (v - oldeps * w1 - delta * w2[q]) * invg;
                x[q] = fma(phi, w[q], x[q]);
            }
            if (!(phibar == phibar) || !(beta == beta)) status = 3;
            else if (phibar / beta1 <= tol) status = 0;
        }
        // ---- epilogue: Q = h^2 sum x and the true residual ||b - A x|| / ||b||
        // (every stencil read of S finished before the last barrier)
#pragma unroll
        for (int q = 0; q < NPT; ++q)
            if (own[q]) S[cidx[q]] = x[q];
        group_sync<T, C::GROUPS>(g);
        double sx = 0.0, rr = 0.0;
#pragma unroll
        for (int q = 0; q < NPT; ++q) {
            if (!own[q]) continue;
            const int c = cidx[q];
            double cE, cW, cN, cS;
            if constexpr (CSMEM) {
                const int i = c % G, j = c / G, e = j * N + i;
                cE = cEg[e]; cW = cEg[e - 1]; cN = cNg[e]; cS = cNg[e - N];
            } else {
                cE = cEo[q]; cW = cWo[q]; cN = cNo[q]; cS = cSo[q];
            }
            const double d = (cE + cW) + (cN + cS);
            double Ax = d * S[c];
            Ax = fma(-cE, S[c + 1], Ax);
            Ax = fma(-cW, S[c - 1], Ax);
            Ax = fma(-cN, S[c + G], Ax);
            Ax = fma(-cS, S[c - G], Ax);
            const double r = h2 - Ax;
            rr = fma(r, r, rr);
            sx += x[q];
        }
        sx = group_sum<T, C::GROUPS>(sx, redA, tg, g);
        rr = group_sum<T, C::GROUPS>(rr, redB, tg, g);
        if (tg == 0) {
            double* o = out + (size_t)job * kRecLen;
            o[0 + slot] = h2 * sx;
            o[2 + slot] = (double)k;
            o[4 + slot] = beta1 > 0.0 ? sqrt(rr) / beta1 : 0.0;
            o[6 + slot] = (double)status;
        }
        group_sync<T, C::GROUPS>(g);   // S / jobslot reuse
    }
}

template <int N, int T, int NPT, bool CSMEM>
static cudaError_t run_minres(const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                              unsigned* ctr, cudaStream_t s) {
    using C = MinresCfg<N, T, NPT, CSMEM>;
    auto kern = minres_kernel<N, T, NPT, CSMEM>;
    static int blocks_per_sm = -1, sms = 0;
    if (blocks_per_sm < 0) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, C::BLOCK, C::SMEM);
        if (e != cudaSuccess) return e;
        int dev;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (blocks_per_sm < 1) return cudaErrorInvalidConfiguration;
    }
    uint64_t need = (nb + C::GROUPS - 1) / C::GROUPS;
    uint64_t grid = std::min<uint64_t>(need, (uint64_t)blocks_per_sm * sms);
    if (grid == 0) return cudaSuccess;
    kern<<<(unsigned)grid, C::BLOCK, C::SMEM, s>>>(a, (int)nb, tol, max_iter, out, slot, ctr);
    return cudaGetLastError();
}

bool minres_supported(int N) { return N == 2 || N == 4 || N == 8 || N == 16 || N == 32 || N == 64; }

cudaError_t launch_minres(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                          unsigned* ctr, cudaStream_t s) {
    switch (N) {
        case 2:  return run_minres<2, 32, 1, false>(a, nb, tol, max_iter, out, slot, ctr, s);
        case 4:  return run_minres<4, 32, 1, false>(a, nb, tol, max_iter, out, slot, ctr, s);
        case 8:  return run_minres<8, 32, 2, false>(a, nb, tol, max_iter, out, slot, ctr, s);
        case 16: return run_minres<16, 64, 4, false>(a, nb, tol, max_iter, out, slot, ctr, s);
        case 32: return run_minres<32, 256, 4, false>(a, nb, tol, max_iter, out, slot, ctr, s);
        case 64: return run_minres<64, 512, 8, true>(a, nb, tol, max_iter, out, slot, ctr, s);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace mlmc
