// k_minres_gm.cu -- K3 for fine meshes (h <= 1/128): MINRES with the vectors in global memory.
//
// Same method and recurrences as k_minres.cu (Eq. (2); R9, R10, R26):
// unpreconditioned binary64 MINRES from x0 = 0 on the 5-point P1 operator,
// stopping on phibar_k/||b|| <= tol, Q from the scalar recurrence of 1^T x_k.
// A system of n = (N-1)^2 >= 16129 unknowns no longer fits one SM's registers
// and shared memory, so one CTA (512 threads) owns one system at a time and its
// r1, r2, w, w2 and the conductance grids live in a per-CTA global scratch
// (L2-resident for h = 1/128: 148 x 0.8 MB); r2 sits in a zero-padded
// (N+1)^2 grid so the stencil needs no branches.  Two block reductions per
// iteration; __syncthreads orders the global writes of one phase before the
// reads of the next.  This is the correctness path for the levels the
// benchmarked configurations never reach (streaming /
// cluster versions are NEXT).
#include <cuda_runtime.h>
#include <cfloat>
#include <cstdint>

#include "internal.h"

namespace mlmc {

constexpr int GMT = 512;

__device__ __forceinline__ double gm_block_sum(double v, double* buf) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = (threadIdx.x & 31) < GMT / 32 ? buf[threadIdx.x & 31] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

size_t minres_gm_scratch_per_cta(int N) {
#ifndef MLMC_TUNING
    (void)N;
    return 0;          // production build: K3c (k_minres_stream.cu) only; this kernel is an A/B variant
#endif
    const size_t G = (size_t)N + 1, n = (size_t)(N - 1) * (N - 1);
    return sizeof(double) * (3 * G * G + 3 * n) + 256;
}

#ifdef MLMC_TUNING
__global__ void __launch_bounds__(GMT) minres_gm_kernel(int N, const double* __restrict__ a_all, int nb, double tol,
                                                        int max_iter, double* __restrict__ out, int slot,
                                                        unsigned* __restrict__ job_counter, double* scratch,
                                                        size_t scratch_doubles) {
    __shared__ double redA[GMT / 32], redB[GMT / 32];
    __shared__ int jobslot;
    const int G = N + 1, C = N - 1, n = C * C, P = 2 * N * N;
    double* base = scratch + (size_t)blockIdx.x * scratch_doubles;
    double* r2g = base;                        // padded grid (N+1)^2, zero boundary
    double* cEg = r2g + (size_t)G * G;         // cE(i,j) at [j*G + i]
    double* cNg = cEg + (size_t)G * G;         // cN(i,j) at [j*G + i]
    double* r1 = cNg + (size_t)G * G;          // node-indexed p = (j-1)C + (i-1)
    double* w = r1 + n;
    double* w2 = w + n;
    const double h = 1.0 / N, h2 = h * h;

    for (;;) {
        if (threadIdx.x == 0) jobslot = (int)atomicAdd(job_counter, 1u);
        __syncthreads();
        const int job = jobslot;
        __syncthreads();
        if (job >= nb) break;
        const double* a = a_all + (size_t)job * P;
        for (int e = threadIdx.x; e < G * G; e += GMT) {
            const int ii = e % G, jj = e / G;
            r2g[e] = (ii >= 1 && ii < N && jj >= 1 && jj < N) ? h2 : 0.0;
            cEg[e] = (ii < N && jj >= 1 && jj < N) ? 0.5 * (__ldg(a + 2 * (jj * N + ii)) + __ldg(a + 2 * ((jj - 1) * N + ii) + 1)) : 0.0;
            cNg[e] = (ii >= 1 && ii < N && jj < N) ? 0.5 * (__ldg(a + 2 * (jj * N + ii) + 1) + __ldg(a + 2 * (jj * N + ii - 1))) : 0.0;
        }
        double pb = 0.0;
        for (int p = threadIdx.x; p < n; p += GMT) {
            r1[p] = h2;
            w[p] = 0.0;
            w2[p] = 0.0;
            pb = fma(h2, h2, pb);
        }
        pb = gm_block_sum(pb, redB);
        double invb = pb > 0.0 ? rsqrt(pb) : 0.0;
        const double beta1 = pb > 0.0 ? pb * invb : 0.0, inv_beta1 = invb, tol_b = tol * beta1;
        double beta = beta1, inv_oldb = 0.0, dbar = 0.0, epsln = 0.0, phibar = beta1, cs = -1.0, sn = 0.0, Xt = 0.0;
        int k = 0, status = beta1 == 0.0 ? 0 : 1;
        while (status == 1 && k < max_iter) {
            ++k;
            const double cr1 = k >= 2 ? beta * inv_oldb : 0.0;
            double pa = 0.0;
            for (int p = threadIdx.x; p < n; p += GMT) {
                const int i = p % C + 1, j = p / C + 1, c = j * G + i;
                const double ce = cEg[c], cw = cEg[c - 1], cn = cNg[c], csth = cNg[c - G];
                const double d = (ce + cw) + (cn + csth);
                const double vC = r2g[c];
                const double t = fma(ce, r2g[c + 1], cw * r2g[c - 1]);
                const double u = fma(cn, r2g[c + G], csth * r2g[c - G]);
                const double Av = fma(d, vC, -(t + u));
                const double y = fma(Av, invb, -(cr1 * r1[p]));
                r1[p] = y;
                pa = fma(vC * invb, y, pa);
            }
            const double alpha = gm_block_sum(pa, redA);
            const double ca = alpha * invb;
            double pbb = 0.0;
            for (int p = threadIdx.x; p < n; p += GMT) {
                const int c = (p / C + 1) * G + p % C + 1;
                const double old = r2g[c];
                const double y = fma(-ca, old, r1[p]);
                r1[p] = old;
                r2g[c] = y;
                pbb = fma(y, y, pbb);
            }
            pbb = gm_block_sum(pbb, redB);
            const double invb_k = invb;
            inv_oldb = invb;
            invb = pbb > 0.0 ? rsqrt(pbb) : 0.0;
            beta = pbb > 0.0 ? pbb * invb : 0.0;
            const double oldeps = epsln;
            const double delta = cs * dbar + sn * alpha;
            const double gbar = sn * dbar - cs * alpha;
            epsln = sn * beta;
            dbar = -cs * beta;
            const double gg = fma(gbar, gbar, beta * beta);
            const double invg = gg > 0.0 ? rsqrt(gg) : 1.0 / DBL_MIN;
            cs = gbar * invg;
            sn = beta * invg;
            const double phi = cs * phibar;
            phibar = sn * phibar;
            double sw = 0.0;
            for (int p = threadIdx.x; p < n; p += GMT) {
                const double v = r1[p] * invb_k;
                const double w1 = w2[p];
                const double wo = w[p];
                const double wn = fma(-delta, wo, fma(-oldeps, w1, v)) * invg;
                w2[p] = wo;
                w[p] = wn;
                sw += wn;
            }
            Xt = fma(phi, sw, Xt);
            if (!(phibar == phibar) || !(beta == beta)) status = 3;
            else if (phibar <= tol_b) status = 0;
        }
        const double X = gm_block_sum(Xt, redA);
        if (threadIdx.x == 0) {
            double* o = out + (size_t)job * kRecLen;
            o[0 + slot] = h2 * X;
            o[2 + slot] = (double)k;
            o[4 + slot] = phibar * inv_beta1;
            o[6 + slot] = (double)status;
        }
        __syncthreads();
    }
}

#endif  // MLMC_TUNING

cudaError_t launch_minres_gm(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                             unsigned* ctr, double* scratch, int nctas, cudaStream_t s) {
    if (nb == 0) return cudaSuccess;
#ifndef MLMC_TUNING
    (void)N; (void)a; (void)tol; (void)max_iter; (void)out; (void)slot; (void)ctr; (void)scratch; (void)nctas; (void)s;
    return cudaErrorNotSupported;
#else
    const int grid = (int)std::min<uint64_t>(nb, (uint64_t)nctas);
    minres_gm_kernel<<<grid, GMT, 0, s>>>(N, a, (int)nb, tol, max_iter, out, slot, ctr, scratch,
                                          minres_gm_scratch_per_cta(N) / sizeof(double));
    return cudaGetLastError();
#endif
}

}  // namespace mlmc
