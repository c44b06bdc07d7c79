// k_minres.cu -- K3: batched, register-resident MINRES for the P1 systems of one mesh level.
//
// Method (paper): MINRES minimises ||b - A x_k||_2 over x0 + K_k(A, r0),
// all arithmetic in binary64, stopped on the relative residual
// ||b - A x_k|| / ||b|| <= tol (Eq. (2); C = 1, R9), x0 = 0,
// no preconditioner (R9).  Lanczos + Givens recurrences of Paige & Saunders
// (alpha, beta, delta, gbar, epsilon, phibar -- the oracle's quantities).
//
// Operator (R10): P1 stiffness on the uniform SW-NE triangulation with
// the centroid coefficient rule = 5-point stencil with edge conductances
//   cE(i,j) = (aL(i,j) + aU(i,j-1))/2   cN(i,j) = (aU(i,j) + aL(i-1,j))/2
//   (A v)_ij = d v_ij - cE(i,j) v_{i+1,j} - cE(i-1,j) v_{i-1,j}
//                     - cN(i,j) v_{i,j+1} - cN(i,j-1) v_{i,j-1},  d = sum of the four.
// b = h^2 1 and Q = int u_h = h^2 sum_i x_i.
//
// QoI without storing the iterate (R26): x_k = x_{k-1} + phi_k w_k, so each
// thread keeps only X_t = sum of its own entries of x_k, updated by
// X_t += phi_k * (sum of its entries of w_k); Q = h^2 * (group sum of X_t) once
// at the end.  The VERIFY instantiation also carries x_k itself and reports the
// true residual ||b - A x_k|| / ||b||, with bit-identical Q.
//
// B200 mapping (column strips): a thread owns R consecutive rows of one grid
// column; its Lanczos vectors r1, r2, directions w, w2 and its stencil
// conductances stay in registers for the whole solve.  North/south neighbours
// are the thread's own registers except at strip ends; east/west neighbours
// and strip-end rows come through a zero-padded shared grid written once per
// iteration.  R is chosen so that the strips cover rows 1..N: the only
// non-node row is the boundary row N at the top of the last strip (a
// "phantom" row whose Lanczos entries are forced to 0 by a select), so the hot
// loops carry no branches.  Groups: one warp per system for h >= 1/16 (strips
// packed into the lanes), a 4-warp CTA for 1/32, a 16-warp CTA for 1/64.
// Two group reductions per iteration (alpha, ||r2||^2), xor butterflies so
// every thread holds bit-identical scalars (uniform stopping); the scalar
// chain between them uses rsqrt instead of sqrt + division.  Groups pull
// systems from an atomic job counter.
#include <cuda_runtime.h>
#include <cfloat>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "internal.h"

namespace mlmc {

__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Thread layout of one system: S strips of R rows; for C <= 32 columns a warp
// carries SPW = floor(32 / C) strips side by side (lane = strip * C + column),
// for C > 32 a strip spans WPR warps (lane = column).  Idle lanes act as a
// phantom strip S (zeros) and never touch a node's cell.
template <int N, int R, int MINB_, bool CS_ = false>
struct StripCfg {
    static constexpr bool CS = CS_;                       // all conductances from shared grids (frees registers)
    static constexpr int C = N - 1;                       // interior columns / rows
    static constexpr int S = (C + R - 1) / R;             // strips per column
    static constexpr bool NARROW = C <= 32;
    static constexpr int SPW = NARROW ? 32 / C : 1;       // strips per warp
    static constexpr int WPR = NARROW ? 1 : (C + 31) / 32;
    static constexpr int NW = NARROW ? (S + SPW - 1) / SPW : S * WPR;   // warps per system
    static constexpr int TPG = 32 * NW;                   // threads per system
    static constexpr int GROUPS = TPG >= 128 ? 1 : 128 / TPG;
    static constexpr int BLOCK = TPG * GROUPS;
    static constexpr int MINB = MINB_;                    // resident CTAs per SM the register budget must allow
    static constexpr int G = NARROW ? N + 1 : 32 * WPR + 2;   // grid pitch
    static constexpr int GR = S * R + R + 2;              // grid rows (phantom strip S for idle lanes)
    static constexpr bool CW_SMEM = CS || N >= 32;        // west conductance from the shared cE grid
    static constexpr int GP = 32 * WPR + 2 > N + 2 ? 32 * WPR + 2 : N + 2;   // conductance grid pitch
    // cE (and with CS cN) grids [row * GP + col], rows 0..GR-1; entries that are not edges hold 0
    static constexpr int SMEM_PER_GROUP = G * GR + 2 * NW + 2 + (CW_SMEM ? GP * GR : 0) + (CS ? GP * GR : 0);
    static constexpr size_t SMEM = sizeof(double) * SMEM_PER_GROUP * GROUPS + 16 * GROUPS;
    static_assert(S * R == C || S * R == C + 1, "strips must end at row C or at the boundary row N");
};

template <int TPG, int GROUPS>
__device__ __forceinline__ void gsync(int g) {
    if constexpr (TPG == 32) {
        __syncwarp();
    } else if constexpr (GROUPS == 1) {
        __syncthreads();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(TPG) : "memory");
    }
}

// Sum over the group; bit-identical in every thread.
template <int TPG, int GROUPS>
__device__ __forceinline__ double gsum(double a, double* buf, int tg, int g) {
    a = warp_allsum(a);
    if constexpr (TPG == 32) {
        __syncwarp();
        return a;
    } else {
        constexpr int NW = TPG / 32;
        if ((tg & 31) == 0) buf[tg >> 5] = a;
        gsync<TPG, GROUPS>(g);
        double s = ((tg & 31) < NW) ? buf[tg & 31] : 0.0;
        return warp_allsum(s);
    }
}

template <int N, int R, int MINB, bool VERIFY, bool PIPE, bool CS>
__global__ void __launch_bounds__(StripCfg<N, R, MINB, CS>::BLOCK, MINB)
minres_strip_kernel(const double* __restrict__ a_all, int nb, double tol, int max_iter, double* __restrict__ out,
                    int slot, unsigned* __restrict__ job_counter) {
    using K = StripCfg<N, R, MINB, CS>;
    constexpr int GP = K::GP;
    constexpr int C = K::C, G = K::G, TPG = K::TPG, GROUPS = K::GROUPS, NW = K::NW, P = 2 * N * N;
    extern __shared__ double smem[];
    const int g = threadIdx.x / TPG, tg = threadIdx.x % TPG;
    double* Sg = smem + g * K::SMEM_PER_GROUP;          // zero-padded exchange grid [row * G + col]
    double* redA = Sg + G * K::GR;                       // alpha partials
    double* redB = redA + NW;                            // ||r2||^2 partials
    double* cEg = redB + NW + 2;                         // CW_SMEM: cE edge grid [j*GP + i]
    double* cNg = cEg + GP * K::GR;                      // CS: cN edge grid [j*GP + i]
    int* jobslot = reinterpret_cast<int*>(smem + K::SMEM_PER_GROUP * GROUPS) + 4 * g;

    // ---- this thread's strip: column i, rows j0 .. j0 + R - 1 (nrows of them are nodes)
    int s, ci;
    bool live;
    if constexpr (K::NARROW) {
        const int w = tg >> 5, l = tg & 31;
        s = w * K::SPW + l / C;
        ci = l % C;
        live = l < K::SPW * C && s < K::S;
        if (!live) s = K::S;                              // idle lane: phantom strip
    } else {
        s = tg / (32 * K::WPR);
        ci = tg % (32 * K::WPR);
        live = ci < C;                                    // idle lanes: columns N.. (zeros)
    }
    const int i = ci + 1, j0 = s * R + 1;
    const int nrows = live ? min(R, C - s * R) : 0;      // R, R-1 (phantom top row) or 0
    const bool live_last = nrows == R;                    // is row R-1 a node?
    const int c0 = j0 * G + i;                            // grid index of the strip's first row
    const double h = 1.0 / N, h2 = h * h;

    for (;;) {
        if (tg == 0) *jobslot = (int)atomicAdd(job_counter, 1u);
        gsync<TPG, GROUPS>(g);
        const int job = *jobslot;
        gsync<TPG, GROUPS>(g);
        if (job >= nb) break;
        const double* a = a_all + (size_t)job * P;

        // ---- prologue: zero the exchange grid, load conductances (registers + cE grid)
        for (int e = tg; e < G * K::GR; e += TPG) Sg[e] = 0.0;
        auto aL = [&](int ii, int jj) { return __ldg(a + 2 * (jj * N + ii)); };
        auto aU = [&](int ii, int jj) { return __ldg(a + 2 * (jj * N + ii) + 1); };
        if constexpr (K::CW_SMEM) {
            for (int e = tg; e < GP * K::GR; e += TPG) {
                const int ii = e % GP, jj = e / GP;
                // edge (ii,jj)-(ii+1,jj): lower tri of cell (ii,jj) + upper tri of cell (ii,jj-1)
                cEg[e] = (ii < N && jj >= 1 && jj < N) ? 0.5 * (aL(ii, jj) + aU(ii, jj - 1)) : 0.0;
                // edge (ii,jj)-(ii,jj+1): upper tri of cell (ii,jj) + lower tri of cell (ii-1,jj)
                if constexpr (K::CS) cNg[e] = (ii >= 1 && ii < N && jj < N) ? 0.5 * (aU(ii, jj) + aL(ii - 1, jj)) : 0.0;
            }
        }
        constexpr int RR = K::CS ? 1 : R;
        double cE[RR], cN[RR], cW[K::CW_SMEM ? 1 : R];
        double cS0 = 0.0, cSlast = 0.0;
#pragma unroll
        for (int r = 0; r < RR; ++r) {
            cE[r] = 0.0;
            cN[r] = 0.0;
            if constexpr (!K::CW_SMEM) cW[K::CW_SMEM ? 0 : r] = 0.0;
            if (!K::CS && r < nrows) {
                const int j = j0 + r;
                cE[r] = 0.5 * (aL(i, j) + aU(i, j - 1));
                cN[r] = 0.5 * (aU(i, j) + aL(i - 1, j));
                if constexpr (!K::CW_SMEM) cW[K::CW_SMEM ? 0 : r] = 0.5 * (aL(i - 1, j) + aU(i - 1, j - 1));
            }
        }
        if (nrows > 0) cS0 = 0.5 * (aU(i, j0 - 1) + aL(i - 1, j0 - 1));
        // South conductance of the strip's top row: 0 if that row is the phantom boundary row,
        // which then has only zero couplings and zero entries, so its y stays exactly 0.
        if (R > 1 && live_last) cSlast = 0.5 * (aU(i, j0 + R - 2) + aL(i - 1, j0 + R - 2));
        if (R == 1) cSlast = cS0;
        gsync<TPG, GROUPS>(g);

        // ---- MINRES state: r1 = r2 = b, w = w2 = 0 (x itself only in VERIFY)
        double r1[R], r2[R], w[R], w2[R], x[VERIFY ? R : 1];
        double pb = 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const bool alive = (r < R - 1) ? live : live_last;
            const double bq = alive ? h2 : 0.0;
            r1[r] = bq; r2[r] = bq; w[r] = 0.0; w2[r] = 0.0;
            if constexpr (VERIFY) x[VERIFY ? r : 0] = 0.0;
            Sg[c0 + r * G] = bq;
            pb = fma(bq, bq, pb);
        }
        pb = gsum<TPG, GROUPS>(pb, redB, tg, g);           // barrier: the grid holds b
        double invb = pb > 0.0 ? rsqrt(pb) : 0.0;          // 1/beta_k
        const double beta1 = pb > 0.0 ? pb * invb : 0.0;
        const double inv_beta1 = invb, tol_b = tol * beta1;
        double beta = beta1, inv_oldb = 0.0, dbar = 0.0, epsln = 0.0, phibar = beta1, cs = -1.0, sn = 0.0;
        double Xt = 0.0;                                    // this thread's share of 1^T x_k
        // Software pipeline: the direction/solution update of iteration k (phase C) and
        // the stencil + alpha partial of iteration k+1 (phase A) are independent, so they
        // share one pass over the rows after the ||r2|| reduction; the Givens scalar
        // chain of k hides behind the stencil of k+1.  Same operations, same order per
        // value as the plain loop.
        const double* Sc = Sg + c0;
        // CW_SMEM: [r*GP] west, [r*GP + 1] own (CS) cE.  An idle lane of a wide layout sits in
        // column N: it reads the all-zero columns N, N+1 so that its entries stay exactly 0.
        const double* cEw = cEg + j0 * GP + (live ? i - 1 : i);
        const double* cNw = cNg + j0 * GP + i;              // CS: [r*GP] own cN
        // conductances of row r: east, west, north, south (south of row r = north of row r-1)
        auto coef = [&](int r, double& ce, double& cw, double& cn, double& cs_) {
            if constexpr (K::CS) {
                ce = cEw[r * GP + 1];
                cn = cNw[r * GP];
            } else {
                ce = cE[K::CS ? 0 : r];
                cn = cN[K::CS ? 0 : r];
            }
            if constexpr (K::CW_SMEM) cw = cEw[r * GP]; else cw = cW[K::CW_SMEM ? 0 : r];
            if (r == R - 1) cs_ = cSlast;
            else if (r == 0) cs_ = cS0;
            else if constexpr (K::CS) cs_ = cNw[(r - 1) * GP];
            else cs_ = cN[K::CS ? 0 : r - 1];
        };
        // phase A of iteration k: y = A v - cr1 r1, v = r2 * invb; y parked in r1; alpha partial
        auto phaseA = [&](int r, double cr1, double& pa) {
            const double vC = r2[r];
            const double vN = (r + 1 < R) ? r2[r + 1 < R ? r + 1 : r] : Sc[r * G + G];
            const double vS = (r > 0) ? r2[r > 0 ? r - 1 : 0] : Sc[-G];
            const double vE = Sc[r * G + 1], vW = Sc[r * G - 1];
            double ce, cw_, cn, cs_;
            coef(r, ce, cw_, cn, cs_);
            const double d = (ce + cw_) + (cn + cs_);
            const double t = fma(ce, vE, cw_ * vW);
            const double u = fma(cn, vN, cs_ * vS);
            const double Av = fma(d, vC, -(t + u));
            const double y = fma(Av, invb, -(cr1 * r1[r]));
            r1[r] = y;
            pa = fma(vC * invb, y, pa);
        };
        int k = 1, status = 1;
        double pa0 = 0.0, pa1 = 0.0;
        if (beta1 == 0.0) {
            status = 0;
            k = 0;
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) phaseA(r, 0.0, (r & 1) ? pa1 : pa0);
        }
        while (status == 1) {
            const double alpha = gsum<TPG, GROUPS>(pa0 + pa1, redA, tg, g);   // all grid reads done
            const double ca = alpha * invb;
            double pb0 = 0.0, pb1 = 0.0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double y = fma(-ca, r2[r], r1[r]);    // phantom rows: 0 - ca * 0
                r1[r] = r2[r];
                r2[r] = y;
                Sg[c0 + r * G] = y;
                if (r & 1) pb1 = fma(y, y, pb1); else pb0 = fma(y, y, pb0);
            }
            const double pbb = gsum<TPG, GROUPS>(pb0 + pb1, redB, tg, g);   // grid holds the new r2
            const double invb_k = invb;                    // v_k = r1 / beta_k below
            inv_oldb = invb;
            invb = pbb > 0.0 ? rsqrt(pbb) : 0.0;
            beta = pbb > 0.0 ? pbb * invb : 0.0;
            // ---- Givens rotation (Paige-Saunders); gamma = hypot(gbar, beta)
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
            if (!(phibar == phibar) || !(beta == beta)) status = 3;
            else if (phibar <= tol_b) status = 0;           // phibar / ||b|| <= tol
            const bool more = status == 1 && k < max_iter;  // uniform across the group
            // phase C of iteration k (r1 holds the previous r2, v_k = r1 * invb_k) fused with
            // phase A of iteration k+1 (which then parks its y in r1)
            double sw = 0.0;
            auto phaseC = [&](int r) {
                const double v = r1[r] * invb_k;
                const double w1 = w2[r];
                w2[r] = w[r];
                w[r] = fma(-delta, w2[r], fma(-oldeps, w1, v)) * invg;
                sw += w[r];
                if constexpr (VERIFY) x[VERIFY ? r : 0] = fma(phi, w[r], x[VERIFY ? r : 0]);
            };
            if (!more) {
#pragma unroll
                for (int r = 0; r < R; ++r) phaseC(r);
                Xt = fma(phi, sw, Xt);
                break;
            }
            const double cr1 = beta * inv_oldb;            // beta_{k+1} / beta_k
            pa0 = 0.0;
            pa1 = 0.0;
            if constexpr (PIPE) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    phaseC(r);
                    phaseA(r, cr1, (r & 1) ? pa1 : pa0);
                }
            } else {                                        // fewer live registers
#pragma unroll
                for (int r = 0; r < R; ++r) phaseC(r);
#pragma unroll
                for (int r = 0; r < R; ++r) phaseA(r, cr1, (r & 1) ? pa1 : pa0);
            }
            Xt = fma(phi, sw, Xt);
            ++k;
        }
        double relres = phibar * inv_beta1;
        const double X = gsum<TPG, GROUPS>(Xt, redA, tg, g);
        if constexpr (VERIFY) {
            // true residual ||b - A x|| / ||b|| (every grid read of the loop precedes a later barrier)
#pragma unroll
            for (int r = 0; r < R; ++r) Sg[c0 + r * G] = x[VERIFY ? r : 0];
            gsync<TPG, GROUPS>(g);
            double rr = 0.0;
            const double* Sc = Sg + c0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const bool alive = (r < R - 1) ? live : live_last;
                double ce, cw_, cn, cs_;
                coef(r, ce, cw_, cn, cs_);
                const double d = (ce + cw_) + (cn + cs_);
                double Ax = d * Sc[r * G];
                Ax = fma(-ce, Sc[r * G + 1], Ax);
                Ax = fma(-cw_, Sc[r * G - 1], Ax);
                Ax = fma(-cn, Sc[r * G + G], Ax);
                Ax = fma(-cs_, Sc[r * G - G], Ax);
                const double res = alive ? h2 - Ax : 0.0;
                rr = fma(res, res, rr);
            }
            rr = gsum<TPG, GROUPS>(rr, redB, tg, g);
            relres = sqrt(rr) * inv_beta1;
        }
        if (tg == 0) {
            double* o = out + (size_t)job * kRecLen;
            o[0 + slot] = h2 * X;
            o[2 + slot] = (double)k;
            o[4 + slot] = relres;
            o[6 + slot] = (double)status;
        }
        gsync<TPG, GROUPS>(g);      // grid reuse by the next job
    }
}

template <int N, int R, int MINB, bool VERIFY, bool PIPE = true, bool CS = false>
static cudaError_t run_minres(const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                              unsigned* ctr, cudaStream_t s) {
    using K = StripCfg<N, R, MINB, CS>;
    auto kern = minres_strip_kernel<N, R, MINB, VERIFY, PIPE, CS>;
    static PerDevice<KernelOcc> occ_cache;
    const KernelOcc occ = occ_of(occ_cache, kern, K::BLOCK, K::SMEM);
    if (occ.err != cudaSuccess) return occ.err;
    uint64_t need = (nb + K::GROUPS - 1) / K::GROUPS;
    uint64_t grid = std::min<uint64_t>(need, (uint64_t)occ.per_sm * occ.sms);
    if (grid == 0) return cudaSuccess;
    kern<<<(unsigned)grid, K::BLOCK, K::SMEM, s>>>(a, (int)nb, tol, max_iter, out, slot, ctr);
    return cudaGetLastError();
}

bool minres_supported(int N) {
    return N == 2 || N == 4 || N == 8 || N == 16 || N == 32 || N == 64 || N == 128 || N == 256 || N == 512;
}

// Kernel shape per mesh (rows per thread R, register budget MINB); alternatives
// selectable with MLMC_MINRES_VARIANT_N<N>=<index> for tuning runs.
[[maybe_unused]] static int variant(int N) {
    static int v[8] = {-2, -2, -2, -2, -2, -2, -2, -2};
    int slot = N == 8 ? 0 : N == 16 ? 1 : N == 32 ? 2 : N == 64 ? 3 : 4;
    if (v[slot] == -2) {
        char name[64];
        std::snprintf(name, sizeof(name), "MLMC_MINRES_VARIANT_N%d", N);
        const char* e = std::getenv(name);
        v[slot] = e ? std::atoi(e) : 0;
    }
    return v[slot];
}

template <bool V>
static cudaError_t minres_dispatch(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out,
                                   int slot, unsigned* ctr, cudaStream_t s) {
    const int var = variant(N);
    switch (N) {
        case 2:  return run_minres<2, 1, 8, V>(a, nb, tol, max_iter, out, slot, ctr, s);
        case 4:  return run_minres<4, 1, 8, V>(a, nb, tol, max_iter, out, slot, ctr, s);
#ifdef MLMC_TUNING
        case 8:
            if (var == 1) return run_minres<8, 2, 6, V, false>(a, nb, tol, max_iter, out, slot, ctr, s);
            if (var == 2) return run_minres<8, 2, 8, V>(a, nb, tol, max_iter, out, slot, ctr, s);
            return run_minres<8, 2, 6, V>(a, nb, tol, max_iter, out, slot, ctr, s);
        case 16:
            if (var == 1) return run_minres<16, 8, 2, V, false>(a, nb, tol, max_iter, out, slot, ctr, s);
            if (var == 2) return run_minres<16, 8, 3, V>(a, nb, tol, max_iter, out, slot, ctr, s);
            if (var == 3) return run_minres<16, 4, 4, V>(a, nb, tol, max_iter, out, slot, ctr, s);
            return run_minres<16, 8, 2, V>(a, nb, tol, max_iter, out, slot, ctr, s);
        case 32:
            // measured (tools/tune_minres.py, configs[1] level 2): v0 1.00 ms, v1 1.14, v2 1.14, v3 1.01
            if (var == 1) return run_minres<32, 8, 3, V, true>(a, nb, tol, max_iter, out, slot, ctr, s);
            if (var == 2) return run_minres<32, 8, 4, V, true, true>(a, nb, tol, max_iter, out, slot, ctr, s);
            if (var == 3) return run_minres<32, 16, 2, V, true, true>(a, nb, tol, max_iter, out, slot, ctr, s);
            return run_minres<32, 8, 3, V, false>(a, nb, tol, max_iter, out, slot, ctr, s);
        case 64:
            // measured (configs[1] level 3, 300 systems): v0 3.24 ms, v1 3.78, v2 4.05, v3 3.62
            if (var == 1) return run_minres<64, 8, 1, V, true, true>(a, nb, tol, max_iter, out, slot, ctr, s);
            if (var == 2) return run_minres<64, 16, 1, V, false>(a, nb, tol, max_iter, out, slot, ctr, s);
            if (var == 3) return run_minres<64, 8, 1, V, false, true>(a, nb, tol, max_iter, out, slot, ctr, s);
            return run_minres<64, 16, 1, V, true, true>(a, nb, tol, max_iter, out, slot, ctr, s);
#endif
        default: return cudaErrorNotSupported;
    }
}

cudaError_t launch_minres(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                          unsigned* ctr, bool verify, const int* order, cudaStream_t s, int xmode, double* xio) {
    if (minres_tile_variant(N) >= 0)
        return launch_minres_tile(N, a, nb, tol, max_iter, out, slot, ctr, verify, order, s, xmode, xio);
    if (xmode) return cudaErrorNotSupported;
    // the column-strip kernel takes the systems in index order
    return verify ? minres_dispatch<true>(N, a, nb, tol, max_iter, out, slot, ctr, s)
                  : minres_dispatch<false>(N, a, nb, tol, max_iter, out, slot, ctr, s);
}

}  // namespace mlmc
