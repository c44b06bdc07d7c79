// k_minres_tile.cu -- K3 v2: batched MINRES with 2-column register tiles (h = 1/8 .. 1/64).
//
// Same method as k_minres.cu (Eq. (2), R9, R10, R26): unpreconditioned
// binary64 MINRES from x0 = 0 on the P1 stiffness matrix of the uniform SW-NE
// triangulation (= the 5-point operator with edge conductances, R10), stopped
// when the Paige-Saunders recurrence residual phibar_k / ||b|| <= tol; the QoI
// Q = h^2 1^T x_k is carried as a per-thread scalar (R26), x itself only in the
// VERIFY instantiation (true residual reported, identical Q).
//
// What changes against the column-strip kernel (profiles/r01_ncu_minres.md):
//  * a thread owns a 2-column x R-row tile: its west/east neighbours inside the
//    tile are registers, so the shared-memory exchange is one STS per node and
//    one LDS per node (was one STS + two LDS), in a plane layout
//    [row][column parity][pair] that keeps every warp access conflict-free;
//  * the diagonal d = cE + cW + cN + cS is formed once per solve (registers or,
//    for h = 1/64, a shared grid) and the conductances are kept negated, so the
//    stencil is one DMUL + four DFMA;
//  * the Lanczos vector is kept unnormalised (p_k = beta_k v_k): alpha =
//    (1/beta_k) sum p_k . y and the w update folds 1/gamma into its three
//    coefficients -- 14 fp64 operations per node and iteration (was ~20);
//  * the iteration loop is unrolled by two so the (p_k, p_{k-1}) and
//    (w_{k-1}, w_{k-2}) register pairs swap roles instead of being copied.
// Tile-local phantom nodes (column N when the last pair overhangs, row N when the
// last strip does) keep exactly zero entries: their conductances are zero and
// their y is scaled by a per-thread 0 instead of 1/beta.
#include <cuda_runtime.h>
#include <cfloat>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "internal.h"

namespace mlmc {
namespace {

// Conductance placement (template CM, bit flags): 1 = diagonal d from a shared grid,
// 2 = west conductance of column 0 from a shared grid; everything else in registers.
template <int N, int R, int MINB_, int CM_>
struct TileCfg {
    static constexpr int CM = CM_;
    static constexpr bool DS = CM & 1, WS = CM & 2;
    static constexpr int C = N - 1;                       // interior columns / rows
    static constexpr int PAIRS = N / 2;                   // pair p: columns 2p+1, 2p+2 (column N is a phantom)
    static constexpr int S = (C + R - 1) / R;             // row strips
    static constexpr int TPS = PAIRS * S;                 // threads per system
    static_assert(TPS % 32 == 0 || TPS == 16, "a system fills whole warps or one half-warp");
    static_assert(S * R == C || S * R == C + 1, "strips end at row C or at the boundary row N");
    static constexpr int NW = TPS >= 32 ? TPS / 32 : 1;
    static constexpr int GROUPS = TPS >= 128 ? 1 : 128 / TPS;
    static constexpr int BLOCK = TPS * GROUPS;
    static constexpr int MINB = MINB_;
    static constexpr int PW = PAIRS + 2;                  // plane pitch: halo pair on both sides
    static constexpr int RP = 2 * PW;                     // grid row pitch (two parity planes)
    static constexpr int ROWS = S * R + 2;                // grid rows 0 .. S*R+1 (0 and S*R+1 stay zero)
    static constexpr int GRID = ROWS * RP;
    static constexpr int DGRID = DS ? S * R * 2 * PAIRS : 0;   // d at [(row-1) * 2 * PAIRS + parity * PAIRS + pair]
    static constexpr int WGRID = WS ? S * R * PAIRS : 0;       // -cW of column 0 at [(row-1) * PAIRS + pair]
    static constexpr int RED = 4 * NW;                         // two reduction buffers of NW (value, value) pairs
    static constexpr int SMEM_PER_GROUP = GRID + DGRID + WGRID + RED;
    static constexpr size_t SMEM = sizeof(double) * SMEM_PER_GROUP * GROUPS + 16 * GROUPS;
};

// Butterfly over the lanes of one system inside a warp (all 32, or one half-warp when TPS = 16:
// two systems share a warp and may diverge, so the half-warp mask is used).
template <int TPS>
__device__ __forceinline__ unsigned lane_mask() {
    if constexpr (TPS >= 32) return 0xffffffffu;
    else return 0xffffu << (threadIdx.x & 16);
}
template <int TPS>
__device__ __forceinline__ double warp_sum_all(double v) {
    constexpr int W = TPS >= 32 ? 32 : TPS;
    const unsigned m = lane_mask<TPS>();
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(m, v, o);
    return v;
}

template <int TPS, int GROUPS>
__device__ __forceinline__ void tsync(int g) {
    if constexpr (TPS <= 32) {
        __syncwarp(lane_mask<TPS>());
    } else if constexpr (GROUPS == 1) {
        __syncthreads();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(TPS) : "memory");
    }
}

// Fixed-order sum of the NW warp partials held in buf[2w + c] (every thread reads all of them,
// so every thread ends with the same bits).
template <int NW>
__device__ __forceinline__ double2 sum_partials(const double* buf) {
    double2 v[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) v[w] = reinterpret_cast<const double2*>(buf)[w];
#pragma unroll
    for (int st = 1; st < NW; st *= 2) {
#pragma unroll
        for (int w = 0; w + st < NW; w += 2 * st) {
            v[w].x += v[w + st].x;
            v[w].y += v[w + st].y;
        }
    }
    return v[0];
}

template <int TPS, int GROUPS>
__device__ __forceinline__ double tsum1(double a, double* buf, int tg, int g) {
    a = warp_sum_all<TPS>(a);
    if constexpr (TPS <= 32) {
        return a;
    } else {
        if ((tg & 31) == 0) reinterpret_cast<double2*>(buf)[tg >> 5] = make_double2(a, 0.0);
        tsync<TPS, GROUPS>(g);
        return sum_partials<TPS / 32>(buf).x;
    }
}

// Iteration k of MINRES, written so that the Givens chain is off the critical path:
//  A(k)   y = A p_k / beta_k - (beta_k / beta_{k-1}) p_{k-1}          (p_k = beta_k v_k, unnormalised)
//  alpha_k = v_k . y                                                   [reduction]
//  B(k)   p_{k+1} = y - alpha_k v_k
//  C(k)   wt_k = v_k - (eps_k / gamma_{k-2}) wt_{k-2} - (delta_k / gamma_{k-1}) wt_{k-1}
//         (wt_k = gamma_k w_k: delta_k and eps_k are known once alpha_k is, gamma_k is not)
//  beta_{k+1} = ||p_{k+1}||                                            [reduction]
//  Givens: gamma_k, phi_k; 1^T x_k = 1^T x_{k-1} + (phi_k / gamma_k) 1^T wt_k
// (A one-reduction variant, beta_{k+1}^2 = ||y||^2 - alpha_k^2, was tried and rejected: without
// re-normalisation the error of ||v_k|| = 1 grows by ~alpha^2/beta^2 per step and the solve diverges.)
template <int N, int R, int MINB, int CM, bool VERIFY>
__global__ void __launch_bounds__(TileCfg<N, R, MINB, CM>::BLOCK, MINB)
minres_tile_kernel(const double* __restrict__ a_all, int nb, double tol, int max_iter, double* __restrict__ out,
                   int slot, unsigned* __restrict__ job_counter) {
    using K = TileCfg<N, R, MINB, CM>;
    constexpr int PAIRS = K::PAIRS, PW = K::PW, RP = K::RP, TPS = K::TPS, GROUPS = K::GROUPS;
    constexpr bool DS = K::DS, WS = K::WS;
    constexpr int P = 2 * N * N;
    extern __shared__ double smem[];
    const int g = threadIdx.x / TPS, tg = threadIdx.x % TPS;
    double* Sg = smem + g * K::SMEM_PER_GROUP;           // exchange grid [row * RP + parity * PW + pair + 1]
    double* Dg = Sg + K::GRID;
    double* Wg = Dg + K::DGRID;
    double* redA = Wg + K::WGRID;
    double* redB = redA + 2 * K::NW;
    int* jobslot = reinterpret_cast<int*>(smem + K::SMEM_PER_GROUP * GROUPS) + 4 * g;

    const int p = tg % PAIRS, s = tg / PAIRS;
    const int i0 = 2 * p + 1, i1 = i0 + 1, j0 = s * R + 1;   // tile: columns i0, i1; rows j0 .. j0+R-1
    const bool col1_live = i1 <= K::C;
    const bool top_live = j0 + R - 1 <= K::C;
    const double h = 1.0 / N, h2 = h * h;
    // own column c of row j at Sg[j*RP + c*PW + p + 1];
    // west of column i0 = parity-1 plane, pair p-1; east of column i1 = parity-0 plane, pair p+1
    double* const own = Sg + j0 * RP + p + 1;
    const double* const westp = Sg + j0 * RP + PW + p;
    const double* const eastp = Sg + j0 * RP + p + 2;
    double* const dgp = Dg + (j0 - 1) * 2 * PAIRS + p;
    double* const wgp = Wg + (j0 - 1) * PAIRS + p;

    for (int e = tg; e < K::GRID; e += TPS) Sg[e] = 0.0;   // halo rows / pairs are never written again

    for (;;) {
        if (tg == 0) *jobslot = (int)atomicAdd(job_counter, 1u);
        tsync<TPS, GROUPS>(g);
        const int job = *jobslot;
        tsync<TPS, GROUPS>(g);
        if (job >= nb) break;
        const double* a = a_all + (size_t)job * P;
        auto aL = [&](int ii, int jj) { return __ldg(a + 2 * (jj * N + ii)); };
        auto aU = [&](int ii, int jj) { return __ldg(a + 2 * (jj * N + ii) + 1); };
        // cE(i,j): edge (i,j)-(i+1,j), lower triangle of cell (i,j) + upper of cell (i,j-1)
        // cN(i,j): edge (i,j)-(i,j+1), upper triangle of cell (i,j) + lower of cell (i-1,j)
        auto cEf = [&](int ii, int jj) { return 0.5 * (aL(ii, jj) + aU(ii, jj - 1)); };
        auto cNf = [&](int ii, int jj) { return 0.5 * (aU(ii, jj) + aL(ii - 1, jj)); };

        // ---- conductances (negated) and diagonal of the tile; phantom nodes get zeros.  Column 1's
        // west conductance is column 0's east one (same edge).
        double nE0[R], nE1[R], nN0[R], nN1[R], nW0[WS ? 1 : R], dg0[DS ? 1 : R], dg1[DS ? 1 : R];
        double nS0 = 0.0, nS1 = 0.0;                    // south conductances of the tile's first row
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int j = j0 + r;
            const bool rl = j <= K::C;
            const double e0 = rl ? cEf(i0, j) : 0.0;
            const double w0 = rl ? cEf(i0 - 1, j) : 0.0;
            const double n0 = rl ? cNf(i0, j) : 0.0;
            const double s0 = rl ? cNf(i0, j - 1) : 0.0;
            const bool l1 = rl && col1_live;
            const double e1 = l1 ? cEf(i1, j) : 0.0;
            const double n1 = l1 ? cNf(i1, j) : 0.0;
            const double s1 = l1 ? cNf(i1, j - 1) : 0.0;
            const double d0 = (e0 + w0) + (n0 + s0);
            const double d1 = l1 ? (e1 + e0) + (n1 + s1) : 0.0;
            nE0[r] = -e0; nE1[r] = -e1; nN0[r] = -n0; nN1[r] = -n1;
            if (r == 0) { nS0 = -s0; nS1 = -s1; }
            if constexpr (WS) wgp[r * PAIRS] = -w0; else nW0[WS ? 0 : r] = -w0;
            if constexpr (DS) {
                dgp[r * 2 * PAIRS] = d0;
                dgp[r * 2 * PAIRS + PAIRS] = d1;
            } else {
                dg0[DS ? 0 : r] = d0;
                dg1[DS ? 0 : r] = d1;
            }
        }

        // ---- MINRES state: X = p_k, Y = p_{k-1} (then y), Wn = wt_{k-1}, Wo = wt_{k-2}
        double X0[R], X1[R], Y0[R], Y1[R], Wn0[R], Wn1[R], Wo0[R], Wo1[R];
        double x0[VERIFY ? R : 1], x1[VERIFY ? R : 1];
        double pb = 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const bool rl = (r < R - 1) || top_live;
            const double b0 = rl ? h2 : 0.0;
            const double b1 = rl && col1_live ? h2 : 0.0;
            X0[r] = b0; X1[r] = b1; Y0[r] = 0.0; Y1[r] = 0.0;
            Wn0[r] = 0.0; Wn1[r] = 0.0; Wo0[r] = 0.0; Wo1[r] = 0.0;
            if constexpr (VERIFY) { x0[VERIFY ? r : 0] = 0.0; x1[VERIFY ? r : 0] = 0.0; }
            own[r * RP] = b0;
            own[r * RP + PW] = b1;
            pb = fma(b0, b0, fma(b1, b1, pb));
        }
        pb = tsum1<TPS, GROUPS>(pb, redB, tg, g);          // barrier: the grid holds p_1 = b
        double invb = pb > 0.0 ? rsqrt(pb) : 0.0;          // 1 / beta_k
        const double beta1 = pb > 0.0 ? pb * invb : 0.0;
        const double inv_beta1 = invb, tol_b = tol * beta1;
        const double m1 = col1_live ? 1.0 : 0.0, mt = top_live ? 1.0 : 0.0;
        double dbar = 0.0, epsln = 0.0, phibar = beta1, cs = -1.0, sn = 0.0, ig1 = 0.0, ig2 = 0.0;
        double Xt = 0.0;                                    // this thread's share of 1^T x_k

        // A: Y <- (A X) / beta_k + ncr * Y; partial of X . y
        auto phaseA = [&](double (&XA)[R], double (&XB)[R], double (&YA)[R], double (&YB)[R], double ib, double ncr,
                          double& pa) {
            const double ib1 = ib * m1, ibt = ib * mt, ibt1 = ibt * m1;
            double pa0 = 0.0, pa1 = 0.0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double vW = westp[r * RP], vE = eastp[r * RP];
                const double vN0 = (r + 1 < R) ? XA[r + 1 < R ? r + 1 : r] : own[R * RP];
                const double vN1 = (r + 1 < R) ? XB[r + 1 < R ? r + 1 : r] : own[R * RP + PW];
                const double vS0 = (r > 0) ? XA[r > 0 ? r - 1 : 0] : own[-RP];
                const double vS1 = (r > 0) ? XB[r > 0 ? r - 1 : 0] : own[-RP + PW];
                const double sS0 = (r > 0) ? nN0[r > 0 ? r - 1 : 0] : nS0;
                const double sS1 = (r > 0) ? nN1[r > 0 ? r - 1 : 0] : nS1;
                const double d0 = DS ? dgp[r * 2 * PAIRS] : dg0[DS ? 0 : r];
                const double d1 = DS ? dgp[r * 2 * PAIRS + PAIRS] : dg1[DS ? 0 : r];
                const double w0 = WS ? wgp[r * PAIRS] : nW0[WS ? 0 : r];
                double t0 = d0 * XA[r];
                double t1 = d1 * XB[r];
                t0 = fma(nE0[r], XB[r], t0);
                t1 = fma(nE0[r], XA[r], t1);
                t0 = fma(w0, vW, t0);
                t1 = fma(nE1[r], vE, t1);
                t0 = fma(nN0[r], vN0, t0);
                t1 = fma(nN1[r], vN1, t1);
                t0 = fma(sS0, vS0, t0);
                t1 = fma(sS1, vS1, t1);
                const double s0 = (r == R - 1) ? ibt : ib;
                const double s1 = (r == R - 1) ? ibt1 : ib1;
                const double y0 = fma(t0, s0, ncr * YA[r]);
                const double y1 = fma(t1, s1, ncr * YB[r]);
                YA[r] = y0;
                YB[r] = y1;
                pa0 = fma(XA[r], y0, pa0);
                pa1 = fma(XB[r], y1, pa1);
            }
            pa = pa0 + pa1;
        };

        int k = 1, status = 1;
        double pa = 0.0;
        if (beta1 == 0.0) {
            status = 0;
            k = 0;
        } else {
            phaseA(X0, X1, Y0, Y1, invb, 0.0, pa);
        }
        auto iterate = [&](double (&XA)[R], double (&XB)[R], double (&YA)[R], double (&YB)[R], double (&WnA)[R],
                           double (&WnB)[R], double (&WoA)[R], double (&WoB)[R]) -> bool {
            const double alpha = invb * tsum1<TPS, GROUPS>(pa, redA, tg, g);   // all grid reads of A(k) done
            const double nca = -alpha * invb;
            const double delta = cs * dbar + sn * alpha;
            const double gbar = sn * dbar - cs * alpha;
            const double c1 = invb, c2 = -epsln * ig2, c3 = -delta * ig1;
            double pb0 = 0.0, pb1 = 0.0, sw0 = 0.0, sw1 = 0.0;
#pragma unroll
            for (int r = 0; r < R; ++r) {                  // B(k) into Y, C(k) into Wo
                const double y0 = fma(nca, XA[r], YA[r]);
                const double y1 = fma(nca, XB[r], YB[r]);
                YA[r] = y0;
                YB[r] = y1;
                own[r * RP] = y0;
                own[r * RP + PW] = y1;
                pb0 = fma(y0, y0, pb0);
                pb1 = fma(y1, y1, pb1);
                const double w0 = fma(c1, XA[r], fma(c2, WoA[r], c3 * WnA[r]));
                const double w1 = fma(c1, XB[r], fma(c2, WoB[r], c3 * WnB[r]));
                WoA[r] = w0;
                WoB[r] = w1;
                sw0 += w0;
                sw1 += w1;
            }
            const double b2 = tsum1<TPS, GROUPS>(pb0 + pb1, redB, tg, g);   // grid holds p_{k+1}
            const double invb_new = b2 > 0.0 ? rsqrt(b2) : 0.0;
            const double beta = b2 * invb_new;              // beta_{k+1}
            // ---- Givens rotation (Paige-Saunders); gamma_k = hypot(gbar, beta_{k+1})
            epsln = sn * beta;
            dbar = -cs * beta;
            const double gg = fma(gbar, gbar, b2);
            const double invg = gg > 0.0 ? rsqrt(gg) : 1.0 / DBL_MIN;
            cs = gbar * invg;
            sn = beta * invg;
            const double phi = cs * phibar;
            phibar = sn * phibar;
            const double phig = phi * invg;                 // x_k = x_{k-1} + (phi_k / gamma_k) wt_k
            Xt = fma(phig, sw0 + sw1, Xt);
            ig2 = ig1;
            ig1 = invg;
            if constexpr (VERIFY) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    x0[VERIFY ? r : 0] = fma(phig, WoA[r], x0[VERIFY ? r : 0]);
                    x1[VERIFY ? r : 0] = fma(phig, WoB[r], x1[VERIFY ? r : 0]);
                }
            }
            if (!(phibar == phibar) || !(beta == beta)) status = 3;
            else if (phibar <= tol_b) status = 0;           // phibar / ||b|| <= tol
            if (status != 1 || k >= max_iter) return false; // uniform across the system
            // A(k+1): X <- A p_{k+1} / beta_{k+1} - (beta_{k+1} / beta_k) p_k
            phaseA(YA, YB, XA, XB, invb_new, -beta * invb, pa);
            invb = invb_new;
            ++k;
            return true;
        };
        if (status == 1) {
            for (;;) {
                if (!iterate(X0, X1, Y0, Y1, Wn0, Wn1, Wo0, Wo1)) break;
                if (!iterate(Y0, Y1, X0, X1, Wo0, Wo1, Wn0, Wn1)) break;
            }
        }
        double relres = phibar * inv_beta1;
        const double Xs = tsum1<TPS, GROUPS>(Xt, redA, tg, g);
        if constexpr (VERIFY) {
            // true residual ||b - A x|| / ||b|| (the loop's last grid reads precede the barrier above)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                own[r * RP] = x0[VERIFY ? r : 0];
                own[r * RP + PW] = x1[VERIFY ? r : 0];
            }
            tsync<TPS, GROUPS>(g);
            double rr = 0.0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const bool rl = (r < R - 1) || top_live;
                const double v0 = own[r * RP], v1 = own[r * RP + PW];
                const double sS0 = (r > 0) ? nN0[r > 0 ? r - 1 : 0] : nS0;
                const double sS1 = (r > 0) ? nN1[r > 0 ? r - 1 : 0] : nS1;
                const double d0 = DS ? dgp[r * 2 * PAIRS] : dg0[DS ? 0 : r];
                const double d1 = DS ? dgp[r * 2 * PAIRS + PAIRS] : dg1[DS ? 0 : r];
                const double w0 = WS ? wgp[r * PAIRS] : nW0[WS ? 0 : r];
                double t0 = d0 * v0;
                t0 = fma(nE0[r], v1, t0);
                t0 = fma(w0, westp[r * RP], t0);
                t0 = fma(nN0[r], own[r * RP + RP], t0);
                t0 = fma(sS0, own[r * RP - RP], t0);
                double t1 = d1 * v1;
                t1 = fma(nE1[r], eastp[r * RP], t1);
                t1 = fma(nE0[r], v0, t1);
                t1 = fma(nN1[r], own[r * RP + RP + PW], t1);
                t1 = fma(sS1, own[r * RP - RP + PW], t1);
                const double res0 = rl ? h2 - t0 : 0.0;
                const double res1 = rl && col1_live ? h2 - t1 : 0.0;
                rr = fma(res0, res0, fma(res1, res1, rr));
            }
            rr = tsum1<TPS, GROUPS>(rr, redB, tg, g);
            relres = sqrt(rr) * inv_beta1;
        }
        if (tg == 0) {
            double* o = out + (size_t)job * kRecLen;
            o[0 + slot] = h2 * Xs;
            o[2 + slot] = (double)k;
            o[4 + slot] = relres;
            o[6 + slot] = (double)status;
        }
        tsync<TPS, GROUPS>(g);      // grid reuse by the next job
    }
}

template <int N, int R, int MINB, int CM, bool VERIFY>
cudaError_t run_tile(const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot, unsigned* ctr,
                     cudaStream_t s) {
    using K = TileCfg<N, R, MINB, CM>;
    auto kern = minres_tile_kernel<N, R, MINB, CM, VERIFY>;
    static int blocks_per_sm = -1, sms = 0;
    if (blocks_per_sm < 0) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, K::BLOCK, K::SMEM);
        if (e != cudaSuccess) return e;
        int dev;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (blocks_per_sm < 1) return cudaErrorInvalidConfiguration;
    }
    const uint64_t need = (nb + K::GROUPS - 1) / K::GROUPS;
    const uint64_t grid = std::min<uint64_t>(need, (uint64_t)blocks_per_sm * sms);
    if (grid == 0) return cudaSuccess;
    kern<<<(unsigned)grid, K::BLOCK, K::SMEM, s>>>(a, (int)nb, tol, max_iter, out, slot, ctr);
    return cudaGetLastError();
}

}  // namespace

// Tile shape per mesh: MLMC_MINRES_TILE_N<N>=<index> selects an alternative for tuning runs;
// -1 hands the mesh back to the column-strip kernel (k_minres.cu).
int minres_tile_variant(int N) {
    static int v[4] = {-2, -2, -2, -2};
    const int slot = N == 8 ? 3 : N == 16 ? 0 : N == 32 ? 1 : N == 64 ? 2 : -1;
    if (slot < 0) return -1;
    if (v[slot] == -2) {
        char name[64];
        std::snprintf(name, sizeof(name), "MLMC_MINRES_TILE_N%d", N);
        const char* e = std::getenv(name);
        v[slot] = e ? std::atoi(e) : 0;
    }
    return v[slot];
}

// Variant table (index = MLMC_MINRES_TILE_N<N>): <N, R, MINB, CM>; measured with tools/tune_minres.py.
template <bool V>
static cudaError_t tile_dispatch(int N, int var, const double* a, uint64_t nb, double tol, int max_iter, double* out,
                                 int slot, unsigned* ctr, cudaStream_t s) {
    switch (N) {
        case 8:   // two systems per warp (16 threads each)
            if (var == 1) return run_tile<8, 2, 5, 0, V>(a, nb, tol, max_iter, out, slot, ctr, s);
            return run_tile<8, 2, 4, 0, V>(a, nb, tol, max_iter, out, slot, ctr, s);
        case 16:
            // measured (configs[1] level 1, 5000 systems): v0 0.28 ms, v1 0.31; strip 0.31
            if (var == 1) return run_tile<16, 2, 4, 0, V>(a, nb, tol, max_iter, out, slot, ctr, s);
            return run_tile<16, 4, 3, 0, V>(a, nb, tol, max_iter, out, slot, ctr, s);
        case 32:
            // measured (configs[1] level 2, 1200 systems): v0 0.66 ms, v1 0.69, v2 0.75, v3 0.74; strip 1.02
            if (var == 1) return run_tile<32, 4, 4, 3, V>(a, nb, tol, max_iter, out, slot, ctr, s);
            if (var == 2) return run_tile<32, 8, 2, 3, V>(a, nb, tol, max_iter, out, slot, ctr, s);
            if (var == 3) return run_tile<32, 4, 4, 1, V>(a, nb, tol, max_iter, out, slot, ctr, s);
            return run_tile<32, 4, 3, 0, V>(a, nb, tol, max_iter, out, slot, ctr, s);
        case 64:
            // measured (configs[1] level 3, 300 systems): v0 2.31 ms, v1 2.40, v2 3.03; strip kernel 3.25
            if (var == 1) return run_tile<64, 8, 1, 1, V>(a, nb, tol, max_iter, out, slot, ctr, s);
            if (var == 2) return run_tile<64, 4, 1, 3, V>(a, nb, tol, max_iter, out, slot, ctr, s);
            return run_tile<64, 8, 1, 3, V>(a, nb, tol, max_iter, out, slot, ctr, s);
        default: return cudaErrorNotSupported;
    }
}

cudaError_t launch_minres_tile(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                               unsigned* ctr, bool verify, cudaStream_t s) {
    const int var = minres_tile_variant(N);
    return verify ? tile_dispatch<true>(N, var, a, nb, tol, max_iter, out, slot, ctr, s)
                  : tile_dispatch<false>(N, var, a, nb, tol, max_iter, out, slot, ctr, s);
}

}  // namespace mlmc
