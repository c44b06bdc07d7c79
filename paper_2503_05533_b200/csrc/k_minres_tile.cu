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
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cfloat>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "internal.h"

namespace mlmc {
namespace {
namespace cg = cooperative_groups;

#ifdef MLMC_TUNING
// job trace of the tuning build (tools/step_trace.py): per system solve {start, end (%globaltimer ns), smid << 32 | N,
// (cluster rank * 2 + record slot: 0 fine, 1 coarse) << 32 | job}
__device__ unsigned long long* g_trace = nullptr;
__device__ unsigned int g_trace_cap = 0;
__device__ unsigned int g_trace_n = 0;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// Conductance placement (template CM, bit flags): 1 = diagonal d from a shared grid,
// 2 = west conductance of column 0 from a shared grid; everything else in registers.
template <int N, int R, int MINB_, int CM_, int CL_ = 1>
struct TileCfg {
    static constexpr int CM = CM_;
    static constexpr bool DS = CM & 1, WS = CM & 2, CS = CM & 4;
    static_assert(!(CS && (DS || WS)), "CS keeps every conductance in shared memory");
    static constexpr int C = N - 1;                       // interior columns / rows
    static constexpr int PAIRS = N / 2;                   // pair p: columns 2p+1, 2p+2 (column N is a phantom)
    static constexpr int S = (C + R - 1) / R;             // row strips of the system
    // CL > 1 (K3b): one system per cluster of CL CTAs, CTA rank c owning strips c SL .. c SL + SL - 1
    static constexpr int CL = CL_;
    static_assert(CL == 1 || (S % CL == 0 && CM == 0), "whole strips per CTA; conductances in registers");
    static constexpr int SL = S / CL;                     // strips per CTA
    static constexpr int TPS = PAIRS * SL;                // threads per system (per CTA when CL > 1)
    static_assert(TPS % 32 == 0 || TPS == 16 || TPS == 8, "a system fills whole warps or a half / quarter warp");
    static_assert(S * R == C || S * R == C + 1, "strips end at row C or at the boundary row N");
    static constexpr int NW = TPS >= 32 ? TPS / 32 : 1;
    static constexpr int GROUPS = TPS >= 128 ? 1 : 128 / TPS;
    static_assert(CL == 1 || GROUPS == 1, "a clustered system fills its CTA");
    static constexpr int BLOCK = TPS * GROUPS;
    static constexpr int MINB = MINB_;
    static constexpr int PW = PAIRS + 2;                  // plane pitch: halo pair on both sides
    static constexpr int RP = 2 * PW;                     // grid row pitch (two parity planes)
    static constexpr int ROWS = SL * R + 2;               // grid rows 0 .. SL*R+1 (halo rows: zero, or the
                                                          // neighbouring CTAs' boundary rows when CL > 1)
    static constexpr int GRID = ROWS * RP;
    static constexpr int DGRID = DS ? S * R * 2 * PAIRS : 0;   // d at [(row-1) * 2 * PAIRS + parity * PAIRS + pair]
    static constexpr int WGRID = WS ? S * R * PAIRS : 0;       // -cW of column 0 at [(row-1) * PAIRS + pair]
    // CS: cE(i, j) at [(j - 1) * 2 PE + (i & 1) * PE + (i >> 1)] for rows 1 .. S*R, cN(i, j) at
    // [j * 2 PE + (i & 1) * PE + (i >> 1)] for rows 0 .. S*R (phantom rows / columns hold zeros)
    static constexpr int PE = PAIRS + 1;
    static constexpr int CEG = CS ? S * R * 2 * PE : 0;
    static constexpr int CNG = CS ? (S * R + 1) * 2 * PE : 0;
    static constexpr int RED = 4 * NW;                         // reduction buffer: NW x (3 partials + pad)
    // CL > 1: every CTA's partials [2 parities][CL][4] (pushed to each CTA), the neighbours' boundary-row
    // t = A p_j [2 parities][2 sides][N] (side 0: the row below this CTA's first row, 1: the row above its
    // last), p_{j-1} of those halo rows [2][N], two mbarriers (one per parity)
    static constexpr int CLX = CL > 1 ? 8 * CL + 4 * N + 2 * N + 2 : 0;
    static constexpr int SMEM_PER_GROUP = GRID + DGRID + WGRID + CEG + CNG + RED + CLX;
    static constexpr size_t SMEM = sizeof(double) * SMEM_PER_GROUP * GROUPS + 16 * GROUPS;
};

// Butterfly over the lanes of one system inside a warp (all 32, or one half-warp when TPS = 16:
// two systems share a warp and may diverge, so the half-warp mask is used).
template <int TPS>
__device__ __forceinline__ unsigned lane_mask() {
    if constexpr (TPS >= 32) return 0xffffffffu;
    else if constexpr (TPS == 16) return 0xffffu << (threadIdx.x & 16);
    else return 0xffu << (threadIdx.x & 24);
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

// Sums of (a, b, c) over the system's threads, bit-identical in every thread.  Inside a warp (or the
// half-warp of a 16-thread system) a reduce-scatter: the first two butterfly levels exchange half of
// the (a, b, c, 0) quadruple each, so lane l ends with the total of quantity (l / (W/4)) & 3 after
// 12 shuffles and 6 adds instead of 30 and 15.  Across warps every thread adds the NW warp totals in
// the same fixed (pairwise) order.
template <int TPS, int GROUPS>
__device__ __forceinline__ double4 tsum3(double a, double b, double c, double* buf, int tg, int g) {
    constexpr int W = TPS >= 32 ? 32 : TPS;
    static_assert(W == 8 || W == 16 || W == 32, "reduce-scatter needs 8, 16 or 32 lanes");
    const unsigned msk = lane_mask<TPS>();
    const int lane = threadIdx.x & (W - 1);
    constexpr int O1 = W / 2, O2 = W / 4;
    // level 1: lanes with the O1 bit clear keep (a, b), the others (c, 0)
    const bool h1 = lane & O1;
    const double k1 = h1 ? c : a, k2 = h1 ? 0.0 : b;
    const double s1 = h1 ? a : c, s2 = h1 ? b : 0.0;
    const double r1 = k1 + __shfl_xor_sync(msk, s1, O1, W);
    const double r2 = k2 + __shfl_xor_sync(msk, s2, O1, W);
    // level 2: keep one of the two
    const bool h2 = lane & O2;
    double v = (h2 ? r2 : r1) + __shfl_xor_sync(msk, h2 ? r1 : r2, O2, W);
#pragma unroll
    for (int o = O2 / 2; o > 0; o >>= 1) v += __shfl_xor_sync(msk, v, o, W);
    // lane l now holds quantity q = (l / O2) & 3: 0 = a, 1 = b, 2 = c, 3 = the zero pad
    if constexpr (TPS <= 32) {
        return make_double4(__shfl_sync(msk, v, 0, W), __shfl_sync(msk, v, O2, W), __shfl_sync(msk, v, 2 * O2, W), 0.0);
    } else {
        // across the NW warps: lane L < 3 NW of every warp loads warp (L mod NW)'s total of quantity L / NW,
        // an xor butterfly over the NW lanes of each group adds them -- ((w0 + w1) + (w2 + w3)) + ..., the same
        // association in every lane (IEEE addition commutes) -- and three shuffles broadcast the totals: per
        // thread 1 load and log2(NW) adds instead of NW double4 loads and 3 (NW - 1) adds
        constexpr int NW = TPS / 32;
        static_assert(3 * NW <= 32 && (NW & (NW - 1)) == 0, "one warp holds the 3 x NW warp totals");
        if ((lane & (O2 - 1)) == 0 && lane < 3 * O2) buf[4 * (tg >> 5) + lane / O2] = v;
        tsync<TPS, GROUPS>(g);
        double u = lane < 3 * NW ? buf[4 * (lane % NW) + lane / NW] : 0.0;
#pragma unroll
        for (int o = 1; o < NW; o <<= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
        return make_double4(__shfl_sync(0xffffffffu, u, 0), __shfl_sync(0xffffffffu, u, NW),
                            __shfl_sync(0xffffffffu, u, 2 * NW), 0.0);
    }
}

// K3b cluster exchange: st.async stores into a peer CTA's shared memory that complete-tx on the peer's
// mbarrier (no cluster-wide barrier and no fence in the step loop); as with TMA multicast, the receiver's
// CTA-scope wait on its own mbarrier makes the tracked bytes visible (no L1 invalidation per step)
__device__ __forceinline__ uint32_t sm32(const void* ptr) { return (uint32_t)__cvta_generic_to_shared(ptr); }
__device__ __forceinline__ uint32_t mapa32(uint32_t a, int r) {
    uint32_t o;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
    return o;
}
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                 "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

// One MINRES step per stencil, one reduction per step (R27):
//   step j:  t = A p_j;  reduce (p_j . t, p_j . p_j, 1 . p_j)           [the only reduction]
//            beta_j = ||p_j||, alpha_j = p_j.t / p_j.p_j (= v_j^T A v_j), sigma_j = 1^T v_j
//            Givens rotation of MINRES iteration k = j-1 (needs alpha_{j-1}, beta_j), stopping test
//            Q += phi_k s_k with s_k = 1^T w_k from s_k = (sigma_k - eps_k s_{k-2} - delta_k s_{k-1}) / gamma_k
//            p_{j+1} = t / beta_j - (alpha_j / beta_j) p_j - (beta_j / beta_{j-1}) p_{j-1}
//            exchange p_{j+1} through shared memory                    [plain barrier]
// p_j = beta_j v_j keeps its true norm (beta from the stored vector, no drift); alpha is the
// Rayleigh quotient (Lanczos variant "A1") instead of v^T (A v - beta v_prev).  Three vectors per
// node (p_{j-1}, p_j, t) instead of five; 11 fp64 operations per node and step.  VERIFY also
// carries w_k and x_k (textbook updates) to report the true residual.
// XM (coarse-to-fine initial guess, NEXT-4, R32): 0 = x0 = 0; 1 = also write the final x_k of every
// system to xio[job][(N-1)^2] (needs VERIFY: x is carried); 2 = start from x0 = P x_c, the P1 interpolation
// of the coarse solution xio[job][(N/2-1)^2] of the same sample (the coarse half of the coupled sample): MINRES
// then runs on A e = r0 = b - A x0 with the SAME stopping rule ||b - A x_k|| <= tol ||b|| (phibar_k <= tol
// ||b||, not tol ||r0||), and Q = h^2 (1^T x0 + 1^T e_k).
template <int N, int R, int MINB, int CM, bool VERIFY, int XM = 0, int CL = 1>
__global__ void __launch_bounds__(TileCfg<N, R, MINB, CM, CL>::BLOCK, MINB)
minres_tile_kernel(const double* __restrict__ a_all, int nb, double tol, int max_iter, double* __restrict__ out,
                   int slot, unsigned* __restrict__ job_counter, const int* __restrict__ order,
                   double* __restrict__ xio) {
    static_assert(XM != 1 || VERIFY, "writing x needs the VERIFY instantiation (x carried)");
    static_assert(CL == 1 || (!VERIFY && XM == 0), "K3b: plain MINRES from x0 = 0");
    using K = TileCfg<N, R, MINB, CM, CL>;
    constexpr int PAIRS = K::PAIRS, PW = K::PW, RP = K::RP, TPS = K::TPS, GROUPS = K::GROUPS;
    constexpr bool DS = K::DS, WS = K::WS, CS = K::CS;
    constexpr int P = 2 * N * N, PE = K::PE;
    extern __shared__ double smem[];
    const int g = threadIdx.x / TPS, tg = threadIdx.x % TPS;
    double* Sg = smem + g * K::SMEM_PER_GROUP;           // exchange grid [row * RP + parity * PW + pair + 1]
    double* Dg = Sg + K::GRID;
    double* Wg = Dg + K::DGRID;
    double* CEg = Wg + K::WGRID;
    double* CNg = CEg + K::CEG;
    double* red = CNg + K::CNG;                           // NW x 4 doubles (3 partials + pad)
    double* part = red + K::RED;                          // CL > 1: [2][CL][4] CTA partials by step parity
    double* thb = part + 8 * CL;                          //         [2][2][N] neighbours' boundary t
    double* hst = thb + 4 * N;                            //         [2][N] p_{j-1} of the two halo rows
    uint64_t* mbar = reinterpret_cast<uint64_t*>(hst + 2 * N);   //     [2] arrivals of the step's pushes
    int* jobslot = reinterpret_cast<int*>(smem + K::SMEM_PER_GROUP * GROUPS) + 4 * g;
    const int rank = CL > 1 ? (int)cg::this_cluster().block_rank() : 0;

    const int p = tg % PAIRS, s = tg / PAIRS;
    const int jl0 = s * R + 1;                            // first row of the tile in this CTA's grid
    const int i0 = 2 * p + 1, i1 = i0 + 1, j0 = rank * K::SL * R + jl0;   // tile: columns i0, i1; rows j0 .. j0+R-1
    const bool col1_live = i1 <= K::C;
    const bool top_live = j0 + R - 1 <= K::C;
    const double h = 1.0 / N, h2 = h * h;
    double* const own = Sg + jl0 * RP + p + 1;
    const double* const westp = Sg + jl0 * RP + PW + p;
    const double* const eastp = Sg + jl0 * RP + p + 2;
    double* const dgp = Dg + (jl0 - 1) * 2 * PAIRS + p;
    double* const wgp = Wg + (jl0 - 1) * PAIRS + p;
    // CL > 1: the first strip keeps the halo row below the CTA (side 0), the last strip the one above (side 1)
    const bool halo_lo = CL > 1 && s == 0 && rank > 0;
    const bool halo_hi = CL > 1 && s == K::SL - 1 && rank < CL - 1;

    for (int e = tg; e < K::GRID; e += TPS) Sg[e] = 0.0;   // halo rows / pairs are never written again
    // K3b: bytes each step's wait expects (every CTA's 3 partials, N t values from each neighbour); the step
    // count gk runs on across jobs (identical in every CTA of the cluster) and picks buffer and phase
    const uint32_t tx_bytes = CL > 1 ? (uint32_t)(24 * CL + (rank > 0 ? 8 * N : 0) + (rank < CL - 1 ? 8 * N : 0)) : 0u;
    uint32_t gk = 0;
    if constexpr (CL > 1) {
        if (tg == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm32(mbar)) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm32(mbar + 1)) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        cg::this_cluster().sync();                       // no push before every peer's barriers exist
    }

    for (;;) {
        int job;
        if constexpr (CL > 1) {          // rank 0 draws the job; the cluster barrier also ends the last job
            auto cl = cg::this_cluster();
            if (rank == 0 && tg == 0) jobslot[0] = (int)atomicAdd(job_counter, 1u);
            cl.sync();
            if (tg == 0) jobslot[1] = *cl.map_shared_rank(jobslot, 0);
            __syncthreads();
            job = jobslot[1];
        } else {
            if (tg == 0) *jobslot = (int)atomicAdd(job_counter, 1u);
            tsync<TPS, GROUPS>(g);
            job = *jobslot;
            tsync<TPS, GROUPS>(g);
        }
        if (job >= nb) break;
#ifdef MLMC_TUNING
        const unsigned long long trace_t0 = (tg == 0 && g_trace) ? gtimer() : 0ull;
#endif
        const int sj = order ? __ldg(order + job) : job;     // longest-first order (order_kernel) if given
        const double* a = a_all + (size_t)sj * P;
        auto aL = [&](int ii, int jj) { return __ldg(a + 2 * (jj * N + ii)); };
        auto aU = [&](int ii, int jj) { return __ldg(a + 2 * (jj * N + ii) + 1); };
        // cE(i,j): edge (i,j)-(i+1,j), lower triangle of cell (i,j) + upper of cell (i,j-1)
        // cN(i,j): edge (i,j)-(i,j+1), upper triangle of cell (i,j) + lower of cell (i-1,j)
        auto cEf = [&](int ii, int jj) { return 0.5 * (aL(ii, jj) + aU(ii, jj - 1)); };
        auto cNf = [&](int ii, int jj) { return 0.5 * (aU(ii, jj) + aL(ii - 1, jj)); };

        // ---- conductances (negated) and diagonal of the tile; phantom nodes get zeros.  Column 1's
        // west conductance is column 0's east one (same edge).
        constexpr int RR = CS ? 1 : R;
        double nE0[RR], nE1[RR], nN0[RR], nN1[RR], nW0[WS || CS ? 1 : R], dg0[DS || CS ? 1 : R], dg1[DS || CS ? 1 : R];
        double nS0 = 0.0, nS1 = 0.0;                    // south conductances of the tile's first row
        if constexpr (DS || CS) dg0[0] = dg1[0] = 0.0;   // placeholders of the shared-memory paths
        if constexpr (WS || CS) nW0[0] = 0.0;
        if constexpr (CS) {
            nE0[0] = nE1[0] = nN0[0] = nN1[0] = 0.0;
            for (int e = tg; e < K::CEG; e += TPS) {
                const int j = e / (2 * PE) + 1, i = 2 * (e % PE) + (e / PE) % 2;
                CEg[e] = (j <= K::C && i <= K::C) ? cEf(i, j) : 0.0;
            }
            for (int e = tg; e < K::CNG; e += TPS) {
                const int j = e / (2 * PE), i = 2 * (e % PE) + (e / PE) % 2;
                CNg[e] = (j <= K::C && i >= 1 && i <= K::C) ? cNf(i, j) : 0.0;
            }
        }
#pragma unroll
        for (int r = 0; r < (CS ? 0 : R); ++r) {
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
        // y = A v (v = this thread's tile of the grid-exchanged vector held in VA/VB)
        auto stencil = [&](const double (&VA)[R], const double (&VB)[R], int r, const double* grid_w,
                           const double* grid_e, const double* grid_own, double& t0, double& t1) {
            const double vW = grid_w[r * RP], vE = grid_e[r * RP];
            const double vN0 = (r + 1 < R) ? VA[r + 1 < R ? r + 1 : r] : grid_own[R * RP];
            const double vN1 = (r + 1 < R) ? VB[r + 1 < R ? r + 1 : r] : grid_own[R * RP + PW];
            const double vS0 = (r > 0) ? VA[r > 0 ? r - 1 : 0] : grid_own[-RP];
            const double vS1 = (r > 0) ? VB[r > 0 ? r - 1 : 0] : grid_own[-RP + PW];
            const double sS0 = (r > 0) ? nN0[r > 0 ? r - 1 : 0] : nS0;
            const double sS1 = (r > 0) ? nN1[r > 0 ? r - 1 : 0] : nS1;
            const double d0 = DS ? dgp[r * 2 * PAIRS] : dg0[DS ? 0 : r];
            const double d1 = DS ? dgp[r * 2 * PAIRS + PAIRS] : dg1[DS ? 0 : r];
            const double w0 = WS ? wgp[r * PAIRS] : nW0[WS ? 0 : r];
            t0 = d0 * VA[r];
            t1 = d1 * VB[r];
            t0 = fma(nE0[r], VB[r], t0);
            t1 = fma(nE0[r], VA[r], t1);
            t0 = fma(w0, vW, t0);
            t1 = fma(nE1[r], vE, t1);
            t0 = fma(nN0[r], vN0, t0);
            t1 = fma(nN1[r], vN1, t1);
            t0 = fma(sS0, vS0, t0);
            t1 = fma(sS1, vS1, t1);
        };

        // CS: the same stencil (same operations, same order) with the conductances from shared memory;
        // sc0 / sc1 carry the previous row's north conductances as this row's south ones
        auto stencil_cs = [&](const double (&VA)[R], const double (&VB)[R], int r, double& t0, double& t1,
                              double& sc0, double& sc1) {
            const int j = j0 + r;
            const double* ce = CEg + (j - 1) * 2 * PE;
            const double* cn = CNg + j * 2 * PE;
            const double w0 = ce[p], e0 = ce[PE + p], e1 = ce[p + 1];
            const double n0 = cn[PE + p], n1 = cn[p + 1];
            if (r == 0) { sc0 = cn[-2 * PE + PE + p]; sc1 = cn[-2 * PE + p + 1]; }
            const double s0 = sc0, s1 = sc1;
            const double vW = westp[r * RP], vE = eastp[r * RP];
            const double vN0 = (r + 1 < R) ? VA[r + 1 < R ? r + 1 : r] : own[R * RP];
            const double vN1 = (r + 1 < R) ? VB[r + 1 < R ? r + 1 : r] : own[R * RP + PW];
            const double vS0 = (r > 0) ? VA[r > 0 ? r - 1 : 0] : own[-RP];
            const double vS1 = (r > 0) ? VB[r > 0 ? r - 1 : 0] : own[-RP + PW];
            const double d0 = (e0 + w0) + (n0 + s0);
            const double d1 = (e1 + e0) + (n1 + s1);
            t0 = d0 * VA[r];
            t1 = d1 * VB[r];
            t0 = fma(-e0, VB[r], t0);
            t1 = fma(-e0, VA[r], t1);
            t0 = fma(-w0, vW, t0);
            t1 = fma(-e1, vE, t1);
            t0 = fma(-n0, vN0, t0);
            t1 = fma(-n1, vN1, t1);
            t0 = fma(-s0, vS0, t0);
            t1 = fma(-s1, vS1, t1);
            sc0 = n0;
            sc1 = n1;
        };

        // ---- state: X = p_{j-1}, Y = p_j, T = A p_j
        double X0[R], X1[R], Y0[R], Y1[R], T0[R], T1[R];
        double Wa0[VERIFY ? R : 1], Wa1[VERIFY ? R : 1], Wb0[VERIFY ? R : 1], Wb1[VERIFY ? R : 1];
        double x0[VERIFY ? R : 1], x1[VERIFY ? R : 1];
        double sum_x0 = 0.0;                                 // 1^T x0 (XM = 2)
        if constexpr (XM == 2) {
            // x0 = P x_c: the coarse P1 function at the fine nodes (coarse SW-NE triangles, R10): a fine node on
            // a coarse node takes its value, one on a horizontal / vertical / diagonal coarse edge the edge mean
            constexpr int CC = N / 2 - 1;
            const double* xc = xio + (size_t)sj * CC * CC;
            auto xcv = [&](int I, int J) -> double {
                return (I >= 1 && I <= CC && J >= 1 && J <= CC) ? __ldg(xc + (J - 1) * CC + (I - 1)) : 0.0;
            };
            auto x0f = [&](int i, int j) -> double {
                if (i > K::C || j > K::C) return 0.0;          // phantom nodes
                const int I = i >> 1, J = j >> 1;
                if (!(i & 1) && !(j & 1)) return xcv(I, J);
                if ((i & 1) && !(j & 1)) return 0.5 * (xcv(I, J) + xcv(I + 1, J));
                if (!(i & 1) && (j & 1)) return 0.5 * (xcv(I, J) + xcv(I, J + 1));
                return 0.5 * (xcv(I, J) + xcv(I + 1, J + 1));
            };
            double XA[R], XB[R];
            double s0 = 0.0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                XA[r] = x0f(i0, j0 + r);
                XB[r] = x0f(i1, j0 + r);
                s0 += XA[r] + XB[r];
                own[r * RP] = XA[r];
                own[r * RP + PW] = XB[r];
            }
            tsync<TPS, GROUPS>(g);                           // the grid holds x0
            double sc0 = 0.0, sc1 = 0.0;
#pragma unroll
            for (int r = 0; r < R; ++r) {                    // r0 = b - A x0 (phantom nodes stay 0)
                double t0, t1;
                if constexpr (CS) stencil_cs(XA, XB, r, t0, t1, sc0, sc1);
                else stencil(XA, XB, r, westp, eastp, own, t0, t1);
                const bool rl = (r < R - 1) || top_live;
                Y0[r] = rl ? h2 - t0 : 0.0;
                Y1[r] = rl && col1_live ? h2 - t1 : 0.0;
                X0[r] = 0.0; X1[r] = 0.0;
                if constexpr (VERIFY) {
                    Wa0[VERIFY ? r : 0] = Wa1[VERIFY ? r : 0] = Wb0[VERIFY ? r : 0] = Wb1[VERIFY ? r : 0] = 0.0;
                    x0[VERIFY ? r : 0] = XA[r];
                    x1[VERIFY ? r : 0] = XB[r];
                }
            }
            sum_x0 = tsum3<TPS, GROUPS>(s0, 0.0, 0.0, red, tg, g).x;   // its barrier also ends the x0 reads
#pragma unroll
            for (int r = 0; r < R; ++r) {
                own[r * RP] = Y0[r];
                own[r * RP + PW] = Y1[r];
            }
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const bool rl = (r < R - 1) || top_live;
                const double b0 = rl ? h2 : 0.0;
                const double b1 = rl && col1_live ? h2 : 0.0;
                X0[r] = 0.0; X1[r] = 0.0; Y0[r] = b0; Y1[r] = b1;
                if constexpr (VERIFY) {
                    Wa0[VERIFY ? r : 0] = Wa1[VERIFY ? r : 0] = Wb0[VERIFY ? r : 0] = Wb1[VERIFY ? r : 0] = 0.0;
                    x0[VERIFY ? r : 0] = x1[VERIFY ? r : 0] = 0.0;
                }
                own[r * RP] = b0;
                own[r * RP + PW] = b1;
            }
            if constexpr (CL > 1) {   // halo rows (the neighbours' boundary rows, all live): p_1 = b, p_0 = 0
                const double hb1 = col1_live ? h2 : 0.0;
                if (halo_lo) {
                    Sg[p + 1] = h2;
                    Sg[PW + p + 1] = hb1;
                    hst[2 * p] = hst[2 * p + 1] = 0.0;
                }
                if (halo_hi) {
                    Sg[(K::SL * R + 1) * RP + p + 1] = h2;
                    Sg[(K::SL * R + 1) * RP + PW + p + 1] = hb1;
                    hst[N + 2 * p] = hst[N + 2 * p + 1] = 0.0;
                }
            }
        }
        tsync<TPS, GROUPS>(g);                               // the grid holds p_1 = b (XM = 2: r0)
        const double bnorm = h2 * (double)K::C;              // ||b||_2 = h^2 sqrt(n), n = C^2
        const double m1 = col1_live ? 1.0 : 0.0, mt = top_live ? 1.0 : 0.0;
        double beta1 = 0.0, tol_b = 0.0, inv_beta1 = 0.0;
        double invb_prev = 0.0, beta_prev = 0.0, alpha_prev = 0.0, sigma_prev = 0.0;
        double dbar = 0.0, epsln = 0.0, phibar = 0.0, cs = -1.0, sn = 0.0, s1q = 0.0, s2q = 0.0, Xq = 0.0;
        int k = 0, status = 1;

        // one step j with roles (XA/XB = p_{j-1}, YA/YB = p_j, grid = p_j); false when done
        auto step = [&](double (&XA)[R], double (&XB)[R], double (&YA)[R], double (&YB)[R]) -> bool {
            double pa0 = 0.0, pa1 = 0.0, pb0 = 0.0, pb1 = 0.0, pc0 = 0.0, pc1 = 0.0;
            double sc0 = 0.0, sc1 = 0.0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                double t0, t1;
                if constexpr (CS) stencil_cs(YA, YB, r, t0, t1, sc0, sc1);
                else stencil(YA, YB, r, westp, eastp, own, t0, t1);
                T0[r] = t0;
                T1[r] = t1;
                pa0 = fma(YA[r], t0, pa0);
                pa1 = fma(YB[r], t1, pa1);
                pb0 = fma(YA[r], YA[r], pb0);
                pb1 = fma(YB[r], YB[r], pb1);
                pc0 += YA[r];
                pc1 += YB[r];
            }
            double4 S = tsum3<TPS, GROUPS>(pa0 + pa1, pb0 + pb1, pc0 + pc1, red, tg, g);
            if constexpr (CL > 1) {
                // K3b: the CTA sums are pushed into every CTA of the cluster and added there in rank order
                // (the same association everywhere); the boundary rows' t = A p_j go to the neighbour that
                // keeps them as a halo row.  One cluster barrier per step publishes both (buffers alternate
                // by step parity); every read after it is local.
                const int par = gk & 1;
                const uint32_t bar = sm32(mbar + par);
                double* tab = part + 4 * CL * par;            // [CL][4] of this parity
                if (tg == 0) mbar_expect_tx(bar, tx_bytes);
                if (tg < 3 * CL) {
                    const int q = tg % 3, dst = tg / 3;
                    st_async_f64(mapa32(sm32(tab + 4 * rank + q), dst), q == 0 ? S.x : (q == 1 ? S.y : S.z),
                                 mapa32(bar, dst));
                }
                if (s == 0 && rank > 0) {                    // first row = the row above rank - 1's last one
                    const uint32_t d = mapa32(sm32(thb + (2 * par + 1) * N + 2 * p), rank - 1);
                    const uint32_t rb = mapa32(bar, rank - 1);
                    st_async_f64(d, T0[0], rb);
                    st_async_f64(d + 8, T1[0], rb);
                }
                if (s == K::SL - 1 && rank < CL - 1) {       // last row = the row below rank + 1's first one
                    const uint32_t d = mapa32(sm32(thb + 2 * par * N + 2 * p), rank + 1);
                    const uint32_t rb = mapa32(bar, rank + 1);
                    st_async_f64(d, T0[R - 1], rb);
                    st_async_f64(d + 8, T1[R - 1], rb);
                }
                mbar_wait_cluster(bar, (gk >> 1) & 1u);
                double sx = 0.0, sy = 0.0, sz = 0.0;
#pragma unroll
                for (int q = 0; q < CL; ++q) {
                    sx += tab[4 * q];
                    sy += tab[4 * q + 1];
                    sz += tab[4 * q + 2];
                }
                S = make_double4(sx, sy, sz, 0.0);
            }
            const double bb = S.y;
            const double invb = bb > 0.0 ? rsqrt(bb) : 0.0;
            const double beta = __dmul_rn(bb, invb);         // beta_j = ||p_j||
            const double alpha = __dmul_rn(S.x, __dmul_rn(invb, invb));   // alpha_j = v_j^T A v_j
            const double sigma = __dmul_rn(S.z, invb);       // 1^T v_j
            // ---- Givens rotation of MINRES iteration k = j-1 (Paige-Saunders), gamma_k = hypot(gbar, beta_j);
            // only the stopping test depends on it, so the p_{j+1} pass below does not wait for it
            double phi = 0.0, oldeps = 0.0, delta = 0.0, invg = 0.0;
            if (k > 0) {
                // explicit roundings: the VERIFY instantiation must produce the same bits
                oldeps = epsln;
                delta = __fma_rn(cs, dbar, __dmul_rn(sn, alpha_prev));
                const double gbar = __fma_rn(sn, dbar, -__dmul_rn(cs, alpha_prev));
                epsln = __dmul_rn(sn, beta);
                dbar = -__dmul_rn(cs, beta);
                const double gg = __fma_rn(gbar, gbar, bb);
                invg = gg > 0.0 ? rsqrt(gg) : 1.0 / DBL_MIN;
                cs = __dmul_rn(gbar, invg);
                sn = __dmul_rn(beta, invg);
                phi = __dmul_rn(cs, phibar);
                phibar = __dmul_rn(sn, phibar);
                // 1^T w_k by the scalar recurrence (R26), Q_k = Q_{k-1} + phi_k 1^T w_k
                const double sq = __dmul_rn(__fma_rn(-delta, s1q, __fma_rn(-oldeps, s2q, sigma_prev)), invg);
                s2q = s1q;
                s1q = sq;
                Xq = __fma_rn(phi, sq, Xq);
            } else {                                         // j = 1: beta_1 = ||b|| (XM = 2: ||r0||)
                beta1 = beta;
                inv_beta1 = invb;
                tol_b = XM == 2 ? tol * bnorm : tol * beta1;  // Eq. (2) is relative to ||b|| either way
                phibar = beta1;
            }
            if constexpr (VERIFY) {
                if (k > 0) {
                    // w_k = (v_k - eps w_{k-2} - delta w_{k-1}) / gamma_k, v_k = p_k / beta_k = X * invb_prev
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const double u0 = (XA[r] * invb_prev - oldeps * Wb0[VERIFY ? r : 0] - delta * Wa0[VERIFY ? r : 0]) * invg;
                        const double u1 = (XB[r] * invb_prev - oldeps * Wb1[VERIFY ? r : 0] - delta * Wa1[VERIFY ? r : 0]) * invg;
                        Wb0[VERIFY ? r : 0] = Wa0[VERIFY ? r : 0];
                        Wb1[VERIFY ? r : 0] = Wa1[VERIFY ? r : 0];
                        Wa0[VERIFY ? r : 0] = u0;
                        Wa1[VERIFY ? r : 0] = u1;
                        x0[VERIFY ? r : 0] = fma(phi, u0, x0[VERIFY ? r : 0]);
                        x1[VERIFY ? r : 0] = fma(phi, u1, x1[VERIFY ? r : 0]);
                    }
                }
            }
            // ---- p_{j+1} = t / beta_j - (alpha_j / beta_j) p_j - (beta_j / beta_{j-1}) p_{j-1}, into X
            const double ct = invb, c1 = -alpha * invb, c0 = k == 0 ? 0.0 : -beta * invb_prev;
            const double ct1 = ct * m1, ctt = ct * mt, ctt1 = ctt * m1;   // phantom nodes stay 0
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double sa = (r == R - 1) ? ctt : ct;
                const double sb = (r == R - 1) ? ctt1 : ct1;
                const double q0 = fma(sa, T0[r], fma(c1, YA[r], c0 * XA[r]));
                const double q1 = fma(sb, T1[r], fma(c1, YB[r], c0 * XB[r]));
                XA[r] = q0;
                XB[r] = q1;
                own[r * RP] = q0;
                own[r * RP + PW] = q1;
            }
            if constexpr (CL > 1) {
                // the halo rows' p_{j+1}, rebuilt from the neighbour's t with the same operations it applies to
                // its own boundary row (a full row: coefficient ct, ct1 on the phantom column), so both copies
                // agree bit for bit; the grid halo row holds p_j, hst p_{j-1}
                const int par = gk & 1;
                ++gk;
                if (halo_lo) {
                    double* gh = Sg + p + 1;
                    const double* tb = thb + 2 * par * N + 2 * p;
                    double* hs = hst + 2 * p;
                    const double y0 = gh[0], y1 = gh[PW];
                    const double q0 = fma(ct, tb[0], fma(c1, y0, c0 * hs[0]));
                    const double q1 = fma(ct1, tb[1], fma(c1, y1, c0 * hs[1]));
                    hs[0] = y0;
                    hs[1] = y1;
                    gh[0] = q0;
                    gh[PW] = q1;
                }
                if (halo_hi) {
                    double* gh = Sg + (K::SL * R + 1) * RP + p + 1;
                    const double* tb = thb + (2 * par + 1) * N + 2 * p;
                    double* hs = hst + N + 2 * p;
                    const double y0 = gh[0], y1 = gh[PW];
                    const double q0 = fma(ct, tb[0], fma(c1, y0, c0 * hs[0]));
                    const double q1 = fma(ct1, tb[1], fma(c1, y1, c0 * hs[1]));
                    hs[0] = y0;
                    hs[1] = y1;
                    gh[0] = q0;
                    gh[PW] = q1;
                }
            }
            // stopping test of iteration k (uniform across the system); the p_{j+1} pass of the
            // last step is discarded
            if (k == 0) {
                if (beta1 == 0.0) { status = 0; return false; }
                if (XM == 2 && beta1 <= tol_b) { status = 0; return false; }   // x0 already meets the tolerance
            } else {
                if (!(phibar == phibar) || !(beta == beta)) { status = 3; return false; }
                if (phibar <= tol_b) { status = 0; return false; }       // phibar / ||b|| <= tol
                if (k >= max_iter) return false;
            }
            tsync<TPS, GROUPS>(g);                           // the grid holds p_{j+1}
            invb_prev = invb;
            beta_prev = beta;
            alpha_prev = alpha;
            sigma_prev = sigma;
            ++k;
            return true;
        };
        for (;;) {
            if (!step(X0, X1, Y0, Y1)) break;
            if (!step(Y0, Y1, X0, X1)) break;
        }
        (void)beta_prev;
        double relres = XM == 2 ? phibar / bnorm : phibar * inv_beta1;
        if constexpr (VERIFY) {
            // true residual ||b - A x|| / ||b||: x goes through the grid (the last step's grid reads
            // precede its reduction barrier)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                own[r * RP] = x0[VERIFY ? r : 0];
                own[r * RP + PW] = x1[VERIFY ? r : 0];
            }
            tsync<TPS, GROUPS>(g);
            double rr = 0.0, sc0 = 0.0, sc1 = 0.0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const bool rl = (r < R - 1) || top_live;
                double t0, t1;
                if constexpr (CS) stencil_cs(x0, x1, r, t0, t1, sc0, sc1);
                else stencil(x0, x1, r, westp, eastp, own, t0, t1);
                const double res0 = rl ? h2 - t0 : 0.0;
                const double res1 = rl && col1_live ? h2 - t1 : 0.0;
                rr = fma(res0, res0, fma(res1, res1, rr));
            }
            rr = tsum3<TPS, GROUPS>(rr, 0.0, 0.0, red, tg, g).x;
            relres = XM == 2 ? sqrt(rr) / bnorm : sqrt(rr) * inv_beta1;
            if constexpr (XM == 1) {                         // the coarse solution for the fine half's x0
                double* xo = xio + (size_t)sj * K::C * K::C;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int j = j0 + r;
                    if (j > K::C) continue;
                    xo[(j - 1) * K::C + (i0 - 1)] = x0[VERIFY ? r : 0];
                    if (col1_live) xo[(j - 1) * K::C + (i1 - 1)] = x1[VERIFY ? r : 0];
                }
            }
        }
#ifdef MLMC_TUNING
        if (tg == 0 && g_trace) {
            const unsigned idx = atomicAdd(&g_trace_n, 1u);
            if (idx < g_trace_cap) {
                unsigned smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                g_trace[4 * (size_t)idx] = trace_t0;
                g_trace[4 * (size_t)idx + 1] = gtimer();
                g_trace[4 * (size_t)idx + 2] = ((unsigned long long)smid << 32) | (unsigned)N;
                g_trace[4 * (size_t)idx + 3] = ((unsigned long long)(rank * 2 + slot) << 32) | (unsigned)job;
            }
        }
#endif
        if (tg == 0 && rank == 0) {
            double* o = out + (size_t)sj * kRecLen;
            o[0 + slot] = h2 * (XM == 2 ? sum_x0 + Xq : Xq);
            o[2 + slot] = (double)k;
            o[4 + slot] = relres;
            o[6 + slot] = (double)status;
        }
        tsync<TPS, GROUPS>(g);      // grid reuse by the next job
    }
    if constexpr (CL > 1) cg::this_cluster().sync();   // no CTA leaves while a peer may still read its memory
}

template <int N, int R, int MINB, int CM, bool VERIFY, int XM = 0>
cudaError_t run_tile(const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot, unsigned* ctr,
                     const int* order, double* xio, cudaStream_t s) {
    // x-modes exist where the coupled sample's other half is a tile mesh: XM 1 on N <= 32 (coarse halves),
    // XM 2 on N >= 16 (fine halves)
    if constexpr ((XM == 1 && N > 32) || (XM == 2 && N < 16) || (XM == 1 && !VERIFY)) {
        return cudaErrorNotSupported;
    } else {
    using K = TileCfg<N, R, MINB, CM>;
    auto kern = minres_tile_kernel<N, R, MINB, CM, VERIFY, XM>;
    static PerDevice<KernelOcc> occ_cache;
    const KernelOcc occ = occ_of(occ_cache, kern, K::BLOCK, K::SMEM);
    if (occ.err != cudaSuccess) return occ.err;
    const uint64_t need = (nb + K::GROUPS - 1) / K::GROUPS;
    uint64_t grid = std::min<uint64_t>(need, (uint64_t)occ.per_sm * occ.sms);
#ifdef MLMC_TUNING
    {   // MLMC_TILE_CTAS_N<N>=c: at most c persistent CTAs (A/B of leaving SMs to the other levels of a step;
        // configs[1] level 3 capped at 128 / 112 / 100 / 90 / 80 CTAs: C2 step 2.33 / 2.33 / 2.39 / 2.65 / 2.81 ms
        // against 2.33 uncapped, tools/gpu_call_r02ai.sh)
        char name[48];
        std::snprintf(name, sizeof(name), "MLMC_TILE_CTAS_N%d", N);
        const char* e = std::getenv(name);
        if (e && std::atoi(e) > 0) grid = std::min<uint64_t>(grid, (uint64_t)std::atoi(e));
    }
#endif
    if (grid == 0) return cudaSuccess;
    kern<<<(unsigned)grid, K::BLOCK, K::SMEM, s>>>(a, (int)nb, tol, max_iter, out, slot, ctr, order, xio);
    return cudaGetLastError();
    }
}

// K3b launch: persistent clusters of CL CTAs (one system each), as many as fit at once
template <int N, int R, int CL>
cudaError_t run_cluster(const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot, unsigned* ctr,
                        const int* order, cudaStream_t s) {
    using K = TileCfg<N, R, 1, 0, CL>;
    auto kern = minres_tile_kernel<N, R, 1, 0, false, 0, CL>;
    static PerDevice<int> mc_cache;                      // per device: smem / cluster attributes, cluster occupancy
    cudaError_t de = cudaSuccess;
    const int max_clusters = mc_cache.get([&]() -> int {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::SMEM);
        if (e == cudaSuccess && CL > 8) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return -(int)e;
        cudaLaunchConfig_t qc = {};
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = CL;
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        qc.gridDim = dim3(CL * 16);
        qc.blockDim = dim3(K::BLOCK);
        qc.dynamicSmemBytes = K::SMEM;
        qc.attrs = qa;
        qc.numAttrs = 1;
        int mcl = 0;
        e = cudaOccupancyMaxActiveClusters(&mcl, kern, &qc);
        if (e != cudaSuccess) return -(int)e;
        return mcl < 1 ? -(int)cudaErrorInvalidConfiguration : mcl;
    }, &de);
    if (de != cudaSuccess) return de;
    if (max_clusters < 0) return (cudaError_t)(-max_clusters);
    const int clusters = (int)std::min<uint64_t>(nb, (uint64_t)max_clusters);
    if (clusters <= 0) return cudaSuccess;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(clusters * CL);
    cfg.blockDim = dim3(K::BLOCK);
    cfg.dynamicSmemBytes = K::SMEM;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a, (int)nb, tol, max_iter, out, slot, ctr, order, (double*)nullptr);
}

}  // namespace

// K3b (SURVEY 2.C, 8(a) a6a "resident" layout): h = 1/128 on 4-CTA clusters (32 rows per CTA), h = 1/256 on
// 16-CTA clusters (16 rows per CTA); each CTA holds its rows like the h = 1/64 tile (8 rows x 2 columns per
// thread, conductances in registers).  MLMC_MINRES_K3B=0 hands those meshes back to K3c (A/B runs).
bool minres_cluster_supported(int N) {
    static int env = -1;
    if (env < 0) {
        const char* e = std::getenv("MLMC_MINRES_K3B");
        env = (e && e[0] == '0') ? 0 : 1;
    }
    return env == 1 && (N == 128 || N == 256);
}

cudaError_t launch_minres_cluster(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                                  unsigned* ctr, const int* order, cudaStream_t s) {
    if (nb == 0) return cudaSuccess;
#ifdef MLMC_TUNING
    {   // MLMC_MINRES_CLUSTER_N128=8: 8-CTA clusters of 128-thread CTAs (two systems' slabs per SM): 21.8 vs
        // 21.7 ms for 148 systems, 61.3 vs 60.3 ms for 441 (tools/gpu_call_r02ae.sh)
        char name[64];
        std::snprintf(name, sizeof(name), "MLMC_MINRES_CLUSTER_N%d", N);
        const char* e = std::getenv(name);
        const int v = e ? std::atoi(e) : 0;
        if (N == 128 && v == 8) return run_cluster<128, 8, 8>(a, nb, tol, max_iter, out, slot, ctr, order, s);
    }
#endif
    switch (N) {
        case 128: return run_cluster<128, 8, 4>(a, nb, tol, max_iter, out, slot, ctr, order, s);
        case 256: return run_cluster<256, 8, 16>(a, nb, tol, max_iter, out, slot, ctr, order, s);
        default: return cudaErrorNotSupported;
    }
}

// Tile shape per mesh: MLMC_MINRES_TILE_N<N>=<index> selects an alternative for tuning runs;
// -1 hands the mesh back to the column-strip kernel (k_minres.cu).
int minres_tile_variant(int N) {
    const int slot = N == 8 ? 3 : N == 16 ? 0 : N == 32 ? 1 : N == 64 ? 2 : -1;
    if (slot < 0) return -1;
#ifndef MLMC_TUNING
    return 0;          // the production build carries only the measured-best shape per mesh (v0)
#else
    static int v[4] = {-2, -2, -2, -2};
    if (v[slot] == -2) {
        char name[64];
        std::snprintf(name, sizeof(name), "MLMC_MINRES_TILE_N%d", N);
        const char* e = std::getenv(name);
        v[slot] = e ? std::atoi(e) : 0;
    }
    return v[slot];
#endif
}

#ifdef MLMC_TUNING
#define IF_TUNING(...) __VA_ARGS__
#else
#define IF_TUNING(...)
#endif
// MLMC_MINRES_K3B_N64=1: h = 1/64 through the K3b cluster kernel (a cross-check of its exchange, not a default)
static bool k3b_n64() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("MLMC_MINRES_K3B_N64");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}
// Variant table (index = MLMC_MINRES_TILE_N<N>): <N, R, MINB, CM>; measured with tools/tune_minres.py.
template <bool V, int XM>
static cudaError_t tile_dispatch(int N, int var, const double* a, uint64_t nb, double tol, int max_iter, double* out,
                                 int slot, unsigned* ctr, const int* order, double* xio, cudaStream_t s) {
    (void)var;
    switch (N) {
        case 8:   // four systems per warp (8 threads each, 4 rows x 2 columns per thread), 16 per CTA
            // (round 2: half as many threads share each system's scalar recurrences as in the former two systems
            // per warp <8, 2, 4>, now v1: C2 step 2.355 / 2.360 vs 2.380 / 2.379 ms, alternating runs)
            IF_TUNING(if (var == 1) return run_tile<8, 2, 4, 0, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            IF_TUNING(if (var == 2) return run_tile<8, 2, 5, 0, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            // (conductances in shared memory with 8 / 6 systems-pairs per SM: 0.133 / 0.127 ms vs 0.109 ms on
            // configs[1] level 0; 16 systems per warp-pair cannot hide the extra shared loads)
            return run_tile<8, 4, 3, 0, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);
        case 16:
            IF_TUNING(if (var == 1) return run_tile<16, 2, 4, 0, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            IF_TUNING(if (var == 2) return run_tile<16, 2, 6, 0, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            // (conductances in shared memory, 6 / 8 CTAs per SM: level-1 pass 0.60 / 0.61 ms vs 0.51 ms)
            // v3 (8 rows per thread, 16 systems per 128-thread CTA: the scalar recurrences shared by half as
            // many threads): 0.266 vs 0.206 ms per level-1 launch, C2 step 2.41 vs 2.36 ms (255 registers, spills)
            IF_TUNING(if (var == 3) return run_tile<16, 8, 2, 0, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            // v4 (capped at 128 registers for 4 CTAs per SM; 168 B spilled): C2 step 2.364 vs 2.342 ms
            IF_TUNING(if (var == 4) return run_tile<16, 4, 4, 0, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            return run_tile<16, 4, 3, 0, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);
        case 32:
            IF_TUNING(if (var == 1) return run_tile<32, 4, 4, 1, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            IF_TUNING(if (var == 2) return run_tile<32, 4, 4, 3, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            IF_TUNING(if (var == 3) return run_tile<32, 2, 3, 0, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            // v4 / v5 (conductances in shared memory, 5 / 4 systems per SM): 0.80 / 0.81 ms vs v0 0.74 ms
            // on configs[1] level 2, bit-identical records
            IF_TUNING(if (var == 4) return run_tile<32, 4, 5, 4, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            IF_TUNING(if (var == 5) return run_tile<32, 4, 4, 4, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            // v6 (8 rows per thread, 2 systems per CTA, 4 per SM): 0.524 vs 0.490 ms per level-2 launch, C2 step
            // 2.344 vs 2.361 ms (within run-to-run noise)
            IF_TUNING(if (var == 6) return run_tile<32, 8, 2, 0, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            // v7 (128 registers, 4 CTAs per SM; 124 B spilled): 0.537 vs 0.496 ms per launch, C2 step 2.397 vs 2.342 ms
            IF_TUNING(if (var == 7) return run_tile<32, 4, 4, 0, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            return run_tile<32, 4, 3, 0, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);
        case 64:
            // measured (configs[1] level 3, 300 systems): v0 2.04 ms, v1 2.23, v2 3.74, v3 3.67, v4 2.97
            // (v2 / v3, 512-thread systems, dropped: the one-warp cross-warp reduction holds <= 10 warps)
            // (v4: every conductance in shared memory, two systems per SM; bit-identical records, but the
            // ~60 shared loads per thread and step outweigh the second resident system); per launch
            // (tools/tune_minres.py): v0 1.671 ms, v5 (west conductances in shared memory, no in-loop
            // spills) 1.723, v6 (diagonal in shared memory) 1.722, v1 1.711 -- v0's few L1-resident
            // spill reloads cost less than the shared loads that remove them
            IF_TUNING(if (var == 1) return run_tile<64, 8, 1, 3, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            IF_TUNING(if (var == 4) return run_tile<64, 8, 2, 4, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            IF_TUNING(if (var == 5) return run_tile<64, 8, 1, 2, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            IF_TUNING(if (var == 6) return run_tile<64, 8, 1, 1, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);)
            // K3b layout at h = 1/64 (one system per 2-CTA cluster of 128-thread CTAs, two systems' slabs per SM):
            // bit-identical records (the pairwise warp-total tree splits into the two CTAs' halves) but 2.03 vs
            // 1.65 ms per level-3 launch, C2 step 2.70 vs 2.34 ms; kept as the cross-check of the cluster
            // exchange (MLMC_MINRES_K3B_N64=1, tests/test_gpu_parity_full.py)
            if constexpr (!V && XM == 0)
                if (k3b_n64()) return run_cluster<64, 8, 2>(a, nb, tol, max_iter, out, slot, ctr, order, s);
            return run_tile<64, 8, 1, 0, V, XM>(a, nb, tol, max_iter, out, slot, ctr, order, xio, s);
        default: return cudaErrorNotSupported;
    }
}

cudaError_t launch_minres_tile(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                               unsigned* ctr, bool verify, const int* order, cudaStream_t s, int xmode, double* xio) {
    const int var = minres_tile_variant(N);
    if (xmode == 1)   // coarse half of a coarse-to-fine pair: x is carried (VERIFY) and written out
        return tile_dispatch<true, 1>(N, var, a, nb, tol, max_iter, out, slot, ctr, order, xio, s);
    if (xmode == 2)
        return verify ? tile_dispatch<true, 2>(N, var, a, nb, tol, max_iter, out, slot, ctr, order, xio, s)
                      : tile_dispatch<false, 2>(N, var, a, nb, tol, max_iter, out, slot, ctr, order, xio, s);
    return verify ? tile_dispatch<true, 0>(N, var, a, nb, tol, max_iter, out, slot, ctr, order, nullptr, s)
                  : tile_dispatch<false, 0>(N, var, a, nb, tol, max_iter, out, slot, ctr, order, nullptr, s);
}

// Job trace (tuning build): buf != nullptr arms it (cap records of 4 u64 on the device, count reset); buf ==
// nullptr disarms it and returns the number of records written (may exceed cap).  Production: NotSupported.
cudaError_t minres_trace(unsigned long long* buf, unsigned cap, unsigned* count) {
#ifdef MLMC_TUNING
    cudaError_t e;
    if (buf) {
        const unsigned zero = 0;
        if ((e = cudaMemcpyToSymbol(g_trace_cap, &cap, sizeof cap)) != cudaSuccess) return e;
        if ((e = cudaMemcpyToSymbol(g_trace_n, &zero, sizeof zero)) != cudaSuccess) return e;
        return cudaMemcpyToSymbol(g_trace, &buf, sizeof buf);
    }
    unsigned long long* none = nullptr;
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return e;
    if (count && (e = cudaMemcpyFromSymbol(count, g_trace_n, sizeof *count)) != cudaSuccess) return e;
    return cudaMemcpyToSymbol(g_trace, &none, sizeof none);
#else
    (void)buf; (void)cap; (void)count;
    return cudaErrorNotSupported;
#endif
}

}  // namespace mlmc
