// k_dd.cu -- K3d: MINRES for ONE fine sample split into row slabs over ranks.
//
// The method is K3c's (Eq. (2); R9, R10, R26, R27): unpreconditioned binary64 MINRES from
// x0 = 0 on the 5-point P1 operator, the Lanczos vector unnormalised (p_{j+1} = A p_j / beta_j -
// (alpha_j/beta_j) p_j - (beta_j/beta_{j-1}) p_{j-1}), one fused reduction (p^T A p, p^T p, 1^T p) per
// step, the Paige-Saunders Givens recurrence and the QoI from the scalar recurrence of 1^T w_k; stop at
// phibar_k / ||b|| <= tol.  Only the data distribution differs.
//
// Distribution.  Rank r of G owns the interior grid rows j0 <= j < j1 (an even split of 1..N-1) and
// stores rows j0-2 .. j1+1 of five binary64 planes: three rotating Lanczos vectors (p_{j-1}, p_j,
// p_{j+1}) and the edge conductances cE, cN (built locally from the sample's coefficients: no
// exchange).  A pass forms p_{j+1} on the tile + 1-node halo from p_j (2-node halo) and p_{j-1}
// (1-node halo) in shared memory, then t_{j+1} = A p_{j+1} and the three partial sums on the owned
// rows; it stores p_{j+1} on the owned rows AND on the halo rows j0-1 and j1, which the neighbours own
// and compute bit-identically (same inputs, same operation order).  So the only halo traffic per step
// is ONE row per neighbour (rows j0+1 -> lower, j1-2 -> upper; received into ghost rows j0-2 and
// j1+1), plus one all-reduce of three doubles -- both issued by the caller between dd_pass_kernel and
// dd_scalar_kernel (torch.distributed / NCCL over NVLink; nothing to exchange for G = 1).
//
// Per step: dd_pass_kernel (tiles of 32 x 16 owned nodes, one CTA each; per-CTA partials summed in
// CTA order by the last CTA to finish: deterministic) -> [exchange] -> dd_scalar_kernel (one thread: the
// Givens step of MINRES iteration k, stopping test, next pass's coefficients, plane rotation); for G = 1
// the last CTA of the pass takes the scalar step itself (one launch per step).  Both
// kernels take their step-dependent values from the device state, so a chunk of steps is a sequence
// of identical launches (CUDA-graph capturable for G = 1).  The working set of a slab (5 planes,
// 10.5 MB at h = 1/512 for G = 1) stays L2-resident, so a step costs ~L2 bandwidth + two launches.
#include <cuda_runtime.h>
#include <algorithm>
#include <cfloat>
#include <cstdint>

#include "internal.h"

namespace mlmc {
namespace {

constexpr int DT = 256;                  // threads per CTA
constexpr int DTW = 32, DTH = 16;        // owned tile (static smem: 4 boxes + PN = 28 KB)
constexpr int DBW = DTW + 4, DBH = DTH + 4;   // loaded box (2-node halo)
constexpr int DPW = DTW + 2, DPH = DTH + 2;   // p_{j+1} region (1-node halo)

__device__ __forceinline__ double ld(const double* plane, int pitch, int lr, int rows, int col, int ncol) {
    return (lr >= 0 && lr < rows && col >= 0 && col < ncol) ? plane[(size_t)lr * pitch + col] : 0.0;
}

// Build the slab planes of one sample from its 2N^2 triangle coefficients (R10): P0 = p_0 = 0,
// P1 = b = h^2 on interior nodes, P2 = 0, cE(i,j) = (aL(i,j) + aU(i,j-1))/2, cN(i,j) = (aU(i,j) + aL(i-1,j))/2.
// Stored column c = i + 1 (c = 0: i = -1, padding); local row r = j - (j0 - 2).
__global__ void dd_init_kernel(const double* __restrict__ a, int N, int j0, int rows, int pitch,
                               double* __restrict__ planes, size_t plane_stride, DDState* __restrict__ st,
                               double tol, int max_iter) {
    const int C = N - 1;
    const double h = 1.0 / N, h2 = h * h;
    const size_t total = (size_t)rows * pitch;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(e / pitch), c = (int)(e % pitch);
        const int j = j0 - 2 + r, i = c - 1;
        const bool in = i >= 1 && i <= C && j >= 1 && j <= C;
        planes[e] = 0.0;
        planes[plane_stride + e] = in ? h2 : 0.0;
        planes[2 * plane_stride + e] = 0.0;
        double ce = 0.0, cn = 0.0;
        if (i >= 0 && i < N && j >= 1 && j < N) ce = 0.5 * (a[2 * (j * N + i)] + a[2 * ((j - 1) * N + i) + 1]);
        if (i >= 1 && i < N && j >= 0 && j < N) cn = 0.5 * (a[2 * (j * N + i) + 1] + a[2 * (j * N + i - 1)]);
        planes[3 * plane_stride + e] = ce;
        planes[4 * plane_stride + e] = cn;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        DDState s{};
        s.tol = tol;
        s.max_iter = max_iter;
        s.cs = -1.0;
        s.c1 = 1.0;                     // pass 0 copies p_1 = b (as K3c)
        s.status = 1;
        st[0] = s;
    }
}

// The MINRES scalars of the pass just reduced (identical on every rank: the sums are the all-reduced
// ones), exactly K3c's post-pass block.  One thread.
__device__ void dd_scalar_step(DDState* __restrict__ st, const double* __restrict__ sums, int N) {
    DDState s = *st;
    if (s.done) return;
    const double h = 1.0 / N, h2 = h * h;
    const double bb = sums[1];
    const double invb = bb > 0.0 ? rsqrt(bb) : 0.0;
    const double beta = __dmul_rn(bb, invb);
    const double alpha = __dmul_rn(sums[0], __dmul_rn(invb, invb));
    const double sigma = __dmul_rn(sums[2], invb);
    const int k = s.k;
    if (k > 0) {
        const double oldeps = s.epsln;
        const double delta = __fma_rn(s.cs, s.dbar, __dmul_rn(s.sn, s.alpha_prev));
        const double gbar = __fma_rn(s.sn, s.dbar, -__dmul_rn(s.cs, s.alpha_prev));
        s.epsln = __dmul_rn(s.sn, beta);
        s.dbar = -__dmul_rn(s.cs, beta);
        const double gg = __fma_rn(gbar, gbar, bb);
        const double invg = gg > 0.0 ? rsqrt(gg) : 1.0 / DBL_MIN;
        s.cs = __dmul_rn(gbar, invg);
        s.sn = __dmul_rn(beta, invg);
        const double phi = __dmul_rn(s.cs, s.phibar);
        s.phibar = __dmul_rn(s.sn, s.phibar);
        const double sq = __dmul_rn(__fma_rn(-delta, s.s1q, __fma_rn(-oldeps, s.s2q, s.sigma_prev)), invg);
        s.s2q = s.s1q;
        s.s1q = sq;
        s.Xq = __fma_rn(phi, sq, s.Xq);
    } else {
        s.beta1 = beta;
        s.inv_beta1 = invb;
        s.tol_b = s.tol * beta;
        s.phibar = beta;
    }
    bool done = false;
    if (k == 0) {
        if (s.beta1 == 0.0) { s.status = 0; done = true; }
    } else {
        if (!(s.phibar == s.phibar) || !(beta == beta)) { s.status = 3; done = true; }
        else if (s.phibar <= s.tol_b) { s.status = 0; done = true; }
        else if (k >= s.max_iter) done = true;
    }
    if (done) {
        s.done = 1;
        s.Q = h2 * s.Xq;
        s.relres = s.phibar * s.inv_beta1;
    } else {
        s.ct = invb;
        s.c1 = -alpha * invb;
        s.c0 = k == 0 ? 0.0 : -beta * s.invb_prev;
        s.invb_prev = invb;
        s.alpha_prev = alpha;
        s.sigma_prev = sigma;
        s.k = k + 1;
        s.step += 1;
    }
    *st = s;
}

__global__ void dd_scalar_kernel(DDState* __restrict__ st, const double* __restrict__ sums, int N) {
    if (threadIdx.x == 0) dd_scalar_step(st, sums, N);
}

// One 32 x 16 tile of a pass: p_{j+1} = ct A p_j + c1 p_j + c0 p_{j-1} on the tile + 1-node halo (shared
// memory), t_{j+1} = A p_{j+1} and the partial sums on the owned nodes; p_{j+1} stored on the owned nodes and on
// the slab's halo rows j0-1 / j1 (the neighbours' rows, bit-identical).  Returns this thread's partials.
struct DDSmem {
    double box[4][DBH][DBW];       // p_j, p_{j-1}, cE, cN
    double PN[DPH][DPW];
};
// send_lo / send_hi (peer-memory exchange, dd_peer_kernel): the row in the lower / upper neighbour's p_{j+1}
// plane that receives this slab's row j0 + 1 / j1 - 2 (its ghost row), or null -- the halo is pushed by the
// tile that forms it, straight into the neighbour's memory (NVLink stores between GPUs)
__device__ __forceinline__ double3 dd_tile(int tile, int N, int j0, int j1, int rows, int pitch, double* planes,
                                           size_t plane_stride, int step, double ct, double c1, double c0, DDSmem& sm,
                                           double* send_lo = nullptr, double* send_hi = nullptr) {
    const int C = N - 1, tid = threadIdx.x, NT = blockDim.x;
    const int tiles_x = (C + DTW - 1) / DTW;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int x0 = 1 + tx * DTW;             // first owned column (grid i)
    const int y0 = j0 + ty * DTH;            // first owned row (grid j)
    const int pcur = (step + 1) % 3, pprev = step % 3, pnext = (step + 2) % 3;
    const double* Pj = planes + (size_t)pcur * plane_stride;
    const double* Pp = planes + (size_t)pprev * plane_stride;
    const double* CE = planes + 3 * plane_stride;
    const double* CN = planes + 4 * plane_stride;
    // box rows y0-2 .. y0+DTH+1 (local r = y - (j0-2)), columns x0-2 .. x0+DTW+1 (stored c = i + 1)
    const int r0 = y0 - 2 - (j0 - 2), c0i = x0 - 2 + 1;
    for (int q = tid; q < DBW * DBH; q += NT) {
        const int bx = q % DBW, by = q / DBW;
        const int r = r0 + by, c = c0i + bx;
        sm.box[0][by][bx] = ld(Pj, pitch, r, rows, c, pitch);
        sm.box[1][by][bx] = ld(Pp, pitch, r, rows, c, pitch);
        sm.box[2][by][bx] = ld(CE, pitch, r, rows, c, pitch);
        sm.box[3][by][bx] = ld(CN, pitch, r, rows, c, pitch);
    }
    __syncthreads();
    const int jlo = max(j0 - 1, 1), jhi = min(j1, C);   // rows where p_{j+1} is formed (owned + halo rows)
    for (int q = tid; q < DPW * DPH; q += NT) {
        const int x = q % DPW, y = q / DPW, bx = x + 1, by = y + 1;
        const int gi = x0 - 1 + x, gj = y0 - 1 + y;
        double pn = 0.0;
        if (gi >= 1 && gi <= C && gj >= jlo && gj <= jhi) {
            const double ce = sm.box[2][by][bx], cw = sm.box[2][by][bx - 1], cn = sm.box[3][by][bx],
                         cs = sm.box[3][by - 1][bx];
            const double d = (ce + cw) + (cn + cs);
            double tv = d * sm.box[0][by][bx];
            tv = fma(-ce, sm.box[0][by][bx + 1], tv);
            tv = fma(-cw, sm.box[0][by][bx - 1], tv);
            tv = fma(-cn, sm.box[0][by + 1][bx], tv);
            tv = fma(-cs, sm.box[0][by - 1][bx], tv);
            pn = fma(ct, tv, fma(c1, sm.box[0][by][bx], c0 * sm.box[1][by][bx]));
        }
        sm.PN[y][x] = pn;
    }
    __syncthreads();
    double* Pn = planes + (size_t)pnext * plane_stride;
    double sa = 0.0, sb = 0.0, sc = 0.0;
    const int ylim = min(y0 + DTH, j1);          // owned rows of this tile
    for (int q = tid; q < DTW * DTH; q += NT) {
        const int x = q % DTW, y = q / DTW;
        const int gi = x0 + x, gj = y0 + y;
        if (gi > C || gj >= ylim) continue;
        const int bx = x + 2, by = y + 2, px = x + 1, py = y + 1;
        const double ce = sm.box[2][by][bx], cw = sm.box[2][by][bx - 1], cn = sm.box[3][by][bx],
                     cs = sm.box[3][by - 1][bx];
        const double d = (ce + cw) + (cn + cs);
        const double pv = sm.PN[py][px];
        double tv = d * pv;
        tv = fma(-ce, sm.PN[py][px + 1], tv);
        tv = fma(-cw, sm.PN[py][px - 1], tv);
        tv = fma(-cn, sm.PN[py + 1][px], tv);
        tv = fma(-cs, sm.PN[py - 1][px], tv);
        sa = fma(pv, tv, sa);
        sb = fma(pv, pv, sb);
        sc += pv;
        Pn[(size_t)(gj - (j0 - 2)) * pitch + gi + 1] = pv;
    }
    // the halo rows j0-1 (first tile row) and j1 (last tile row) of p_{j+1}: the neighbours' values, bit for bit
    if (ty == 0 && j0 - 1 >= 1)
        for (int x = tid; x < DTW; x += NT)
            if (x0 + x <= C) Pn[(size_t)1 * pitch + x0 + x + 1] = sm.PN[0][x + 1];
    if (y0 + DTH >= j1 && j1 <= C) {
        const int py = j1 - (y0 - 1);
        for (int x = tid; x < DTW; x += NT)
            if (x0 + x <= C) Pn[(size_t)(j1 - (j0 - 2)) * pitch + x0 + x + 1] = sm.PN[py][x + 1];
    }
    if (send_lo && y0 <= j0 + 1 && j0 + 1 < ylim) {          // row j0 + 1 -> rank - 1's ghost row
        const int py = j0 + 1 - (y0 - 1);
        for (int x = tid; x < DTW; x += NT)
            if (x0 + x <= C) send_lo[x0 + x + 1] = sm.PN[py][x + 1];
    }
    if (send_hi && y0 <= j1 - 2 && j1 - 2 < ylim) {          // row j1 - 2 -> rank + 1's ghost row
        const int py = j1 - 2 - (y0 - 1);
        for (int x = tid; x < DTW; x += NT)
            if (x0 + x <= C) send_hi[x0 + x + 1] = sm.PN[py][x + 1];
    }
    __syncthreads();                              // box / PN free for the next tile
    return make_double3(sa, sb, sc);
}

// CTA sum of (a, b, c) in a fixed order, valid in thread 0
__device__ __forceinline__ double3 dd_block_sum(double a, double b, double c, double (*red)[32]) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    const int tid = threadIdx.x;
    if ((tid & 31) == 0) { red[0][tid >> 5] = a; red[1][tid >> 5] = b; red[2][tid >> 5] = c; }
    __syncthreads();
    double3 t = make_double3(0.0, 0.0, 0.0);
    if (tid == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { t.x += red[0][w]; t.y += red[1][w]; t.z += red[2][w]; }
    return t;
}

__global__ void __launch_bounds__(DT)
dd_pass_kernel(int N, int j0, int j1, int rows, int pitch, double* __restrict__ planes, size_t plane_stride,
               DDState* __restrict__ st, double* __restrict__ partials, unsigned* __restrict__ counter,
               double* __restrict__ sums, int fuse) {
    __shared__ DDSmem sm;
    __shared__ double red[3][32];
    __shared__ bool last;
    const DDState s = *st;
    if (s.done) return;
    const int tid = threadIdx.x;
    const double3 p = dd_tile(blockIdx.x, N, j0, j1, rows, pitch, planes, plane_stride, s.step, s.ct, s.c1, s.c0, sm);
    const double3 t = dd_block_sum(p.x, p.y, p.z, red);
    if (tid == 0) {
        partials[3 * blockIdx.x + 0] = t.x;
        partials[3 * blockIdx.x + 1] = t.y;
        partials[3 * blockIdx.x + 2] = t.z;
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    if (tid < 32) {
        __threadfence();
        // lane l sums CTAs l, l+32, ... in order, then a fixed shuffle tree: deterministic for a given grid
        double a = 0.0, b = 0.0, c = 0.0;
        for (unsigned k = tid; k < gridDim.x; k += 32) {
            a += __ldcg(partials + 3 * k);
            b += __ldcg(partials + 3 * k + 1);
            c += __ldcg(partials + 3 * k + 2);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
            c += __shfl_xor_sync(0xffffffffu, c, o);
        }
        if (tid == 0) {
            sums[0] = a;
            sums[1] = b;
            sums[2] = c;
            *counter = 0u;
            // world = 1: nothing to all-reduce, so the last CTA also takes the scalar step (every CTA of
            // this launch has read the state before it arrived at the counter)
            if (fuse) dd_scalar_step(st, sums, N);
        }
    }
}

// World = 1, the whole solve in ONE cooperative launch: every resident CTA slot loops over the steps; each CTA takes
// tiles blockIdx.x, blockIdx.x + gridDim.x, ...; per step its partials go to partials[CTA], a grid barrier
// (arrival counter + acquire spin; all CTAs are co-resident by the cooperative launch) publishes them and
// the pass's p_{j+1}, and EVERY CTA adds the partials in CTA order and runs the identical scalar step on its
// own copy of the state (CTA 0 keeps the global one) -- one barrier per MINRES step, no launches.
__global__ void __launch_bounds__(DT)
dd_persistent_kernel(int N, int j0, int j1, int rows, int pitch, double* __restrict__ planes, size_t plane_stride,
                     DDState* __restrict__ st, double* __restrict__ partials, unsigned* __restrict__ counter,
                     double* __restrict__ sums, int ntiles) {
    __shared__ DDSmem sm;
    __shared__ double red[3][32];
    __shared__ DDState ls;
    const int tid = threadIdx.x;
    if (tid == 0) ls = *st;
    __syncthreads();
    for (unsigned gen = 1;; ++gen) {
        if (ls.done) break;                          // identical in every CTA
        double a = 0.0, b = 0.0, c = 0.0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const double3 p = dd_tile(t, N, j0, j1, rows, pitch, planes, plane_stride, ls.step, ls.ct, ls.c1, ls.c0,
                                      sm);
            a += p.x; b += p.y; c += p.z;
        }
        const double3 tsum = dd_block_sum(a, b, c, red);
        if (tid < 32) {
            // partials double-buffered by generation parity: a CTA can be one generation ahead of a slower one
            // that is still reading (it cannot be two: that needs the slower one's next arrival)
            double* pg = partials + 3 * (size_t)gridDim.x * (gen & 1u);
            if (tid == 0) {
                volatile double* pv = pg + 3 * blockIdx.x;
                pv[0] = tsum.x;
                pv[1] = tsum.y;
                pv[2] = tsum.z;
                __threadfence();                     // partials and this CTA's p_{j+1} stores before the arrival
                atomicAdd(counter, 1u);
                const unsigned target = gen * gridDim.x;
                unsigned seen;
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(counter) : "memory");
                } while (seen < target);
            }
            __syncwarp();
            // warp 0 adds the CTA partials: lane l takes CTAs l, l + 32, ... in order, then a fixed xor tree
            // (identical association in every lane and every CTA)
            double A = 0.0, B = 0.0, Cc = 0.0;
            for (unsigned k = tid; k < gridDim.x; k += 32) {
                A += __ldcg(pg + 3 * k);
                B += __ldcg(pg + 3 * k + 1);
                Cc += __ldcg(pg + 3 * k + 2);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                A += __shfl_xor_sync(0xffffffffu, A, o);
                B += __shfl_xor_sync(0xffffffffu, B, o);
                Cc += __shfl_xor_sync(0xffffffffu, Cc, o);
            }
            if (tid == 0) {
                double S[3] = {A, B, Cc};
                dd_scalar_step(&ls, S, N);
            }
        }
        __syncthreads();                             // ls (next coefficients / done) and p_{j+1} visible
    }
    if (blockIdx.x == 0 && tid == 0) {
        *st = ls;
        sums[0] = sums[1] = sums[2] = 0.0;
    }
}
// ---- World > 1 with the exchange fused into the kernel (peer memory).  Each rank runs
// its slab as dd_persistent_kernel does, and the step's collective lives in the same kernel: the tiles that
// form rows j0 + 1 / j1 - 2 store them straight into the neighbours' ghost rows (peer pointers: NVLink stores
// between GPUs), each rank's leader CTA adds its CTAs' partials and stores the rank partial into EVERY rank's
// rank-partial table, then increments every rank's arrival counter (system-scope atomics); every CTA waits
// for its rank's counter to reach world x step and adds the world rank partials in rank order -- identical on
// every rank -- before its own copy of the scalar step.  One launch covers ranks rank0 .. rank0 + gridDim.y - 1:
// all of them for the one-GPU emulation (a cooperative launch: every CTA of every rank co-resident), one per
// process on a multi-GPU node (each rank's grid cooperative on its GPU; the ranks wait on one another only
// through the counters, and all ranks launch).
struct DDPeerParams {
    int N, world, rank0;
    int j0[kDDMaxRanks], j1[kDDMaxRanks], rows[kDDMaxRanks], tiles[kDDMaxRanks];
    double* planes[kDDMaxRanks];
    size_t plane_stride[kDDMaxRanks];
    DDState* st[kDDMaxRanks];
    double* partials[kDDMaxRanks];     // this rank's CTA partials, [2][ctas][3]
    unsigned* counter[kDDMaxRanks];    // this rank's CTA arrivals
    double* rpart[kDDMaxRanks];        // rank partial table, [2][kDDMaxRanks][3] (written by every rank)
    unsigned* xcounter[kDDMaxRanks];   // rank arrivals (incremented by every rank)
    double* sums[kDDMaxRanks];
};

__global__ void __launch_bounds__(DT)
dd_peer_kernel(const __grid_constant__ DDPeerParams P) {
    __shared__ DDSmem sm;
    __shared__ double red[3][32];
    __shared__ DDState ls;
    const int tid = threadIdx.x, r = P.rank0 + blockIdx.y, W = P.world, pitch = P.N + 2;
    if (tid == 0) ls = *P.st[r];
    __syncthreads();
    for (unsigned gen = 1;; ++gen) {
        if (ls.done) break;                          // identical in every CTA of every rank
        const int pnext = (ls.step + 2) % 3;
        double* send_lo = r > 0 ? P.planes[r - 1] + (size_t)pnext * P.plane_stride[r - 1] +
                                      (size_t)(P.rows[r - 1] - 1) * pitch : nullptr;
        double* send_hi = r + 1 < W ? P.planes[r + 1] + (size_t)pnext * P.plane_stride[r + 1] : nullptr;
        double a = 0.0, b = 0.0, c = 0.0;
        for (int t = blockIdx.x; t < P.tiles[r]; t += gridDim.x) {
            const double3 q = dd_tile(t, P.N, P.j0[r], P.j1[r], P.rows[r], pitch, P.planes[r], P.plane_stride[r],
                                      ls.step, ls.ct, ls.c1, ls.c0, sm, send_lo, send_hi);
            a += q.x; b += q.y; c += q.z;
        }
        const double3 tsum = dd_block_sum(a, b, c, red);
        if (tid < 32) {
            double* pg = P.partials[r] + 3 * (size_t)gridDim.x * (gen & 1u);
            if (tid == 0) {
                volatile double* pv = pg + 3 * blockIdx.x;
                pv[0] = tsum.x;
                pv[1] = tsum.y;
                pv[2] = tsum.z;
                // the peer halo stores and the partial before the arrival (gpu scope: the leader's system-scope
                // release below is ordered after this CTA's writes by the acquire of the counter -- causality
                // carries them to the other GPUs' acquiring readers)
                __threadfence();
                atomicAdd(P.counter[r], 1u);
            }
            if (blockIdx.x == 0) {                   // the rank's leader: rank partial -> every rank's table
                if (tid == 0) {
                    unsigned seen;
                    do {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(P.counter[r]) : "memory");
                    } while (seen < gen * gridDim.x);
                }
                __syncwarp();
                double A = 0.0, B = 0.0, Cc = 0.0;
                for (unsigned k = tid; k < gridDim.x; k += 32) {
                    A += __ldcg(pg + 3 * k);
                    B += __ldcg(pg + 3 * k + 1);
                    Cc += __ldcg(pg + 3 * k + 2);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    A += __shfl_xor_sync(0xffffffffu, A, o);
                    B += __shfl_xor_sync(0xffffffffu, B, o);
                    Cc += __shfl_xor_sync(0xffffffffu, Cc, o);
                }
                if (tid < W) {                       // lane q stores into rank q's table
                    volatile double* t = P.rpart[tid] + 3 * ((size_t)(gen & 1u) * kDDMaxRanks + r);
                    t[0] = A;
                    t[1] = B;
                    t[2] = Cc;
                }
                __syncwarp();
                if (tid == 0) {
                    __threadfence_system();
                    for (int q = 0; q < W; ++q) atomicAdd_system(P.xcounter[q], 1u);
                }
            }
            if (tid == 0) {                          // every CTA: all ranks' partials of this step are in
                unsigned seen;
                do {
                    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(seen) : "l"(P.xcounter[r]) : "memory");
                } while (seen < gen * (unsigned)W);
                const volatile double* t = P.rpart[r] + 3 * (size_t)(gen & 1u) * kDDMaxRanks;
                double S[3] = {0.0, 0.0, 0.0};
                for (int q = 0; q < W; ++q) {        // rank order: identical on every rank
                    S[0] += t[3 * q];
                    S[1] += t[3 * q + 1];
                    S[2] += t[3 * q + 2];
                }
                dd_scalar_step(&ls, S, P.N);
            }
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && tid == 0) *P.st[r] = ls;
}

}  // namespace

int dd_tiles(int N, int j0, int j1) {
    const int C = N - 1;
    return ((C + DTW - 1) / DTW) * ((j1 - j0 + DTH - 1) / DTH);
}

cudaError_t launch_dd_init(const double* a, int N, int j0, int rows, int pitch, double* planes, size_t plane_stride,
                           DDState* st, double tol, int max_iter, cudaStream_t s) {
    const size_t total = (size_t)rows * pitch;
    const unsigned grid = (unsigned)std::min<size_t>((total + 255) / 256, 148 * 8);
    dd_init_kernel<<<grid, 256, 0, s>>>(a, N, j0, rows, pitch, planes, plane_stride, st, tol, max_iter);
    return cudaGetLastError();
}

cudaError_t launch_dd_pass(int N, int j0, int j1, int rows, int pitch, double* planes, size_t plane_stride,
                           DDState* st, double* partials, unsigned* counter, double* sums, bool fuse_scalar,
                           cudaStream_t s) {
    dd_pass_kernel<<<dd_tiles(N, j0, j1), DT, 0, s>>>(N, j0, j1, rows, pitch, planes, plane_stride, st, partials,
                                                     counter, sums, fuse_scalar ? 1 : 0);
    return cudaGetLastError();
}

// World = 1: the whole solve as one cooperative launch (all resident CTA slots); cudaErrorCooperativeLaunchTooLarge
// etc. if the device cannot co-schedule the grid (the caller then falls back to per-step launches).
cudaError_t launch_dd_persistent(int N, int j0, int j1, int rows, int pitch, double* planes, size_t plane_stride,
                                 DDState* st, double* partials, unsigned* counter, double* sums, cudaStream_t s) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dd_persistent_kernel, DT, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int ntiles = dd_tiles(N, j0, j1);
    // every resident CTA slot (all co-resident: cooperative launch), at most one tile each where they suffice
    int grid = std::min(sms * per_sm, ntiles);
    void* args[] = {&N, &j0, &j1, &rows, &pitch, &planes, &plane_stride, &st, &partials, &counter, &sums, (void*)&ntiles};
    e = cudaMemsetAsync(counter, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    e = cudaLaunchCooperativeKernel((const void*)dd_persistent_kernel, dim3(grid), dim3(DT), args, 0, s);
    if (e != cudaSuccess) return e;
    return cudaMemsetAsync(counter, 0, sizeof(unsigned), s);
}

// ranks rank0 .. rank0 + nranks - 1 in one cooperative launch (the caller zeroed the counters); every
// pointer in P device-accessible from this GPU (peer-mapped for other GPUs' ranks)
cudaError_t launch_dd_peer(const DDPeerLaunch& L, cudaStream_t s) {
    DDPeerParams P{};
    P.N = L.N;
    P.world = L.world;
    P.rank0 = L.rank0;
    for (int q = 0; q < L.world; ++q) {
        P.j0[q] = L.j0[q]; P.j1[q] = L.j1[q]; P.rows[q] = L.rows[q]; P.tiles[q] = dd_tiles(L.N, L.j0[q], L.j1[q]);
        P.planes[q] = L.planes[q]; P.plane_stride[q] = L.plane_stride[q]; P.st[q] = L.st[q];
        P.partials[q] = L.partials[q]; P.counter[q] = L.counter[q]; P.rpart[q] = L.rpart[q];
        P.xcounter[q] = L.xcounter[q]; P.sums[q] = L.sums[q];
    }
    int dev = 0, sms = 0, per_sm = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dd_peer_kernel, DT, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1 || L.nranks < 1) return cudaErrorInvalidConfiguration;
    int mt = 0;
    for (int q = L.rank0; q < L.rank0 + L.nranks; ++q) mt = std::max(mt, P.tiles[q]);
    const int ctas = std::max(1, std::min(mt, sms * per_sm / L.nranks));
    void* args[] = {&P};
    return cudaLaunchCooperativeKernel((const void*)dd_peer_kernel, dim3(ctas, L.nranks), dim3(DT), args, 0, s);
}

cudaError_t launch_dd_scalar(DDState* st, const double* sums, int N, cudaStream_t s) {
    dd_scalar_kernel<<<1, 32, 0, s>>>(st, sums, N);
    return cudaGetLastError();
}

}  // namespace mlmc
