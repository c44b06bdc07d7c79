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

__global__ void __launch_bounds__(DT)
dd_pass_kernel(int N, int j0, int j1, int rows, int pitch, double* __restrict__ planes, size_t plane_stride,
               DDState* __restrict__ st, double* __restrict__ partials, unsigned* __restrict__ counter,
               double* __restrict__ sums, int fuse) {
    __shared__ double box[4][DBH][DBW];       // p_j, p_{j-1}, cE, cN
    __shared__ double PN[DPH][DPW];
    __shared__ double red[3][DT / 32];
    __shared__ bool last;
    const DDState s = *st;
    if (s.done) return;
    const int C = N - 1, tid = threadIdx.x;
    const int tiles_x = (C + DTW - 1) / DTW;
    const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    const int x0 = 1 + tx * DTW;             // first owned column (grid i)
    const int y0 = j0 + ty * DTH;            // first owned row (grid j)
    const int pcur = (s.step + 1) % 3, pprev = s.step % 3, pnext = (s.step + 2) % 3;
    const double* Pj = planes + (size_t)pcur * plane_stride;
    const double* Pp = planes + (size_t)pprev * plane_stride;
    const double* CE = planes + 3 * plane_stride;
    const double* CN = planes + 4 * plane_stride;
    // box rows y0-2 .. y0+DTH+1 (local r = y - (j0-2)), columns x0-2 .. x0+DTW+1 (stored c = i + 1)
    const int r0 = y0 - 2 - (j0 - 2), c0 = x0 - 2 + 1;
    for (int q = tid; q < DBW * DBH; q += DT) {
        const int bx = q % DBW, by = q / DBW;
        const int r = r0 + by, c = c0 + bx;
        box[0][by][bx] = ld(Pj, pitch, r, rows, c, pitch);
        box[1][by][bx] = ld(Pp, pitch, r, rows, c, pitch);
        box[2][by][bx] = ld(CE, pitch, r, rows, c, pitch);
        box[3][by][bx] = ld(CN, pitch, r, rows, c, pitch);
    }
    __syncthreads();
    const int jlo = max(j0 - 1, 1), jhi = min(j1, C);   // rows where p_{j+1} is formed (owned + halo rows)
    for (int q = tid; q < DPW * DPH; q += DT) {
        const int x = q % DPW, y = q / DPW, bx = x + 1, by = y + 1;
        const int gi = x0 - 1 + x, gj = y0 - 1 + y;
        double pn = 0.0;
        if (gi >= 1 && gi <= C && gj >= jlo && gj <= jhi) {
            const double ce = box[2][by][bx], cw = box[2][by][bx - 1], cn = box[3][by][bx], cs = box[3][by - 1][bx];
            const double d = (ce + cw) + (cn + cs);
            double tv = d * box[0][by][bx];
            tv = fma(-ce, box[0][by][bx + 1], tv);
            tv = fma(-cw, box[0][by][bx - 1], tv);
            tv = fma(-cn, box[0][by + 1][bx], tv);
            tv = fma(-cs, box[0][by - 1][bx], tv);
            pn = fma(s.ct, tv, fma(s.c1, box[0][by][bx], s.c0 * box[1][by][bx]));
        }
        PN[y][x] = pn;
    }
    __syncthreads();
    double* Pn = planes + (size_t)pnext * plane_stride;
    double sa = 0.0, sb = 0.0, sc = 0.0;
    const int ylim = min(y0 + DTH, j1);          // owned rows of this tile
    for (int q = tid; q < DTW * DTH; q += DT) {
        const int x = q % DTW, y = q / DTW;
        const int gi = x0 + x, gj = y0 + y;
        if (gi > C || gj >= ylim) continue;
        const int bx = x + 2, by = y + 2, px = x + 1, py = y + 1;
        const double ce = box[2][by][bx], cw = box[2][by][bx - 1], cn = box[3][by][bx], cs = box[3][by - 1][bx];
        const double d = (ce + cw) + (cn + cs);
        const double pv = PN[py][px];
        double tv = d * pv;
        tv = fma(-ce, PN[py][px + 1], tv);
        tv = fma(-cw, PN[py][px - 1], tv);
        tv = fma(-cn, PN[py + 1][px], tv);
        tv = fma(-cs, PN[py - 1][px], tv);
        sa = fma(pv, tv, sa);
        sb = fma(pv, pv, sb);
        sc += pv;
        Pn[(size_t)(gj - (j0 - 2)) * pitch + gi + 1] = pv;
    }
    // the halo rows j0-1 (first tile row) and j1 (last tile row) of p_{j+1}: the neighbours' values, bit for bit
    if (ty == 0 && j0 - 1 >= 1)
        for (int x = tid; x < DTW; x += DT)
            if (x0 + x <= C) Pn[(size_t)1 * pitch + x0 + x + 1] = PN[0][x + 1];
    if (y0 + DTH >= j1 && j1 <= C) {
        const int py = j1 - (y0 - 1);
        for (int x = tid; x < DTW; x += DT)
            if (x0 + x <= C) Pn[(size_t)(j1 - (j0 - 2)) * pitch + x0 + x + 1] = PN[py][x + 1];
    }
    // block partial sums (fixed order), then the last CTA adds the partials in CTA order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
        sb += __shfl_xor_sync(0xffffffffu, sb, o);
        sc += __shfl_xor_sync(0xffffffffu, sc, o);
    }
    if ((tid & 31) == 0) { red[0][tid >> 5] = sa; red[1][tid >> 5] = sb; red[2][tid >> 5] = sc; }
    __syncthreads();
    if (tid == 0) {
        double a = 0.0, b = 0.0, c = 0.0;
        for (int w = 0; w < DT / 32; ++w) { a += red[0][w]; b += red[1][w]; c += red[2][w]; }
        partials[3 * blockIdx.x + 0] = a;
        partials[3 * blockIdx.x + 1] = b;
        partials[3 * blockIdx.x + 2] = c;
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

cudaError_t launch_dd_scalar(DDState* st, const double* sums, int N, cudaStream_t s) {
    dd_scalar_kernel<<<1, 32, 0, s>>>(st, sums, N);
    return cudaGetLastError();
}

}  // namespace mlmc
