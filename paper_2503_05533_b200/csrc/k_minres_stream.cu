// k_minres_stream.cu -- K3c: MINRES for the fine meshes (h <= 1/128), streamed through HBM.
//
// Same method as the on-chip kernels (Eq. (2); R9, R10, R26, R27): unpreconditioned
// binary64 MINRES from x0 = 0 on the 5-point P1 operator, stopped when the Paige-Saunders residual
// phibar_k / ||b|| <= tol, the QoI from the scalar recurrence of 1^T w_k.  The Lanczos vector is
// kept unnormalised (p_j = beta_j v_j, R27), so a MINRES step needs p_j, p_{j-1} and the operator.
//
// B200 mapping.  A system of n = (N-1)^2 >= 16129 unknowns no longer fits an SM, so one CTA (512
// threads, persistent, job counter) owns one system at a time and keeps five (N+1) x (N+2) binary64
// planes in a per-CTA global scratch: three rotating Lanczos vectors (zero Dirichlet ring) and the
// edge conductances cE, cN.  ONE pass over the grid per MINRES step:
//   for each 64 x 32 tile (double-buffered TMA boxes of 68 x 36 with a 2-node halo, zero-filled
//   outside the array, 4 planes per box = p_j, p_{j-1}, cE, cN):
//     t_j     = A p_j                                on the tile + 1-node halo (recomputed, not stored)
//     p_{j+1} = t_j/beta_j - (alpha_j/beta_j) p_j - (beta_j/beta_{j-1}) p_{j-1}   (tile + halo, smem)
//     t_{j+1} = A p_{j+1}                            on the tile
//     partial sums of p_{j+1}.t_{j+1}, p_{j+1}.p_{j+1}, 1.p_{j+1};  store p_{j+1} (tile) to HBM
//   one block reduction -> beta_{j+1}, alpha_{j+1}, sigma_{j+1}; Givens rotation of MINRES
//   iteration j; stopping test.
// HBM traffic per node and step: p_j, p_{j-1}, cE, cN read (the halos are L2 hits) and p_{j+1}
// written = 40 bytes -- the algorithmic minimum of this formulation (the
// textbook five-vector MINRES of SURVEY section 8(d) would move 80).  The FP64 work (two stencils,
// ~25 flops per node) sits well under the HBM time, so the kernel is HBM-bound by construction.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cfloat>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include <cooperative_groups.h>

#include "internal.h"

namespace mlmc {
namespace {
namespace cg = cooperative_groups;

constexpr int ST = 512;                  // threads per CTA
constexpr int TW = 64, TH = 32;          // tile of interior nodes
constexpr int BW = TW + 4, BH = TH + 4;  // TMA box (2-node halo)
constexpr int PW = TW + 2, PH = TH + 2;  // p_{j+1} region (1-node halo)
constexpr int NPLANE = 5;                // P0, P1, P2, CE, CN
constexpr int PL_CE = 3, PL_CN = 4;
constexpr int BOX = BW * BH;             // doubles per plane box
constexpr int BOX_BYTES = BOX * 8;       // 19584 = 153 * 128
constexpr int STAGE = 4 * BOX;           // doubles per stage (p_j, p_{j-1}, cE, cN)
constexpr size_t SMEM = (size_t)(2 * STAGE + PW * PH + 3 * (ST / 32) + 8) * 8 + 2 * 8 + 16;

// row pitch: grid columns 0..N stored at 1..N+1 (column 0 = padding), N + 2 doubles (16-byte multiple)
__host__ __device__ constexpr int pitch(int N) { return N + 2; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_box(uint32_t dst, const CUtensorMap* map, int x, int y, int plane, int slot,
                                        uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
            "r"(dst), "l"(map), "r"(x), "r"(y), "r"(plane), "r"(slot), "r"(bar)
        : "memory");
}

// Block sums of (a, b, c), bit-identical in every thread (fixed pairwise order over the warps).
__device__ __forceinline__ double3 bsum3(double a, double b, double c, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    constexpr int NW = ST / 32;
    __syncthreads();                                   // red is free (previous use finished)
    if ((threadIdx.x & 31) == 0) {
        red[3 * (threadIdx.x >> 5) + 0] = a;
        red[3 * (threadIdx.x >> 5) + 1] = b;
        red[3 * (threadIdx.x >> 5) + 2] = c;
    }
    __syncthreads();
    double v[NW][3];
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        v[w][0] = red[3 * w];
        v[w][1] = red[3 * w + 1];
        v[w][2] = red[3 * w + 2];
    }
#pragma unroll
    for (int st = 1; st < NW; st *= 2)
#pragma unroll
        for (int w = 0; w + st < NW; w += 2 * st) {
            v[w][0] += v[w + st][0];
            v[w][1] += v[w + st][1];
            v[w][2] += v[w + st][2];
        }
    return make_double3(v[0][0], v[0][1], v[0][2]);
}

// issue the 4 boxes of tile i of a pass reading planes (pc = p_j, pp = p_{j-1}) into stage s
__device__ __forceinline__ void issue_tile(const CUtensorMap* map, double* stage0, uint32_t bar0, int tiles_x, int cta,
                                           int i, int s, int pc, int pp) {
    // box origin: grid node (x0 - 2, y0 - 2); node (i, j) is stored at column i + 1, so the innermost
    // box coordinate x0 - 1 = 64 tx is even -- TMA needs the box start 16-byte aligned
    const int x = 1 + (i % tiles_x) * TW - 1, y = 1 + (i / tiles_x) * TH - 2;
    const uint32_t dst = smem_u32(stage0 + s * STAGE), bar = bar0 + 8 * s;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(4 * BOX_BYTES) : "memory");
    tma_box(dst, map, x, y, pc, cta, bar);
    tma_box(dst + BOX_BYTES, map, x, y, pp, cta, bar);
    tma_box(dst + 2 * BOX_BYTES, map, x, y, PL_CE, cta, bar);
    tma_box(dst + 3 * BOX_BYTES, map, x, y, PL_CN, cta, bar);
}

// CS > 1: one system per thread-block cluster of CS CTAs (the tiles of a pass dealt round-robin to the
// CTAs, every CTA reading the halos from the shared planes in HBM/L2); the block partials are summed
// across the cluster through distributed shared memory in rank order (identical in every CTA), and
// the cluster barrier of that exchange also publishes each pass's p_{j+1} to the whole cluster.  For
// fewer systems than SMs and long, uneven solves (the finest levels) -- a lone system gets CS SMs.
template <int CS>
__global__ void __launch_bounds__(ST, 1)
minres_stream_kernel(const __grid_constant__ CUtensorMap map, int N, const double* __restrict__ a_all, int nb,
                     double tol, int max_iter, double* __restrict__ out, int slot, unsigned* __restrict__ job_counter,
                     double* __restrict__ scratch, const int* __restrict__ order) {
    // all shared memory is dynamic so that the TMA boxes start 128-byte aligned:
    // [stage 0 | stage 1 | p_{j+1} tile | block partials | cluster partials | mbarriers | job slots]
    extern __shared__ __align__(128) double sm[];
    double* stage0 = sm;
    double* PN = sm + 2 * STAGE;                       // p_{j+1} on the tile + halo, [PH][PW]
    double* red = PN + PW * PH;                        // 3 x 16 warp partials
    double* part = red + 3 * (ST / 32);                // [2][4]: this CTA's block sums, by step parity
    uint64_t* bars = reinterpret_cast<uint64_t*>(part + 8);
    int& jobslot = *reinterpret_cast<int*>(bars + 2);
    int& jobmine = *(reinterpret_cast<int*>(bars + 2) + 1);
    const int G = N + 1, GP = pitch(N), C = N - 1;
    const size_t PLANE = (size_t)G * GP;
    const int tiles_x = (C + TW - 1) / TW, tiles_y = (C + TH - 1) / TH, T = tiles_x * tiles_y;
    const int P = 2 * N * N, tid = threadIdx.x;
    const int rank = CS > 1 ? (int)cg::this_cluster().block_rank() : 0;
    const int cta = blockIdx.x / CS;                   // system slot: scratch planes + tensor-map coordinate
    const int Tr = (T - rank + CS - 1) / CS;           // this CTA's tiles: rank, rank + CS, ...
    double* base = scratch + (size_t)cta * NPLANE * PLANE;
    const double h = 1.0 / N, h2 = h * h;
    const uint32_t bar0 = smem_u32(&bars[0]);
    if (tid == 0) {
        mbar_init(bar0);
        mbar_init(bar0 + 8);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t phase = 0;                                // bit s: parity to wait for on stage s

    const CUtensorMap* mp = &map;                      // the __grid_constant__ parameter itself (param space)
    for (;;) {
        int job;
        if constexpr (CS > 1) {
            auto cl = cg::this_cluster();
            if (rank == 0 && tid == 0) jobslot = (int)atomicAdd(job_counter, 1u);
            cl.sync();
            if (tid == 0) jobmine = *cl.map_shared_rank(&jobslot, 0);
            __syncthreads();
            job = jobmine;
        } else {
            if (tid == 0) jobslot = (int)atomicAdd(job_counter, 1u);
            __syncthreads();
            job = jobslot;
            __syncthreads();
        }
        if (job >= nb) break;
        const int sj = order ? __ldg(order + job) : job;
        const double* a = a_all + (size_t)sj * P;
        // ---- planes: cE, cN from the coefficients (R10); p_0 = 0, p_1 = b, third vector's ring = 0
        for (size_t e = (size_t)rank * ST + tid; e < PLANE; e += (size_t)CS * ST) {
            const int i = (int)(e % GP) - 1, j = (int)(e / GP);   // column 0 is padding (i = -1)
            const bool in = i >= 1 && i <= C && j >= 1 && j <= C;
            base[e] = 0.0;                                                  // P0 = p_0
            base[PLANE + e] = in ? h2 : 0.0;                                // P1 = p_1 = b
            base[2 * PLANE + e] = 0.0;                                      // P2
            double ce = 0.0, cn = 0.0;
            if (i >= 0 && i < N && j >= 1 && j < N) ce = 0.5 * (__ldg(a + 2 * (j * N + i)) + __ldg(a + 2 * ((j - 1) * N + i) + 1));
            if (i >= 1 && i < N && j < N) cn = 0.5 * (__ldg(a + 2 * (j * N + i) + 1) + __ldg(a + 2 * (j * N + i - 1)));
            base[PL_CE * PLANE + e] = ce;
            base[PL_CN * PLANE + e] = cn;
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");        // generic writes -> TMA reads
        if constexpr (CS > 1) cg::this_cluster().sync();
        else __syncthreads();
        int pprev = 0, pcur = 1, pnext = 2;             // plane roles: p_{j-1}, p_j, p_{j+1}
        // pass coefficients: p_{j+1} = ct t_j + c1 p_j + c0 p_{j-1}; the first pass copies p_1
        double ct = 0.0, c1 = 1.0, c0 = 0.0;
        if (tid == 0) {
            if (Tr > 0) issue_tile(mp, stage0, bar0, tiles_x, cta, rank, 0, pcur, pprev);
            if (Tr > 1) issue_tile(mp, stage0, bar0, tiles_x, cta, rank + CS, 1, pcur, pprev);
        }
        double beta1 = 0.0, tol_b = 0.0, inv_beta1 = 0.0, invb_prev = 0.0, alpha_prev = 0.0, sigma_prev = 0.0;
        double dbar = 0.0, epsln = 0.0, phibar = 0.0, cs = -1.0, sn = 0.0, s1q = 0.0, s2q = 0.0, Xq = 0.0;
        int k = 0, status = 1;
        for (int pass = 0;; ++pass) {
            double sa = 0.0, sb = 0.0, sc = 0.0;
            double* gnext = base + (size_t)pnext * PLANE;
            for (int u = 0; u < Tr; ++u) {
                const int s = u & 1, t = rank + u * CS;
                mbar_wait(bar0 + 8 * s, (phase >> s) & 1u);
                phase ^= 1u << s;
                const double* Pj = stage0 + s * STAGE;
                const double* Pp = Pj + BOX;
                const double* CE = Pj + 2 * BOX;
                const double* CN = Pj + 3 * BOX;
                const int x0 = 1 + (t % tiles_x) * TW, y0 = 1 + (t / tiles_x) * TH;
                // p_{j+1} on the tile + 1-node halo (box coordinates bx = x + 1, by = y + 1)
                for (int q = tid; q < PW * PH; q += ST) {
                    const int x = q % PW, y = q / PW, bx = x + 1, by = y + 1, c = by * BW + bx;
                    const int gi = x0 - 1 + x, gj = y0 - 1 + y;
                    double pn = 0.0;
                    if (gi >= 1 && gi <= C && gj >= 1 && gj <= C) {
                        const double ce = CE[c], cw = CE[c - 1], cn = CN[c], cs2 = CN[c - BW];
                        const double d = (ce + cw) + (cn + cs2);
                        double tv = d * Pj[c];
                        tv = fma(-ce, Pj[c + 1], tv);
                        tv = fma(-cw, Pj[c - 1], tv);
                        tv = fma(-cn, Pj[c + BW], tv);
                        tv = fma(-cs2, Pj[c - BW], tv);
                        pn = fma(ct, tv, fma(c1, Pj[c], c0 * Pp[c]));
                    }
                    PN[q] = pn;
                }
                __syncthreads();
                // t_{j+1} = A p_{j+1} on the tile, partial sums, store p_{j+1}
                for (int q = tid; q < TW * TH; q += ST) {
                    const int x = q % TW, y = q / TW;
                    const int gi = x0 + x, gj = y0 + y;
                    if (gi > C || gj > C) continue;
                    const int c = (y + 2) * BW + (x + 2), pc = (y + 1) * PW + (x + 1);
                    const double ce = CE[c], cw = CE[c - 1], cn = CN[c], cs2 = CN[c - BW];
                    const double d = (ce + cw) + (cn + cs2);
                    const double pv = PN[pc];
                    double tv = d * pv;
                    tv = fma(-ce, PN[pc + 1], tv);
                    tv = fma(-cw, PN[pc - 1], tv);
                    tv = fma(-cn, PN[pc + PW], tv);
                    tv = fma(-cs2, PN[pc - PW], tv);
                    sa = fma(pv, tv, sa);
                    sb = fma(pv, pv, sb);
                    sc += pv;
                    gnext[(size_t)gj * GP + gi + 1] = pv;
                }
                __syncthreads();                        // stage s and PN are free
                if (tid == 0 && u + 2 < Tr) issue_tile(mp, stage0, bar0, tiles_x, cta, t + 2 * CS, s, pcur, pprev);
            }
            double3 S = bsum3(sa, sb, sc, red);
            if constexpr (CS > 1) {
                // cluster sum in rank order; the barrier also publishes this pass's p_{j+1} stores
                auto cl = cg::this_cluster();
                asm volatile("fence.proxy.async.global;" ::: "memory");
                double* mine = part + 4 * (k & 1);
                if (tid == 0) { mine[0] = S.x; mine[1] = S.y; mine[2] = S.z; }
                cl.sync();
                double3 T3 = make_double3(0.0, 0.0, 0.0);
#pragma unroll
                for (int r = 0; r < CS; ++r) {
                    const double* pr = cl.map_shared_rank(mine, r);
                    T3.x += pr[0];
                    T3.y += pr[1];
                    T3.z += pr[2];
                }
                S = T3;
            }
            // ---- scalars of Lanczos step j+1 (p_{j+1} = the vector just formed), as in the tile kernel
            const double bb = S.y;
            const double invb = bb > 0.0 ? rsqrt(bb) : 0.0;
            const double beta = __dmul_rn(bb, invb);
            const double alpha = __dmul_rn(S.x, __dmul_rn(invb, invb));
            const double sigma = __dmul_rn(S.z, invb);
            if (k > 0) {
                const double oldeps = epsln;
                const double delta = __fma_rn(cs, dbar, __dmul_rn(sn, alpha_prev));
                const double gbar = __fma_rn(sn, dbar, -__dmul_rn(cs, alpha_prev));
                epsln = __dmul_rn(sn, beta);
                dbar = -__dmul_rn(cs, beta);
                const double gg = __fma_rn(gbar, gbar, bb);
                const double invg = gg > 0.0 ? rsqrt(gg) : 1.0 / DBL_MIN;
                cs = __dmul_rn(gbar, invg);
                sn = __dmul_rn(beta, invg);
                const double phi = __dmul_rn(cs, phibar);
                phibar = __dmul_rn(sn, phibar);
                const double sq = __dmul_rn(__fma_rn(-delta, s1q, __fma_rn(-oldeps, s2q, sigma_prev)), invg);
                s2q = s1q;
                s1q = sq;
                Xq = __fma_rn(phi, sq, Xq);
            } else {
                beta1 = beta;
                inv_beta1 = invb;
                tol_b = tol * beta1;
                phibar = beta1;
            }
            bool done = false;
            if (k == 0) {
                if (beta1 == 0.0) { status = 0; done = true; }
            } else {
                if (!(phibar == phibar) || !(beta == beta)) { status = 3; done = true; }
                else if (phibar <= tol_b) { status = 0; done = true; }
                else if (k >= max_iter) done = true;
            }
            if (done) break;
            // next pass: p_{j+2} = t/beta - (alpha/beta) p_{j+1} - (beta/beta_prev) p_j
            ct = invb;
            c1 = -alpha * invb;
            c0 = k == 0 ? 0.0 : -beta * invb_prev;
            invb_prev = invb;
            alpha_prev = alpha;
            sigma_prev = sigma;
            ++k;
            const int old = pprev;
            pprev = pcur;
            pcur = pnext;
            pnext = old;
            if constexpr (CS == 1) {
                asm volatile("fence.proxy.async.global;" ::: "memory");    // this pass's stores -> next TMA reads
                __syncthreads();
            }
            if (tid == 0) {
                if (Tr > 0) issue_tile(mp, stage0, bar0, tiles_x, cta, rank, 0, pcur, pprev);
                if (Tr > 1) issue_tile(mp, stage0, bar0, tiles_x, cta, rank + CS, 1, pcur, pprev);
            }
        }
        if (tid == 0 && rank == 0) {
            double* o = out + (size_t)sj * kRecLen;
            o[0 + slot] = h2 * Xq;
            o[2 + slot] = (double)k;
            o[4 + slot] = phibar * inv_beta1;
            o[6 + slot] = (double)status;
        }
        __syncthreads();
    }
    if constexpr (CS > 1) cg::this_cluster().sync();   // no CTA leaves while another may read its shared memory
}

// ---- tensor map over the scratch: [slot][plane][row][col] binary64, boxes of BW x BH x 1 x 1
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

}  // namespace

bool encode_tensor_map(void* map, bool f64, int rank, void* base, const uint64_t* dims, const uint64_t* strides,
                       const uint32_t* box) {
    auto enc = encode_fn();
    if (!enc || rank < 1 || rank > 5) return false;
    cuuint64_t d[5], st[4];
    cuuint32_t b[5], e[5];
    for (int k = 0; k < rank; ++k) { d[k] = dims[k]; b[k] = box[k]; e[k] = 1; }
    for (int k = 0; k + 1 < rank; ++k) st[k] = strides[k];
    return enc(static_cast<CUtensorMap*>(map), f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
               (cuuint32_t)rank, base, d, st, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool minres_stream_supported(int N) { return N == 128 || N == 256 || N == 512; }

size_t minres_stream_scratch_per_cta(int N) { return sizeof(double) * NPLANE * (size_t)(N + 1) * pitch(N); }

namespace {
template <int CS>
cudaError_t run_stream(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                       unsigned* ctr, double* scratch, int nctas, const int* order, cudaStream_t s) {
    auto kern = minres_stream_kernel<CS>;
    // per device: the smem attribute is set per device and the cluster occupancy is queried there
    static PerDevice<int> mc_cache;
    cudaError_t de = cudaSuccess;
    const int max_clusters = mc_cache.get([&]() -> int {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
        if (e != cudaSuccess) return -(int)e;
        if (CS == 1) return 1 << 30;
        cudaLaunchConfig_t qc = {};
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = CS;
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        qc.gridDim = dim3(CS * 16);
        qc.blockDim = dim3(ST);
        qc.dynamicSmemBytes = SMEM;
        qc.attrs = qa;
        qc.numAttrs = 1;
        int mcl = 0;
        e = cudaOccupancyMaxActiveClusters(&mcl, kern, &qc);
        if (e != cudaSuccess) return -(int)e;
        return mcl < 1 ? -(int)cudaErrorInvalidConfiguration : mcl;
    }, &de);
    if (de != cudaSuccess) return de;
    if (max_clusters < 0) return (cudaError_t)(-max_clusters);
    const int systems = (int)std::min<uint64_t>(std::min<uint64_t>(nb, (uint64_t)nctas), (uint64_t)max_clusters);
    if (systems <= 0) return cudaSuccess;
    CUtensorMap map;
    const uint64_t dims[4] = {(uint64_t)pitch(N), (uint64_t)(N + 1), (uint64_t)NPLANE, (uint64_t)systems};
    const uint64_t strides[3] = {(uint64_t)pitch(N) * 8, (uint64_t)pitch(N) * (N + 1) * 8,
                                 (uint64_t)pitch(N) * (N + 1) * 8 * NPLANE};
    const uint32_t box[4] = {BW, BH, 1, 1};
    if (!encode_tensor_map(&map, true, 4, scratch, dims, strides, box)) return cudaErrorInvalidValue;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    cfg.gridDim = dim3(systems * CS);
    cfg.blockDim = dim3(ST);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = s;
    if (CS > 1) {
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    return cudaLaunchKernelEx(&cfg, kern, map, N, a, (int)nb, tol, max_iter, out, slot, ctr, scratch, order);
}
}  // namespace

// CTAs per system: MLMC_STREAM_CLUSTER=1|2|4|8 overrides; by default 2 on every streamed mesh -- fixed
// per mesh, so that a sample's result does not depend on the batch it is drawn in (the cluster size
// fixes the partial-sum order).  Measured on configs[4] (tools/k3c_cluster.py, tools/gpu_k3c_cs2.sh):
// 100 systems at h = 1/512 8.61 / 4.67 / 3.62 / 3.75 s at 1 / 2 / 4 / 8 CTAs, at h = 1/256 821 / 456 /
// 385 / 486 ms, at h = 1/128 78 / 47 / 48 / 75 ms; 148 equal-length systems (bench.py k3c_fine_meshes)
// 0.80 / 0.76 of HBM at h = 1/256 and 0.78 / 0.78 at 1/512 for 1 / 2 CTAs, but 0.57 / 0.63 for 4 (clusters
// of 4 leave SMs of every GPC idle); 441 systems at h = 1/128: 122 / 135 ms for 1 / 2.
int minres_stream_cluster(int N) {
#ifndef MLMC_TUNING
    (void)N;
    return 2;          // production build: 2-CTA clusters on every streamed mesh
#endif
    static int env = -2;
    if (env == -2) {
        const char* e = std::getenv("MLMC_STREAM_CLUSTER");
        env = e ? std::atoi(e) : -1;
    }
    (void)N;
    if (env == 1 || env == 2 || env == 4 || env == 8) return env;
    return 2;
}

cudaError_t launch_minres_stream(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                                 unsigned* ctr, double* scratch, int nctas, cudaStream_t s, const int* order) {
    if (nb == 0) return cudaSuccess;
    if (!minres_stream_supported(N)) return cudaErrorNotSupported;
#ifdef MLMC_TUNING
    switch (minres_stream_cluster(N)) {
        case 8: return run_stream<8>(N, a, nb, tol, max_iter, out, slot, ctr, scratch, nctas, order, s);
        case 4: return run_stream<4>(N, a, nb, tol, max_iter, out, slot, ctr, scratch, nctas, order, s);
        case 2: return run_stream<2>(N, a, nb, tol, max_iter, out, slot, ctr, scratch, nctas, order, s);
        default: return run_stream<1>(N, a, nb, tol, max_iter, out, slot, ctr, scratch, nctas, order, s);
    }
#else
    return run_stream<2>(N, a, nb, tol, max_iter, out, slot, ctr, scratch, nctas, order, s);
#endif
}

}  // namespace mlmc
