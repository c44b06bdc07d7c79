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
// The matrix is the 5-point P1 operator (R10).  In natural ordering its band
// width is bw = N - 1 and the factor fills the band: W = N entries per row and
// per column of L.  The system is padded to n_pad = N(N-1) = (N-1) W rows with
// identity rows (zero right-hand side) so that every loop runs over whole
// blocks of W rows.
//
// B200 mapping (K4): two kernels per batch pass.
//  K4a chol_factor_kernel -- one W-lane warp segment per sample (32/W samples
//    per warp).  Right-looking factorisation with the W-row band window in
//    registers: lane l owns the window row r = l (mod W) and keeps A(r, c) in
//    register c mod W, so step k addresses registers with the compile-time
//    index k mod W (k unrolled by W).  Step k: pivot by one shuffle (its update
//    comes off the shared-memory round trip: lane k+1 squares its own entry),
//    sqrt and reciprocal in u_f, column scaled by the reciprocal (R29), column
//    through shared memory into the rank-1 update (W-1 FMAs per lane in u_f; the
//    pivot lane then reloads its window row with row k+W).  The factor leaves
//    in two lane-major layouts, one per substitution direction, W entries per
//    lane and block plus the reciprocal pivots in u_s (R28):
//      LF[b][l][u] = L(r_l(u), bW+u)   r_l(u) = the row = l (mod W) lane l
//                                     holds at forward step u
//      LB[b][l][u] = L(bW+u, c_l(u))   c_l(u) = the column = l (mod W) lane l
//                                     holds at backward step u
//    LB is assembled in shared-memory tiles (scattered per step, copied out per
//    block).  The factor format u_f sets the bytes: the paper's memory-
//    reference argument is literal here -- fp16 halves the factor.
//  K4b chol_refine_kernel -- persistent, one segment per sample (job counter).
//    Every substitution streams the sample's factor blocks back from HBM into
//    an NS-slot shared-memory ring with TMA bulk copies (cp.async.bulk,
//    mbarrier completion).  Column-oriented substitutions with rotating
//    ownership: lane l holds the pending right-hand-side entry of its window
//    row; per row one shuffle, one FMA, one multiply on the chain, all in u_s.
//    Residual (binary64, conductances rebuilt from the triangle coefficients)
//    and x (binary64, a per-segment global scratch, L1/L2 resident).
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cfloat>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "internal.h"

namespace mlmc {
namespace {

template <typename T> struct FT;
template <> struct FT<double> {
    static __device__ __forceinline__ double from(double v) { return v; }
    static __device__ __forceinline__ double fnma(double a, double b, double c) { return fma(-a, b, c); }
    static __device__ __forceinline__ double sqrt_(double a) { return sqrt(a); }
    static __device__ __forceinline__ bool pos_finite(double a) { return a > 0.0 && a <= DBL_MAX; }
    static __device__ __forceinline__ float to_f(double v) { return (float)v; }
    static __device__ __forceinline__ double to_d(double v) { return v; }
    static __device__ __forceinline__ double rcp(double v) { return __drcp_rn(v); }
    static __device__ __forceinline__ double scale(double a, double inv) { return __dmul_rn(a, inv); }
};
template <> struct FT<float> {
    static __device__ __forceinline__ float from(double v) { return __double2float_rn(v); }
    static __device__ __forceinline__ float fnma(float a, float b, float c) { return __fmaf_rn(-a, b, c); }
    static __device__ __forceinline__ float sqrt_(float a) { return __fsqrt_rn(a); }
    static __device__ __forceinline__ bool pos_finite(float a) { return a > 0.0f && a <= FLT_MAX; }
    static __device__ __forceinline__ float to_f(float v) { return v; }
    static __device__ __forceinline__ double to_d(float v) { return (double)v; }
    static __device__ __forceinline__ float rcp(float v) { return __frcp_rn(v); }
    static __device__ __forceinline__ float scale(float a, float inv) { return __fmul_rn(a, inv); }
};
template <> struct FT<__half> {
    static __device__ __forceinline__ __half from(double v) { return __double2half(v); }
    static __device__ __forceinline__ __half fnma(__half a, __half b, __half c) { return __hfma(__hneg(a), b, c); }
    static __device__ __forceinline__ __half sqrt_(__half a) { return __float2half_rn(__fsqrt_rn(__half2float(a))); }
    static __device__ __forceinline__ bool pos_finite(__half a) {
        const float f = __half2float(a);
        return f > 0.0f && f <= 65504.0f;
    }
    static __device__ __forceinline__ float to_f(__half v) { return __half2float(v); }
    static __device__ __forceinline__ double to_d(__half v) { return (double)__half2float(v); }
    static __device__ __forceinline__ float rcp(__half v) { return __frcp_rn(__half2float(v)); }
    static __device__ __forceinline__ __half scale(__half a, float inv) { return __float2half_rn(__half2float(a) * inv); }
};
// quarter precision (NEXT-2, the paper's q43 of P:86 / R17): OCP E4M3 storage, every operation computed
// in binary32 and rounded once to E4M3 (round to nearest even, saturating at +-448: the hardware format;
// the SPEC's q43 saturates at 240 -- same grid below it)
using fp8 = __nv_fp8_e4m3;
template <> struct FT<fp8> {
    static __device__ __forceinline__ float f(fp8 v) { return (float)v; }
    static __device__ __forceinline__ fp8 from(double v) { return fp8((float)v); }
    static __device__ __forceinline__ fp8 fnma(fp8 a, fp8 b, fp8 c) { return fp8(__fmaf_rn(-f(a), f(b), f(c))); }
    static __device__ __forceinline__ fp8 sqrt_(fp8 a) { return fp8(__fsqrt_rn(f(a))); }
    static __device__ __forceinline__ bool pos_finite(fp8 a) {
        const float x = f(a);
        return x > 0.0f && x < 448.0f;                 // 448 = saturated
    }
    static __device__ __forceinline__ float to_f(fp8 v) { return f(v); }
    static __device__ __forceinline__ double to_d(fp8 v) { return (double)f(v); }
    static __device__ __forceinline__ float rcp(fp8 v) { return __frcp_rn(f(v)); }
    static __device__ __forceinline__ fp8 scale(fp8 a, float inv) { return fp8(f(a) * inv); }
};
// type of the reciprocal pivot used to scale a column: max(F, binary32)
template <typename F> struct Inv { using T = F; };
template <> struct Inv<__half> { using T = float; };
template <> struct Inv<fp8> { using T = float; };

// shuffle of a factor-format value (E4M3 through its byte)
template <typename F>
__device__ __forceinline__ F shfl_f(unsigned mask, F v, int src, int w) {
    if constexpr (std::is_same_v<F, fp8>) {
        fp8 r;
        r.__x = (__nv_fp8_storage_t)__shfl_sync(mask, (unsigned)v.__x, src, w);
        return r;
    } else {
        return __shfl_sync(mask, v, src, w);
    }
}

// correctly rounded reciprocal in the substitution precision (R28); binary16 via binary32 (u_s = u_f
// is selectable for fidelity, R24)
__device__ __forceinline__ float rcp_s(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double rcp_s(double x) { return __drcp_rn(x); }
__device__ __forceinline__ __half rcp_s(__half x) { return __float2half_rn(__frcp_rn(__half2float(x))); }
// factor entry -> substitution precision S
template <typename S, typename F> __device__ __forceinline__ S to_s(F v) {
    if constexpr (sizeof(S) == 8) return FT<F>::to_d(v);
    else if constexpr (sizeof(S) == 4) return FT<F>::to_f(v);
    else return __float2half_rn(FT<F>::to_f(v));
}
// a substitution-precision value, exactly, in binary64 (d is rounded once, straight to u: Algorithm 1 step 8,
// a binary32 detour dropped the bits of binary64 corrections)
__device__ __forceinline__ double s_to_d(double v) { return v; }
__device__ __forceinline__ double s_to_d(float v) { return (double)v; }
__device__ __forceinline__ double s_to_d(__half v) { return (double)__half2float(v); }
// -a * b + c in S with one rounding
__device__ __forceinline__ float sfnma(float a, float b, float c) { return fmaf(-a, b, c); }
__device__ __forceinline__ double sfnma(double a, double b, double c) { return fma(-a, b, c); }
__device__ __forceinline__ __half sfnma(__half a, __half b, __half c) { return __hfma(__hneg(a), b, c); }

// if (l == u) { cur = nxt; y = yk; } as one setp + two predicated moves, kept in place (volatile) so
// the compiler does not materialise all W lane predicates of an unrolled block up front
__device__ __forceinline__ void pivot_take(int l, int u, float& cur, float nxt, float& y, float yk) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %2, %3;\n\t@p mov.f32 %0, %4;\n\t@p mov.f32 %1, %5;\n}"
                 : "+f"(cur), "+f"(y)
                 : "r"(l), "r"(u), "f"(nxt), "f"(yk));
}
__device__ __forceinline__ void pivot_take(int l, int u, double& cur, double nxt, double& y, double yk) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %2, %3;\n\t@p mov.f64 %0, %4;\n\t@p mov.f64 %1, %5;\n}"
                 : "+d"(cur), "+d"(y)
                 : "r"(l), "r"(u), "d"(nxt), "d"(yk));
}
__device__ __forceinline__ void pivot_take(int l, int u, __half& cur, __half nxt, __half& y, __half yk) {
    unsigned short c = __half_as_ushort(cur), yy = __half_as_ushort(y);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %2, %3;\n\t@p mov.b16 %0, %4;\n\t@p mov.b16 %1, %5;\n}"
                 : "+h"(c), "+h"(yy)
                 : "r"(l), "r"(u), "h"(__half_as_ushort(nxt)), "h"(__half_as_ushort(yk)));
    cur = __ushort_as_half(c);
    y = __ushort_as_half(yy);
}

// ---- geometry of one mesh / format pair
template <int N, typename F, typename S>
struct Geo {
    static constexpr int W = N;                        // band entries per row / column, segment width
    static constexpr int n = (N - 1) * (N - 1);
    static constexpr int NB = N - 1;                   // blocks of W rows / columns
    static constexpr int NPAD = NB * W;                // padded system size N(N-1) >= n
    static constexpr int SEGS = 32 / W;                // samples per warp
    static constexpr int FE = W * (int)sizeof(F);      // bytes of one lane row of a block
    static constexpr int C = FE / 16;                  // 16-byte chunks per lane row (0: scalar access)
    static constexpr int EPC = 16 / (int)sizeof(F);    // entries per chunk
    static constexpr int LPR = C >= 8 ? 1 : (C > 0 ? 8 / C : 1);   // lane rows per 128-byte bank row
    static constexpr int HDR = W * FE;                 // reciprocal pivots (S) after the W lane rows
    static constexpr int BLK = ((HDR + W * (int)sizeof(S) + 127) / 128) * 128;   // block stride (bytes)
    static constexpr size_t FBYTES = (size_t)2 * NB * BLK;   // LF + LB of one sample
    static_assert(W >= 2 && W <= 32 && (W & (W - 1)) == 0, "segment width must be a power of two <= 32");
    // byte offset of entry e of lane row r inside a block: 16-byte chunks rotated per lane row so that
    // a quarter-warp reading chunk i of 8 consecutive lane rows hits 8 distinct bank groups
    static __device__ __forceinline__ int off(int r, int e) {
        if constexpr (C == 0) return r * FE + e * (int)sizeof(F);
        else return r * FE + (((e / EPC) + r / LPR) % C) * 16 + (e % EPC) * (int)sizeof(F);
    }
};

// lane row r of a block (shared memory) -> W values in precision S
template <class G, typename F, typename S>
__device__ __forceinline__ void load_row(const unsigned char* blk, int r, S (&lv)[G::W]) {
    if constexpr (G::C == 0) {
#pragma unroll
        for (int e = 0; e < G::W; ++e) lv[e] = to_s<S>(*reinterpret_cast<const F*>(blk + G::off(r, e)));
    } else {
#pragma unroll
        for (int i = 0; i < G::C; ++i) {
            const uint4 q = *reinterpret_cast<const uint4*>(blk + G::off(r, i * G::EPC));
            F t[G::EPC];
            memcpy(t, &q, 16);
#pragma unroll
            for (int e = 0; e < G::EPC; ++e) lv[i * G::EPC + e] = to_s<S>(t[e]);
        }
    }
}
// W factor values -> lane row r of a block (global)
template <class G, typename F>
__device__ __forceinline__ void store_row(unsigned char* blk, int r, const F (&vals)[G::W]) {
    if constexpr (G::C == 0) {
#pragma unroll
        for (int e = 0; e < G::W; ++e) *reinterpret_cast<F*>(blk + G::off(r, e)) = vals[e];
    } else {
#pragma unroll
        for (int i = 0; i < G::C; ++i) {
            uint4 q;
            memcpy(&q, &vals[i * G::EPC], 16);
            *reinterpret_cast<uint4*>(blk + G::off(r, i * G::EPC)) = q;
        }
    }
}
// raw copy of lane row r (shared -> global), same layout
template <class G, typename F>
__device__ __forceinline__ void copy_row(unsigned char* dst, const unsigned char* src, int r) {
    if constexpr (G::C == 0) {
#pragma unroll
        for (int e = 0; e < G::W; ++e)
            *reinterpret_cast<F*>(dst + G::off(r, e)) = *reinterpret_cast<const F*>(src + G::off(r, e));
    } else {
#pragma unroll
        for (int i = 0; i < G::C; ++i)
            *reinterpret_cast<uint4*>(dst + G::off(r, i * G::EPC)) =
                *reinterpret_cast<const uint4*>(src + G::off(r, i * G::EPC));
    }
}

// Entries of row r of A (interior node (i, j), r = (j-1)(N-1) + (i-1)) from the triangle
// coefficients: cE(i,j) = (aL(i,j) + aU(i,j-1))/2, cN(i,j) = (aU(i,j) + aL(i-1,j))/2 (R10).
template <int N>
struct Coef {
    const double* a;
    __device__ __forceinline__ double aL(int i, int j) const { return __ldg(a + 2 * (j * N + i)); }
    __device__ __forceinline__ double aU(int i, int j) const { return __ldg(a + 2 * (j * N + i) + 1); }
    __device__ __forceinline__ double cE(int i, int j) const { return 0.5 * (aL(i, j) + aU(i, j - 1)); }
    __device__ __forceinline__ double cN(int i, int j) const { return 0.5 * (aU(i, j) + aL(i - 1, j)); }
    // diagonal, west coupling (column r-1) and south coupling (column r-(N-1)) of row r; identity for r >= n
    __device__ __forceinline__ void row(int r, double& dg, double& we, double& so) const {
        constexpr int n = (N - 1) * (N - 1);
        if (r >= n) { dg = 1.0; we = 0.0; so = 0.0; return; }
        const int i = r % (N - 1) + 1, j = r / (N - 1) + 1;
        const double e = cE(i, j), w = cE(i - 1, j), no = cN(i, j), s = cN(i, j - 1);
        dg = (e + w) + (no + s);
        we = i > 1 ? -w : 0.0;
        so = j > 1 ? -s : 0.0;
    }
};

// ======================================================================== K4a: factorisation
constexpr int kFacWarps = 4;
#ifndef FAC_MINB_DEFAULT
#define FAC_MINB_DEFAULT 4
#endif

template <int N, typename F, typename S>
struct FacCfg {
    using G = Geo<N, F, S>;
    // binary64 factors at W = 32 keep neither the finished column entries nor the broadcast column in
    // registers (the window alone is 64 registers): the forward layout goes through a third tile
    static constexpr bool LIGHT = sizeof(F) == 8 && N == 32;
    // shared memory per segment: two LB tiles | [LF tile] | column buffer (2 x W entries)
    static constexpr int OFF_F = 2 * G::BLK;
    static constexpr int OFF_C = (LIGHT ? 3 : 2) * G::BLK;
    static constexpr int SEG_BYTES = ((OFF_C + 2 * G::W * (int)sizeof(F) + 127) / 128) * 128;
    static constexpr int SMEM = SEG_BYTES * G::SEGS * kFacWarps;
    // resident CTAs the register allocation is bounded for (MLMC_CHOL_FAC_MINB overrides for tuning)
    static constexpr int MINB = sizeof(F) == 8 ? 2 : FAC_MINB_DEFAULT;
};

// Factorise samples [0, nb): factor of sample j at fac + j * FBYTES; status (0 ok, 2 breakdown) to
// out[j*8 + 6 + slot].
template <int N, typename F, typename S>
__global__ void __launch_bounds__(32 * kFacWarps, FacCfg<N, F, S>::MINB)
chol_factor_kernel(const double* __restrict__ a_all, int nb, unsigned char* __restrict__ fac,
                   double* __restrict__ out, int slot) {
    using G = Geo<N, F, S>;
    using K = FacCfg<N, F, S>;
    constexpr int W = G::W, NB = G::NB, SEGS = G::SEGS, BLK = G::BLK;
    constexpr int P = 2 * N * N;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(16) uint4 zrow[16];         // 256 zero bytes (re-initialised window rows)
    static_assert(G::C <= 16, "zero row too short");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int seg = lane / W, l = lane % W;
    const unsigned mask = 0xffffffffu;
    if (threadIdx.x < 16) zrow[threadIdx.x] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const int job = (blockIdx.x * kFacWarps + warp) * SEGS + seg;
    const bool live = job < nb;
    unsigned char* base = smem + (size_t)(warp * SEGS + seg) * K::SEG_BYTES;
    F* colbuf = reinterpret_cast<F*>(base + K::OFF_C);
    unsigned char* LF = fac + (size_t)(live ? job : 0) * G::FBYTES;
    unsigned char* LB = LF + (size_t)NB * BLK;
    const Coef<N> A{a_all + (size_t)(live ? job : 0) * P};

    // the tile of block 0 keeps zeros where no column exists (c < 0)
    for (int e = l; e < BLK / 16; e += W) reinterpret_cast<uint4*>(base)[e] = make_uint4(0, 0, 0, 0);
    F Rw[W];
#pragma unroll
    for (int c = 0; c < W; ++c) Rw[c] = FT<F>::from(0.0);
    {
        // row l: diagonal in slot l, west (column l-1) in slot l-1, south (column l-(N-1), only
        // for l = W-1) in slot (l+1) mod W
        double dg, we, so;
        A.row(l, dg, we, so);
#pragma unroll
        for (int u = 0; u < W; ++u) {
            if (u == ((l + 1) & (W - 1))) Rw[u] = FT<F>::from(so);
            if (u == ((l + W - 1) & (W - 1))) Rw[u] = FT<F>::from(we);
            if (u == l) Rw[u] = FT<F>::from(dg);
        }
    }
    __syncwarp(mask);
    bool ok = true;
    F pnext = FT<F>::from(0.0);
    for (int b = 0; b < NB; ++b) {
        const int k0 = b * W;
        unsigned char* Tc = base + (b & 1) * BLK;          // LB tile of block b (rows k0 .. k0+W-1)
        unsigned char* Tn = base + ((b + 1) & 1) * BLK;    // LB tile of block b+1
        // the row each lane takes after its pivot step in this block: k0 + W + l (loads issued early)
        F dgn = FT<F>::from(0.0), wen = FT<F>::from(0.0), son = FT<F>::from(0.0);
        if (b + 1 < NB) {
            double dg, we, so;
            A.row(k0 + W + l, dg, we, so);
            dgn = FT<F>::from(dg);
            wen = FT<F>::from(we);
            son = FT<F>::from(so);
        }
        F lcol[K::LIGHT ? 1 : W];
        unsigned char* TF = base + K::OFF_F;            // LF tile (LIGHT)
        S rdl = (S)0.0;
#pragma unroll
        for (int u = 0; u < W; ++u) {
            const int d = (l - u) & (W - 1);          // this lane holds row k0 + u + d
            // pivot: lane u's diagonal, from the fast path of the previous step (k > 0)
            F piv = shfl_f<F>(mask, (b == 0 && u == 0) ? Rw[0] : pnext, u, W);
            if (!FT<F>::pos_finite(piv)) { ok = false; piv = FT<F>::from(1.0); }
            const F lkk = FT<F>::sqrt_(piv);
            const typename Inv<F>::T inv = FT<F>::rcp(lkk);
            S rk;                                      // 1 / L(k,k) in u_s for the substitutions (R28)
            if constexpr (sizeof(S) == sizeof(inv)) rk = inv;
            else rk = rcp_s(to_s<S>(lkk));
            const F lc = d == 0 ? lkk : FT<F>::scale(Rw[u], inv);   // L(k0+u+d, k0+u)
            // the next pivot's update: lane u+1 squares its own column entry (the same operation the
            // rank-1 update below performs with the shared copy), off the shared-memory round trip
            pnext = FT<F>::fnma(lc, lc, Rw[(u + 1) % W]);
            if constexpr (K::LIGHT) *reinterpret_cast<F*>(TF + G::off(l, u)) = lc;
            else lcol[K::LIGHT ? 0 : u] = lc;
            if (l == u) rdl = rk;
            *reinterpret_cast<F*>((l >= u ? Tc : Tn) + G::off(u, l)) = lc;
            F* cb = colbuf + (u & 1) * W;
            cb[d] = lc;
            __syncwarp(mask);
            if constexpr (K::LIGHT) {
#pragma unroll
                for (int j = 1; j < W; ++j) Rw[(u + j) % W] = FT<F>::fnma(lc, cb[j], Rw[(u + j) % W]);
            } else {
                F cv[W];
                if constexpr (G::C == 0) {
#pragma unroll
                    for (int j = 0; j < W; ++j) cv[j] = cb[j];
                } else {
#pragma unroll
                    for (int i = 0; i < G::C; ++i) {
                        const uint4 q = reinterpret_cast<const uint4*>(cb)[i];
                        memcpy(&cv[i * G::EPC], &q, 16);
                    }
                }
#pragma unroll
                for (int j = 1; j < W; ++j) Rw[(u + j) % W] = FT<F>::fnma(lc, cv[j], Rw[(u + j) % W]);
            }
            if (l == u) {                              // row k0+u is done: this lane takes row k0+u+W
                if constexpr (G::C == 0) {
#pragma unroll
                    for (int c = 0; c < W; ++c) Rw[c] = FT<F>::from(0.0);
                } else {                               // zero the window row with vector loads
#pragma unroll
                    for (int i = 0; i < G::C; ++i) {
                        const uint4 q = zrow[i];
                        memcpy(&Rw[i * G::EPC], &q, 16);
                    }
                }
                Rw[u] = dgn;
                Rw[(u + W - 1) % W] = wen;
                Rw[(u + 1) % W] = son;
            }
        }
        __syncwarp(mask);
        if (live) {
            unsigned char* gF = LF + (size_t)b * BLK;
            unsigned char* gB = LB + (size_t)b * BLK;
            if constexpr (K::LIGHT) copy_row<G, F>(gF, TF, l);
            else store_row<G, F>(gF, l, lcol);
            copy_row<G, F>(gB, Tc, l);
            reinterpret_cast<S*>(gF + G::HDR)[l] = rdl;
            reinterpret_cast<S*>(gB + G::HDR)[l] = rdl;
        }
        __syncwarp(mask);
    }
    if (live && l == 0) out[(size_t)job * kRecLen + 6 + slot] = ok ? 0.0 : 2.0;
}

// ======================================================================== K4b: refinement
// ---- mbarrier / bulk-copy primitives (PTX)
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
// (A slot is refilled only after every lane of the segment has consumed the values it read from it
// and passed a __syncwarp, so no proxy fence is issued per fill.)
// The factor is streamed once per substitution and evicted first from L2, which keeps the small,
// re-read working set (x, the coefficients) resident.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}

// Working / residual precision u = u_r of Algorithm 1 (steps 4 and 8): binary64, binary32, or binary16 with
// every operation computed in binary32 and rounded once to binary16 (as the factor formats, R17).
template <typename U> struct VT {
    static __device__ __forceinline__ U from(double v) { return (U)v; }
    static __device__ __forceinline__ double to_d(U v) { return (double)v; }
    static __device__ __forceinline__ U mul(U a, U b) { return a * b; }
    static __device__ __forceinline__ U fnma(U a, U b, U c) { return fma(-a, b, c); }
    static __device__ __forceinline__ U sub(U a, U b) { return a - b; }
    static __device__ __forceinline__ U add(U a, U b) { return a + b; }
};
template <> struct VT<__half> {
    static __device__ __forceinline__ __half from(double v) { return __double2half(v); }
    static __device__ __forceinline__ double to_d(__half v) { return (double)__half2float(v); }
    static __device__ __forceinline__ __half mul(__half a, __half b) {
        return __float2half_rn(__half2float(a) * __half2float(b));
    }
    static __device__ __forceinline__ __half fnma(__half a, __half b, __half c) {
        return __float2half_rn(fmaf(-__half2float(a), __half2float(b), __half2float(c)));
    }
    static __device__ __forceinline__ __half sub(__half a, __half b) {
        return __float2half_rn(__half2float(a) - __half2float(b));
    }
    static __device__ __forceinline__ __half add(__half a, __half b) {
        return __float2half_rn(__half2float(a) + __half2float(b));
    }
};

template <int N, typename F, typename S, int NS_, int WPC_>
struct RefCfg {
    using G = Geo<N, F, S>;
    static constexpr int NS = NS_;                     // ring slots
    static constexpr int WPC = WPC_;                   // warps per CTA
    // shared memory per segment: ring (NS blocks) | v (u_s) | mbarriers
    static constexpr int OFF_V = NS * G::BLK;
    static constexpr int OFF_B = OFF_V + ((G::NPAD * (int)sizeof(S) + 15) / 16) * 16;
    static constexpr int SEG_BYTES = ((OFF_B + NS * 8 + 127) / 128) * 128;
    static constexpr int SMEM = SEG_BYTES * G::SEGS * WPC;
    static constexpr size_t XBYTES = (size_t)G::NPAD * 8;   // global x scratch per resident segment
};

// FIFO ring of factor blocks for one segment (NS slots).  The blocks are consumed in a fixed
// sequence -- forward pass LF[0..NB-1], backward pass LB[NB-1..0], forward, ... -- so fill
// position p goes to slot p % NS and completes phase (p / NS) & 1 of that slot's mbarrier; the
// producer (the segment's lane 0) keeps NS-1 positions ahead of the consumer.  Counters are
// absolute across jobs (the mbarrier phases are).
template <int NB, int BLK, int NS>
struct Ring {
    unsigned char* buf;     // slot 0 (generic address)
    uint32_t sbuf, bar;     // shared addresses of slot 0 and barrier 0
    const unsigned char* lf;
    const unsigned char* lb;
    unsigned iss, use, pass, j;   // next fill: pass index and block position within the pass
    uint64_t pol;                 // L2 policy of the fills

    __device__ __forceinline__ const unsigned char* acquire(bool leader) {
        __syncwarp();                                   // all lanes are done with position use-1
        while (iss < use + NS) {
            const unsigned char* src = (pass & 1) ? lb + (size_t)(NB - 1 - j) * BLK : lf + (size_t)j * BLK;
            if (leader) bulk_load(sbuf + (iss % NS) * BLK, src, BLK, bar + 8 * (iss % NS), pol);
            ++iss;
            if (++j == NB) { j = 0; ++pass; }
        }
        mbar_wait(bar + 8 * (use % NS), (use / NS) & 1u);
        const unsigned char* p = buf + (use % NS) * BLK;
        ++use;
        return p;
    }
    __device__ __forceinline__ void start(const unsigned char* f_lf, const unsigned char* f_lb) {
        lf = f_lf;
        lb = f_lb;
        pass = 0;
        j = 0;
    }
    __device__ __forceinline__ void drain() {
        while (use < iss) {
            mbar_wait(bar + 8 * (use % NS), (use / NS) & 1u);
            ++use;
        }
        __syncwarp();
    }
};

// Forward substitution L y = v in place (u_s).  LF block b gives lane l the entries L(r_l(u), bW+u)
// of the row it owns at step u and 1/L(bW+l, bW+l).  Per row: a shuffle, an FMA and a multiply on
// the chain; the pivot lane then takes the row W further on.
template <class G, typename F, typename S, class R>
__device__ __forceinline__ void forward(R& ring, S* v, int l, bool leader) {
    constexpr int W = G::W, NB = G::NB;
    S cur = v[l];
    for (int b = 0; b < NB; ++b) {
        const unsigned char* blk = ring.acquire(leader);
        S lv[W];
        load_row<G, F, S>(blk, l, lv);
        const S rd = reinterpret_cast<const S*>(blk + G::HDR)[l];
        const int k0 = b * W;
        const S nxt = b + 1 < NB ? v[k0 + W + l] : (S)0.0;
        S yv = (S)0.0;
        S t = cur * rd;                              // y of this lane's row if it is the next pivot
#pragma unroll
        for (int u = 0; u < W; ++u) {
            const S yk = __shfl_sync(0xffffffffu, t, u, W);
            const S c2 = sfnma(lv[u], yk, cur);
            t = c2 * rd;
            cur = c2;
            pivot_take(l, u, cur, nxt, yv, yk);
        }
        v[k0 + l] = yv;
    }
    __syncwarp();
}

// Backward substitution L^T x = v in place (u_s).  LB block b gives lane l the entries
// L(bW+u, c_l(u)) of row bW+u at the column it owns at step u.
template <class G, typename F, typename S, class R>
__device__ __forceinline__ void backward(R& ring, S* v, int l, bool leader) {
    constexpr int W = G::W, NB = G::NB;
    S cur = v[(NB - 1) * W + l];
    for (int b = NB - 1; b >= 0; --b) {
        const unsigned char* blk = ring.acquire(leader);
        S lv[W];
        load_row<G, F, S>(blk, l, lv);
        const S rd = reinterpret_cast<const S*>(blk + G::HDR)[l];
        const int k0 = b * W;
        const S nxt = b > 0 ? v[k0 - W + l] : (S)0.0;
        S xv = (S)0.0;
        S t = cur * rd;
#pragma unroll
        for (int u = W - 1; u >= 0; --u) {
            const S xk = __shfl_sync(0xffffffffu, t, u, W);
            const S c2 = sfnma(lv[u], xk, cur);
            t = c2 * rd;
            cur = c2;
            pivot_take(l, u, cur, nxt, xv, xk);
        }
        v[k0 + l] = xv;
    }
    __syncwarp();
}

// U: the working precision u = u_r of x and of the residual (Algorithm 1 steps 4 and 8; double or float)
template <int N, typename F, typename S, int NS, int WPC, typename U = double>
__global__ void __launch_bounds__(32 * WPC)
chol_refine_kernel(const double* __restrict__ a_all, int nb, double tol, int i_max, double* __restrict__ out,
                   int slot, unsigned* __restrict__ job_counter, const unsigned char* __restrict__ fac,
                   double* __restrict__ xscratch) {
    using G = Geo<N, F, S>;
    using K = RefCfg<N, F, S, NS, WPC>;
    constexpr int W = G::W, n = G::n, NB = G::NB, NPAD = G::NPAD, SEGS = G::SEGS, BLK = G::BLK;
    constexpr int P = 2 * N * N, PER = NPAD / W;     // vector entries per lane (= NB)
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int seg = lane / W, l = lane % W;
    const unsigned mask = 0xffffffffu;
    const bool leader = l == 0;
    unsigned char* base = smem + (size_t)(warp * SEGS + seg) * K::SEG_BYTES;
    S* v = reinterpret_cast<S*>(base + K::OFF_V);
    U* xs = reinterpret_cast<U*>(xscratch + (((size_t)blockIdx.x * WPC + warp) * SEGS + seg) * NPAD);
    Ring<NB, BLK, NS> ring;
    ring.buf = base;
    ring.sbuf = smem_u32(base);
    ring.bar = smem_u32(base + K::OFF_B);
    ring.iss = ring.use = 0;
    ring.pol = policy_evict_first();
    if (leader) {
#pragma unroll
        for (int q = 0; q < NS; ++q) mbar_init(ring.bar + 8 * q);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const double h = 1.0 / N, h2 = h * h;
    const double bnorm = h2 * sqrt((double)n);

    for (;;) {
        int jb = 0;
        if (lane == 0) jb = (int)atomicAdd(job_counter, (unsigned)SEGS);
        jb = __shfl_sync(mask, jb, 0);
        if (jb >= nb) break;
        const int job = jb + seg;
        const bool live = job < nb;
        const int jj = live ? job : nb - 1;
        const Coef<N> A{a_all + (size_t)jj * P};
        const unsigned char* LF = fac + (size_t)jj * G::FBYTES;
        ring.start(LF, LF + (size_t)NB * BLK);
        double* orec = out + (size_t)jj * kRecLen;
        const bool ok = orec[6 + slot] == 0.0;        // factorisation status from K4a
        bool active = live && ok;
        int status = ok ? 1 : 2, it = -1;
        double rel = 1.0;
#pragma unroll 4
        for (int q = 0; q < PER; ++q) {
            const int e = l + q * W;
            v[e] = e < n ? (S)h2 : (S)0.0;             // b in u_s
        }
        __syncwarp(mask);
        // it = -1: step 2, x0 = (L L^T)^-1 b;  it >= 0: steps 4-8
        for (;;) {
            if (it >= 0) {
                // ---- step 4: r = b - A x in binary64 (rounded to u_s for the correction solve)
                double part = 0.0;
                if (active) {
#pragma unroll 4
                    for (int q = 0; q < PER; ++q) {
                        const int e = l + q * W;
                        using V = VT<U>;
                        U r = V::from(0.0);
                        if (e < n) {
                            const int i = e % (N - 1) + 1, j = e / (N - 1) + 1;
                            const double ce = A.cE(i, j), cw = A.cE(i - 1, j), cn = A.cN(i, j), cs = A.cN(i, j - 1);
                            // the matrix entries in u_r, every product and sum in u_r (fused where the
                            // hardware fuses: one rounding per FMA)
                            const U ue = V::from(ce), uw = V::from(cw), un = V::from(cn), us = V::from(cs),
                                    ud = V::from((ce + cw) + (cn + cs));
                            U Ax = V::mul(ud, xs[e]);
                            if (i < N - 1) Ax = V::fnma(ue, xs[e + 1], Ax);
                            if (i > 1) Ax = V::fnma(uw, xs[e - 1], Ax);
                            if (j < N - 1) Ax = V::fnma(un, xs[e + N - 1], Ax);
                            if (j > 1) Ax = V::fnma(us, xs[e - (N - 1)], Ax);
                            r = V::sub(V::from(h2), Ax);
                            const double rd = V::to_d(r);
                            part = fma(rd, rd, part);
                        }
                        v[e] = (S)V::to_d(r);
                    }
                }
#pragma unroll
                for (int o = W / 2; o > 0; o >>= 1) part += __shfl_xor_sync(mask, part, o, W);
                if (active) {
                    rel = sqrt(part) / bnorm;
                    if (!(rel == rel) || rel > DBL_MAX) { status = 3; active = false; }
                    else if (rel < tol) { status = 0; active = false; }        // step 5
                    else if (it == i_max) { active = false; }
                }
                if (!__any_sync(mask, active)) break;
                __syncwarp(mask);
            }
            // ---- steps 2 / 7: (L L^T)^-1 v in u_s;  step 8: x += d in binary64
            forward<G, F, S>(ring, v, l, leader);
            backward<G, F, S>(ring, v, l, leader);
            if (it < 0) {
#pragma unroll 4
                for (int q = 0; q < PER; ++q) xs[l + q * W] = VT<U>::from(s_to_d(v[l + q * W]));
            } else if (active) {                       // step 8: x += d in u (d rounded to u first)
#pragma unroll 4
                for (int q = 0; q < PER; ++q)
                    xs[l + q * W] = VT<U>::add(xs[l + q * W], VT<U>::from(s_to_d(v[l + q * W])));
            }
            if (it < 0 || active) ++it;
            __syncwarp(mask);
        }
        ring.drain();
        double sx = 0.0;
        for (int q = 0; q < PER; ++q) sx += VT<U>::to_d(xs[l + q * W]);   // padded rows hold exact zeros
#pragma unroll
        for (int o = W / 2; o > 0; o >>= 1) sx += __shfl_xor_sync(mask, sx, o, W);
        if (live && leader) {
            orec[0 + slot] = status == 2 ? 0.0 : h2 * sx;
            orec[2 + slot] = (double)(it < 0 ? 0 : it);
            orec[4 + slot] = rel;
            orec[6 + slot] = (double)status;
        }
        __syncwarp(mask);
    }
}

// ======================================================================== launch
template <int N, typename F, typename S, int NS = 3, int WPC = 4, typename U = double>
struct Launch {
    using G = Geo<N, F, S>;
    using KF = FacCfg<N, F, S>;
    using KR = RefCfg<N, F, S, NS, WPC>;
    static cudaError_t setup(int& grid_max) {
        static PerDevice<KernelOcc> cache;                 // the smem attributes are per device
        cudaError_t de = cudaSuccess;
        KernelOcc occ = cache.get([] {
            KernelOcc o;
            o.err = cudaFuncSetAttribute(chol_factor_kernel<N, F, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         KF::SMEM);
            return o.err == cudaSuccess ? kernel_occ(chol_refine_kernel<N, F, S, NS, WPC, U>, 32 * WPC, KR::SMEM) : o;
        }, &de);
        if (de != cudaSuccess) occ.err = de;
        if (occ.err != cudaSuccess) return occ.err;
        grid_max = occ.per_sm * occ.sms;
        return cudaSuccess;
    }
    static constexpr uint64_t per_cta = (uint64_t)WPC * G::SEGS;
    static size_t fac_bytes(uint64_t nb) { return (nb * G::FBYTES + 255) & ~(size_t)255; }
    // scratch of a launch over nb systems: every factor (LF + LB) + x of every resident refine segment
    static cudaError_t scratch(size_t& bytes, uint64_t nb) {
        int gm = 0;
        cudaError_t e = setup(gm);
        const uint64_t grid = std::min<uint64_t>((nb + per_cta - 1) / per_cta, (uint64_t)gm);
        bytes = fac_bytes(nb) + (size_t)grid * per_cta * KR::XBYTES;
        return e;
    }
    static cudaError_t run(const double* a, uint64_t nb, double tol, int i_max, double* out, int slot, unsigned* ctr,
                           void* scr, size_t bytes, cudaStream_t s) {
        if (nb == 0) return cudaSuccess;
        int gm = 0;
        cudaError_t e = setup(gm);
        if (e != cudaSuccess) return e;
        size_t need = 0;
        scratch(need, nb);
        if (need > bytes) return cudaErrorInvalidValue;
        unsigned char* fac = static_cast<unsigned char*>(scr);
        double* xs = reinterpret_cast<double*>(fac + fac_bytes(nb));
        const uint64_t fgrid = (nb + kFacWarps * G::SEGS - 1) / (kFacWarps * G::SEGS);
        chol_factor_kernel<N, F, S><<<(unsigned)fgrid, 32 * kFacWarps, KF::SMEM, s>>>(a, (int)nb, fac, out, slot);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        const uint64_t grid = std::min<uint64_t>((nb + per_cta - 1) / per_cta, (uint64_t)gm);
        chol_refine_kernel<N, F, S, NS, WPC, U><<<(unsigned)grid, 32 * WPC, KR::SMEM, s>>>(a, (int)nb, tol, i_max,
                                                                                        out, slot, ctr, fac, xs);
        return cudaGetLastError();
    }
};

#ifdef MLMC_TUNING
constexpr bool kTuning = true;
#else
constexpr bool kTuning = false;
#endif
// Ring depth / CTA shape of the refinement kernel for the h = 1/32 factors (MLMC_CHOL_VARIANT
// selects for tuning runs).
int chol_variant() {
#ifndef MLMC_TUNING
    return 0;
#else
    static int v = -2;
    if (v == -2) {
        const char* e = std::getenv("MLMC_CHOL_VARIANT");
        v = e ? std::atoi(e) : 0;
    }
    return v;
#endif
}

template <int N, typename F, typename S, typename U, class Fn>
cudaError_t with_shape_u(Fn&& fn) {
    if constexpr (N == 32 && sizeof(S) == 4) {
        if constexpr (sizeof(U) == 8 && kTuning) {
            switch (chol_variant()) {
                // measured (configs[2] level 2, 100k coupled samples, fp16 / fp32 factor): <3,4> 72.5 / 42.4 ms,
                // <4,4> 78.6 / 47.5, <2,4> 69.6 / 41.4, <2,2> 68.9 / 41.4, <3,8> 77.5 / 46.7
                case 1: return fn(Launch<N, F, S, 4, 4, U>{});
                case 2: return fn(Launch<N, F, S, 2, 4, U>{});
                case 3: return fn(Launch<N, F, S, 3, 4, U>{});
                case 4: return fn(Launch<N, F, S, 3, 8, U>{});
                default: break;
            }
        }
        return fn(Launch<N, F, S, 2, 2, U>{});
    } else {
        return fn(Launch<N, F, S, 3, 4, U>{});
    }
}

// u = u_r: binary64 (the default), binary32 or binary16 (the paper's "..ss" / "..hh" quads, Table 1 right,
// P:596-607)
template <int N, typename F, typename S, class Fn>
cudaError_t with_shape(int vfmt, Fn&& fn) {
    if (vfmt == MLMC_FMT_F32) return with_shape_u<N, F, S, float>(fn);
    if (vfmt == MLMC_FMT_F16) return with_shape_u<N, F, S, __half>(fn);
    if constexpr (sizeof(S) == 2) return cudaErrorNotSupported;   // binary16 substitutions: u, u_r <= s
    else return with_shape_u<N, F, S, double>(fn);
}

// (u_f, u_s) -> instantiation; returns cudaErrorNotSupported for combinations not built.
template <int N, class Fn>
cudaError_t with_types(int u_f, int u_s, int vfmt, Fn&& fn) {
    if (u_f == MLMC_FMT_E4M3) {
        if (u_s == MLMC_FMT_F16) return with_shape<N, fp8, __half>(vfmt, fn);
        if (u_s == MLMC_FMT_F32) return with_shape<N, fp8, float>(vfmt, fn);
        if (u_s == MLMC_FMT_F64) return with_shape<N, fp8, double>(vfmt, fn);
    } else if (u_f == MLMC_FMT_F16) {
        if (u_s == MLMC_FMT_F16) return with_shape<N, __half, __half>(vfmt, fn);
        if (u_s == MLMC_FMT_F32) return with_shape<N, __half, float>(vfmt, fn);
        if (u_s == MLMC_FMT_F64) return with_shape<N, __half, double>(vfmt, fn);
    } else if (u_f == MLMC_FMT_F32) {
        if (u_s == MLMC_FMT_F32) return with_shape<N, float, float>(vfmt, fn);
        if (u_s == MLMC_FMT_F64) return with_shape<N, float, double>(vfmt, fn);
    } else if (u_f == MLMC_FMT_F64) {
        if (u_s == MLMC_FMT_F32) return with_shape<N, double, float>(vfmt, fn);
        if (u_s == MLMC_FMT_F64) return with_shape<N, double, double>(vfmt, fn);
    }
    return cudaErrorNotSupported;
}

template <class Fn>
cudaError_t with_mesh(int N, int u_f, int u_s, int vfmt, Fn&& fn) {
    switch (N) {
        case 2: return with_types<2>(u_f, u_s, vfmt, fn);
        case 4: return with_types<4>(u_f, u_s, vfmt, fn);
        case 8: return with_types<8>(u_f, u_s, vfmt, fn);
        case 16: return with_types<16>(u_f, u_s, vfmt, fn);
        case 32: return with_types<32>(u_f, u_s, vfmt, fn);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace

bool chol_supported(int N, int u_f, int u_s, int u) {
    if (!(N == 2 || N == 4 || N == 8 || N == 16 || N == 32)) return false;
    if (!(u_f == MLMC_FMT_E4M3 || u_f == MLMC_FMT_F16 || u_f == MLMC_FMT_F32 || u_f == MLMC_FMT_F64)) return false;
    if (u_s == MLMC_FMT_F16)   // binary16 substitutions with a quarter / half factor and u = u_r <= binary32
        return (u_f == MLMC_FMT_E4M3 || u_f == MLMC_FMT_F16) && (u == MLMC_FMT_F16 || u == MLMC_FMT_F32);
    if (!(u_s == MLMC_FMT_F32 || u_s == MLMC_FMT_F64)) return false;
    return true;
}

size_t chol_scratch_bytes(int N, int u_f, int u_s, uint64_t nb, int u) {
    size_t bytes = 0;
    cudaError_t e = with_mesh(N, u_f, u_s, u, [&](auto L) { return decltype(L)::scratch(bytes, nb); });
    return e == cudaSuccess ? bytes : 0;
}

cudaError_t launch_chol_ir(int N, const double* a, uint64_t nb, int u_f, int u_s, double tol, int i_max, double* out,
                           int slot, unsigned* ctr, void* scratch, size_t bytes, cudaStream_t s, int u) {
    return with_mesh(N, u_f, u_s, u, [&](auto L) {
        return decltype(L)::run(a, nb, tol, i_max, out, slot, ctr, scratch, bytes, s);
    });
}

}  // namespace mlmc
