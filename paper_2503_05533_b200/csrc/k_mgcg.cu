// k_mgcg.cu -- K3m: multigrid-preconditioned conjugate gradients for the on-chip meshes (NEXT-4).
//
// SURVEY section 8(f) NEXT-4 ("multigrid-preconditioned Krylov, the optimal solver, gamma = 2",
// P:439): the same P1 system A x = b (R10) and the same accuracy contract as the paper's
// MINRES -- stop at the first k with ||r_k||_2 / ||b||_2 <= tol (the relative residual of Eq. (2),
// P:70-73, R9; r_k the CG recurrence residual) -- solved by preconditioned CG in binary64 with one
// symmetric V(1,1) cycle in binary32 as the preconditioner.  The QoI is carried as
// 1^T x_k = sum_i alpha_i 1^T p_i (a scalar, no x vector; cf. R26).
//
// Hierarchy: the P1 meshes are nested (h, 2h, ..., 1/2).  P = P1 interpolation on the coarse
// triangles (a fine node on a coarse horizontal, vertical or SW-NE diagonal edge takes the mean of its
// two endpoints), restriction = P^T, and the coarse operators are Galerkin-exact: for piecewise-
// constant coefficients P^T A_h P is the P1 stiffness of the coarse mesh whose triangle coefficients
// are the means of the four fine triangles inside each coarse triangle (the coarse basis functions
// are linear on the coarse triangle), so every level is again R10's 5-point conductance operator.
// Smoother: red-black Gauss-Seidel, red then black before the coarse correction, black then red
// after (symmetric: M^-1 is SPD, CG applies); the single unknown of the h = 1/2 level is solved
// exactly.
//
// B200 mapping: a group of T threads per system (persistent CTAs, job counter), every grid of the
// system in shared memory (binary64: p and the fine conductances; binary32: u, f, residual and the
// conductances of every level), r and A p in registers (thread-strided nodes); two fused reductions
// per CG step.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cfloat>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace mlmc {
namespace {

// PC = false (plain CG): only the binary64 grids -- no binary32 V-cycle hierarchy (it reserved
// ~114 KB at N = 64 that CG never reads and halved its residency)
template <int N, int T, int GROUPS_, bool PC = true>
struct MgCfg {
    static constexpr int GROUPS = GROUPS_;
    static constexpr int BLOCK = T * GROUPS;
    static constexpr int C = N - 1;
    static constexpr int n = C * C;
    static constexpr int PER = (n + T - 1) / T;                // fine nodes per thread
    static constexpr int G = N + 1;                            // grid side, Dirichlet ring included
    static constexpr int LV = __builtin_ctz(N);                // levels N, N/2, ..., 2
    static constexpr int D_P = 0, D_CE = G * G, D_CN = 2 * G * G, D_END = 3 * G * G;   // binary64 grids
    static __host__ __device__ constexpr int gl(int l) { return (N >> l) + 1; }
    // binary32 grids per level l: u, f, t, cE, cN (gl(l)^2 floats each)
    static __host__ __device__ constexpr int foff(int l) {
        int o = 0;
        for (int k = 0; k < l; ++k) o += 5 * gl(k) * gl(k);
        return o;
    }
    static constexpr int F_END = PC ? (foff(LV) + 3) / 4 * 4 : 0;   // keeps what follows 16-byte aligned
    static constexpr int NW = T >= 32 ? T / 32 : 1;
    static constexpr size_t SYS = (((size_t)D_END * 8 + (size_t)F_END * 4 + (size_t)2 * NW * 8 + 16) + 127) / 128 * 128;
    static constexpr size_t SMEM = SYS * GROUPS;
    static_assert((N & (N - 1)) == 0 && N >= 4, "power-of-two mesh");
};

template <int T, int GROUPS>
__device__ __forceinline__ void gsync(int g) {
    if constexpr (T < 32) __syncwarp(0xffffu << (threadIdx.x & 16));
    else if constexpr (T == 32) __syncwarp();
    else if constexpr (GROUPS == 1) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(T) : "memory");
}

// sums of (a, b) over the group's threads, identical in every thread (fixed order)
template <int T, int GROUPS>
__device__ __forceinline__ double2 gsum2(double a, double b, double* red, int tg, int g) {
    constexpr int W = T >= 32 ? 32 : T;
    const unsigned msk = T >= 32 ? 0xffffffffu : (0xffffu << (threadIdx.x & 16));
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) {
        a += __shfl_xor_sync(msk, a, o, W);
        b += __shfl_xor_sync(msk, b, o, W);
    }
    if constexpr (T <= 32) {
        return make_double2(a, b);
    } else {
        constexpr int NW = T / 32;
        gsync<T, GROUPS>(g);                                   // previous readers of red are done
        if ((tg & 31) == 0) { red[2 * (tg >> 5)] = a; red[2 * (tg >> 5) + 1] = b; }
        gsync<T, GROUPS>(g);
        double sa = red[0], sb = red[1];
#pragma unroll
        for (int w = 1; w < NW; ++w) { sa += red[2 * w]; sb += red[2 * w + 1]; }
        return make_double2(sa, sb);
    }
}

struct Lvl {             // one level's binary32 grids (side Gl = Nl + 1, node (i, j) at j * Gl + i)
    float *u, *f, *t, *ce, *cn;
    int Nl, Gl;
};

// red-black Gauss-Seidel sweep over the interior nodes of colour `col` ((i + j) % 2 == col):
// rows come in pairs holding C nodes of each colour (C = Nl - 1 is odd)
template <int T, int GROUPS>
__device__ __forceinline__ void rbgs(const Lvl& L, int col, int tg, int g) {
    const int C = L.Nl - 1;
    for (int q = tg; q < ((C + 1) / 2) * C; q += T) {
        const int pr = q / C, w = q % C;
        int j = 2 * pr + 1;
        int i0 = ((1 + j) & 1) == col ? 1 : 2;
        const int n1 = (C - i0) / 2 + 1;
        int i = i0 + 2 * w;
        if (w >= n1) {
            ++j;
            if (j > C) continue;
            i0 = ((1 + j) & 1) == col ? 1 : 2;
            i = i0 + 2 * (w - n1);
        }
        const int c = j * L.Gl + i;
        const float ce = L.ce[c], cw = L.ce[c - 1], cn = L.cn[c], cs = L.cn[c - L.Gl];
        float s = L.f[c];
        s = fmaf(ce, L.u[c + 1], s);
        s = fmaf(cw, L.u[c - 1], s);
        s = fmaf(cn, L.u[c + L.Gl], s);
        s = fmaf(cs, L.u[c - L.Gl], s);
        L.u[c] = s / ((ce + cw) + (cn + cs));
    }
    gsync<T, GROUPS>(g);
}

// conductances of a level from its triangle coefficients (aL at t[c], aU at f[c] for cell (i, j),
// c = j * Gl + i): cE(i,j) = (aL(i,j) + aU(i,j-1))/2, cN(i,j) = (aU(i,j) + aL(i-1,j))/2 (R10)
template <int T, int GROUPS>
__device__ __forceinline__ void level_conductances(const Lvl& L, int tg, int g) {
    const int Nl = L.Nl, Gl = L.Gl;
    for (int c = tg; c < Gl * Gl; c += T) {
        const int i = c % Gl, j = c / Gl;
        L.ce[c] = (i < Nl && j >= 1 && j < Nl) ? 0.5f * (L.t[c] + L.f[c - Gl]) : 0.0f;
        L.cn[c] = (i >= 1 && i < Nl && j < Nl) ? 0.5f * (L.f[c] + L.t[c - 1]) : 0.0f;
    }
    gsync<T, GROUPS>(g);
}

#ifndef MG_SMALL
#define MG_SMALL 8    // levels of side < MG_SMALL run on one warp
#endif
// ---- compile-time level operations.  A level of side NL is processed by NT threads (the whole group
// on the big levels; one warp once NL <= 16, synchronised by __syncwarp) -- every loop bound and
// index division is a compile-time constant.
template <int NT, int T, int GROUPS>
__device__ __forceinline__ void lsync(int g) {
    if constexpr (NT == T) gsync<T, GROUPS>(g);
    else __syncwarp();
}

template <int NL, int NT, int T, int GROUPS>
__device__ __forceinline__ void l_rbgs(const Lvl& L, int col, int tg, int g) {
    constexpr int C = NL - 1, GL = NL + 1, UR = NL >= 128 ? 4 : 1;   // big (global-memory) levels: more loads in flight
#pragma unroll (UR)
    for (int q = tg; q < ((C + 1) / 2) * C; q += NT) {
        const int pr = q / C, w = q % C;
        int j = 2 * pr + 1;
        int i0 = ((1 + j) & 1) == col ? 1 : 2;
        const int n1 = (C - i0) / 2 + 1;
        int i = i0 + 2 * w;
        if (w >= n1) {
            ++j;
            if (j > C) continue;
            i0 = ((1 + j) & 1) == col ? 1 : 2;
            i = i0 + 2 * (w - n1);
        }
        const int c = j * GL + i;
        const float ce = L.ce[c], cw = L.ce[c - 1], cn = L.cn[c], cs = L.cn[c - GL];
        float s = L.f[c];
        s = fmaf(ce, L.u[c + 1], s);
        s = fmaf(cw, L.u[c - 1], s);
        s = fmaf(cn, L.u[c + GL], s);
        s = fmaf(cs, L.u[c - GL], s);
        L.u[c] = __fdividef(s, (ce + cw) + (cn + cs));
    }
    lsync<NT, T, GROUPS>(g);
}

// levels of side NL: [u | f | t | cE | cN] at fb + offset, offsets of the halving sequence N, N/2, ...
template <int N, int NL>
__device__ __forceinline__ Lvl lvl_at(float* fb) {
    int off = 0;
#pragma unroll
    for (int k = N; k > NL; k >>= 1) off += 5 * (k + 1) * (k + 1);
    constexpr int sz = (NL + 1) * (NL + 1);
    float* b0 = fb + off;
    return Lvl{b0, b0 + sz, b0 + 2 * sz, b0 + 3 * sz, b0 + 4 * sz, NL, NL + 1};
}

// V(1,1) cycle from level NL down (u_NL = M^-1 f_NL; u starts at 0)
template <int N, int NL, int T, int GROUPS>
__device__ __forceinline__ void vcyc(float* fb, int tg, int g) {
    constexpr int NT = NL >= MG_SMALL ? T : (T >= 32 ? 32 : T);
    constexpr int GL = NL + 1, C = NL - 1, UR = NL >= 128 ? 4 : 1;
    const Lvl L = lvl_at<N, NL>(fb);
    if (NT != T && tg >= NT) return;                    // small levels: one warp
    if constexpr (NL == 2) {                            // one unknown: exact
        if (tg == 0) {
            constexpr int c = GL + 1;
            L.u[c] = L.f[c] / ((L.ce[c] + L.ce[c - 1]) + (L.cn[c] + L.cn[c - GL]));
        }
        lsync<NT, T, GROUPS>(g);
    } else {
        // first red sweep from u = 0 (the Dirichlet ring of u is zeroed once per system in mg_setup):
        // red nodes u = f / diag, black nodes u = 0 -- one pass instead of a zero fill plus a sweep
#pragma unroll (UR)
        for (int e = tg; e < C * C; e += NT) {
            const int i = e % C + 1, j = e / C + 1, c = j * GL + i;
            float v = 0.0f;
            if (!((i + j) & 1)) v = __fdividef(L.f[c], (L.ce[c] + L.ce[c - 1]) + (L.cn[c] + L.cn[c - GL]));
            L.u[c] = v;
        }
        lsync<NT, T, GROUPS>(g);
        l_rbgs<NL, NT, T, GROUPS>(L, 1, tg, g);
#pragma unroll (UR)
        for (int e = tg; e < C * C; e += NT) {         // t = f - A u
            const int c = (e / C + 1) * GL + (e % C + 1);
            const float ce = L.ce[c], cw = L.ce[c - 1], cn = L.cn[c], cs = L.cn[c - GL];
            float Au = ((ce + cw) + (cn + cs)) * L.u[c];
            Au = fmaf(-ce, L.u[c + 1], Au);
            Au = fmaf(-cw, L.u[c - 1], Au);
            Au = fmaf(-cn, L.u[c + GL], Au);
            Au = fmaf(-cs, L.u[c - GL], Au);
            L.t[c] = L.f[c] - Au;
        }
        lsync<NT, T, GROUPS>(g);
        // f_{NL/2} = P^T t: coarse (I, J) gathers fine (2I, 2J) with weight 1 and its E, W, N, S, NE, SW
        // neighbours with weight 1/2 (P1 prolongation on SW-NE triangles)
        constexpr int NC = NL / 2, GC = NC + 1, CC = NC - 1;
        const Lvl Cv = lvl_at<N, NC>(fb);
        for (int e = tg; e < GC * GC; e += NT) {
            const int I = e % GC, J = e / GC;
            float v = 0.0f;
            if (I >= 1 && I <= CC && J >= 1 && J <= CC) {
                const int c = (2 * J) * GL + 2 * I;
                v = L.t[c] + 0.5f * ((L.t[c + 1] + L.t[c - 1]) + (L.t[c + GL] + L.t[c - GL]) +
                                     (L.t[c + GL + 1] + L.t[c - GL - 1]));
            }
            Cv.f[e] = v;
        }
        lsync<NT, T, GROUPS>(g);
        vcyc<N, NC, T, GROUPS>(fb, tg, g);
        if constexpr (NT == T && NC < MG_SMALL && T > 32) gsync<T, GROUPS>(g);   // the warp's small levels are done
#pragma unroll (UR)
        for (int e = tg; e < C * C; e += NT) {         // u += P u_{NL/2}
            const int i = e % C + 1, j = e / C + 1, c = j * GL + i;
            const int I = i >> 1, J = j >> 1;
            const float* U = Cv.u;
            float v;
            if (!(i & 1) && !(j & 1)) v = U[J * GC + I];
            else if ((i & 1) && !(j & 1)) v = 0.5f * (U[J * GC + I] + U[J * GC + I + 1]);
            else if (!(i & 1) && (j & 1)) v = 0.5f * (U[J * GC + I] + U[(J + 1) * GC + I]);
            else v = 0.5f * (U[J * GC + I] + U[(J + 1) * GC + I + 1]);                // SW-NE diagonal
            L.u[c] += v;
        }
        lsync<NT, T, GROUPS>(g);
        l_rbgs<NL, NT, T, GROUPS>(L, 1, tg, g);
        l_rbgs<NL, NT, T, GROUPS>(L, 0, tg, g);
    }
}

// level l's grids (runtime l)
template <int N>
__device__ __forceinline__ Lvl level_rt(float* fb, int l) {
    int off = 0;
    for (int k = 0; k < l; ++k) off += 5 * ((N >> k) + 1) * ((N >> k) + 1);
    const int gl = (N >> l) + 1, sz = gl * gl;
    float* b0 = fb + off;
    return Lvl{b0, b0 + sz, b0 + 2 * sz, b0 + 3 * sz, b0 + 4 * sz, N >> l, gl};
}

// Per-system set-up: binary64 fine conductances cE, cN and p = 0; binary32 triangle coefficients,
// conductances and zero u (Dirichlet rings included) on every level.
template <int N, int T, int GROUPS>
__device__ __forceinline__ void mg_setup(const double* __restrict__ a, double* cE, double* cN, double* pg, float* fb,
                                         int tg, int g) {
    constexpr int G = N + 1, LV = __builtin_ctz(N);
    const Lvl L0 = level_rt<N>(fb, 0);
    for (int c = tg; c < G * G; c += T) {
        const int i = c % G, j = c / G;
        const bool cell = i < N && j >= 0 && j < N;
        const double aL = cell ? __ldg(a + 2 * (j * N + i)) : 0.0;          // aL of cell (i, j)
        const double aU = cell ? __ldg(a + 2 * (j * N + i) + 1) : 0.0;      // aU
        const double ce = (i < N && j >= 1 && j < N) ? 0.5 * (aL + __ldg(a + 2 * ((j - 1) * N + i) + 1)) : 0.0;
        const double cn = (i >= 1 && i < N && j < N) ? 0.5 * (aU + __ldg(a + 2 * (j * N + i - 1))) : 0.0;
        cE[c] = ce;
        cN[c] = cn;
        pg[c] = 0.0;
        L0.t[c] = (float)aL;
        L0.f[c] = (float)aU;
        L0.ce[c] = (float)ce;
        L0.cn[c] = (float)cn;
        L0.u[c] = 0.0f;
    }
    gsync<T, GROUPS>(g);
    for (int l = 1; l < LV; ++l) {
        // coarse lower triangle of cell (I, J) = mean of fine L(2I,2J), L(2I+1,2J), U(2I+1,2J),
        // L(2I+1,2J+1); upper = mean of U(2I,2J), L(2I,2J+1), U(2I,2J+1), U(2I+1,2J+1)
        const Lvl F = level_rt<N>(fb, l - 1);
        const Lvl Cv = level_rt<N>(fb, l);
        const int Gf = F.Gl, Gc = Cv.Gl, Nc = Cv.Nl;
        for (int e = tg; e < Gc * Gc; e += T) {
            const int I = e % Gc, J = e / Gc;
            float aL = 0.0f, aU = 0.0f;
            if (I < Nc && J < Nc) {
                const int c = (2 * J) * Gf + 2 * I;
                aL = 0.25f * ((F.t[c] + F.t[c + 1]) + (F.f[c + 1] + F.t[c + Gf + 1]));
                aU = 0.25f * ((F.f[c] + F.t[c + Gf]) + (F.f[c + Gf] + F.f[c + Gf + 1]));
            }
            Cv.t[e] = aL;
            Cv.f[e] = aU;
            Cv.u[e] = 0.0f;
        }
        gsync<T, GROUPS>(g);
        level_conductances<T, GROUPS>(Cv, tg, g);
    }
}

// Plain CG's set-up (PC = false): the binary64 fine conductances and p = 0 only
template <int N, int T, int GROUPS>
__device__ __forceinline__ void cg_setup(const double* __restrict__ a, double* cE, double* cN, double* pg, int tg,
                                         int g) {
    constexpr int G = N + 1;
    for (int c = tg; c < G * G; c += T) {
        const int i = c % G, j = c / G;
        const double ce = (i < N && j >= 1 && j < N)
                              ? 0.5 * (__ldg(a + 2 * (j * N + i)) + __ldg(a + 2 * ((j - 1) * N + i) + 1)) : 0.0;
        const double cn = (i >= 1 && i < N && j < N)
                              ? 0.5 * (__ldg(a + 2 * (j * N + i) + 1) + __ldg(a + 2 * (j * N + i - 1))) : 0.0;
        cE[c] = ce;
        cN[c] = cn;
        pg[c] = 0.0;
    }
    gsync<T, GROUPS>(g);
}

// PC = false: plain CG (NEXT-4) -- z = r, no V-cycle; everything else identical
template <int N, int T, int GROUPS, bool PC = true>
__global__ void __launch_bounds__(MgCfg<N, T, GROUPS, PC>::BLOCK)
mgcg_kernel(const double* __restrict__ a_all, int nb, double tol, int max_iter, double* __restrict__ out, int slot,
            unsigned* __restrict__ job_counter, const int* __restrict__ order, const int* __restrict__ nb_dev,
            int ok_status) {
    if (nb_dev) nb = *nb_dev;
    using K = MgCfg<N, T, GROUPS, PC>;
    constexpr int G = K::G, C = K::C, n = K::n, PER = K::PER, P = 2 * N * N;
    extern __shared__ __align__(128) unsigned char smem[];
    const int g = threadIdx.x / T, tg = threadIdx.x % T;
    unsigned char* base = smem + (size_t)g * K::SYS;
    double* dg = reinterpret_cast<double*>(base);
    double* pg = dg + K::D_P;
    double* cE = dg + K::D_CE;
    double* cN = dg + K::D_CN;
    float* fb = reinterpret_cast<float*>(dg + K::D_END);
    double* red = reinterpret_cast<double*>(fb + K::F_END);
    int* jobslot = reinterpret_cast<int*>(red + 2 * K::NW);
    const double h = 1.0 / N, h2 = h * h;

    // the thread's fine interior nodes: e = tg + k T, (i, j) = (e % C + 1, e / C + 1)
    auto cidx = [&](int k) {
        const int e = tg + k * T;
        return (e / C + 1) * G + (e % C + 1);
    };
    auto live = [&](int k) { return tg + k * T < n; };

    auto vcycle = [&]() {
        vcyc<N, N, T, GROUPS>(fb, tg, g);
        if constexpr (N < MG_SMALL && T > 32) gsync<T, GROUPS>(g);
    };

    for (;;) {
        if (tg == 0) jobslot[0] = (int)atomicAdd(job_counter, 1u);
        gsync<T, GROUPS>(g);
        const int job = jobslot[0];
        gsync<T, GROUPS>(g);
        if (job >= nb) break;
        const int sj = order ? __ldg(order + job) : job;
        const double* a = a_all + (size_t)sj * P;
        if constexpr (PC) mg_setup<N, T, GROUPS>(a, cE, cN, pg, fb, tg, g);
        else cg_setup<N, T, GROUPS>(a, cE, cN, pg, tg, g);
        const Lvl L0 = level_rt<N>(fb, 0);

        // ---- PCG from x0 = 0: r = b, z = M^-1 r, p = z
        double r[PER], q[PER];
        double rr = 0.0;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            r[k] = live(k) ? h2 : 0.0;
            if (PC && live(k)) L0.f[cidx(k)] = (float)h2;
            rr = fma(r[k], r[k], rr);
        }
        if constexpr (PC) {
            gsync<T, GROUPS>(g);
            vcycle();
        }
        double rz = 0.0;
#pragma unroll
        for (int k = 0; k < PER; ++k)
            if (live(k)) {
                const double z = PC ? (double)L0.u[cidx(k)] : r[k];
                pg[cidx(k)] = z;
                rz = fma(r[k], z, rz);
            }
        double2 S = gsum2<T, GROUPS>(rz, rr, red, tg, g);
        rz = S.x;
        const double bnorm = sqrt(S.y);
        const double tol_b = tol * bnorm;
        double Xq = 0.0, rnorm = bnorm;
        int it = 0, status = 1;
        if (bnorm == 0.0) status = 0;
        while (status == 1 && it < max_iter) {
            // q = A p (binary64), p.q and 1^T p
            double pq = 0.0, sp = 0.0;
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                q[k] = 0.0;
                if (live(k)) {
                    const int c = cidx(k);
                    const double ce = cE[c], cw = cE[c - 1], cn = cN[c], cs = cN[c - G];
                    const double pv = pg[c];
                    double Ap = ((ce + cw) + (cn + cs)) * pv;
                    Ap = fma(-ce, pg[c + 1], Ap);
                    Ap = fma(-cw, pg[c - 1], Ap);
                    Ap = fma(-cn, pg[c + G], Ap);
                    Ap = fma(-cs, pg[c - G], Ap);
                    q[k] = Ap;
                    pq = fma(pv, Ap, pq);
                    sp += pv;
                }
            }
            S = gsum2<T, GROUPS>(pq, sp, red, tg, g);
            const double alpha = rz / S.x;
            Xq = fma(alpha, S.y, Xq);                          // 1^T x += alpha 1^T p
            rr = 0.0;
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                r[k] = fma(-alpha, q[k], r[k]);
                if (PC && live(k)) L0.f[cidx(k)] = (float)r[k];
                rr = fma(r[k], r[k], rr);
            }
            ++it;
            if constexpr (PC) {
                gsync<T, GROUPS>(g);
                vcycle();
            }
            double rz_new = 0.0;
            double zk[PER];
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                zk[k] = live(k) ? (PC ? (double)L0.u[cidx(k)] : r[k]) : 0.0;
                rz_new = fma(r[k], zk[k], rz_new);
            }
            S = gsum2<T, GROUPS>(rz_new, rr, red, tg, g);
            rnorm = sqrt(S.y);
            if (!(rnorm == rnorm)) { status = 3; break; }
            if (rnorm <= tol_b) { status = 0; break; }         // ||r_k|| / ||b|| <= tol
            const double beta = S.x / rz;
            rz = S.x;
#pragma unroll
            for (int k = 0; k < PER; ++k)
                if (live(k)) pg[cidx(k)] = fma(beta, pg[cidx(k)], zk[k]);
            gsync<T, GROUPS>(g);
        }
        if (tg == 0) {
            double* o = out + (size_t)sj * kRecLen;
            o[0 + slot] = h2 * Xq;
            o[2 + slot] = (double)it;
            o[4 + slot] = bnorm > 0.0 ? rnorm / bnorm : 0.0;
            o[6 + slot] = (double)(status == 0 ? ok_status : status);
        }
        gsync<T, GROUPS>(g);
    }
}

// ---- K3m-g: the same MG-PCG for the streamed meshes (h = 1/128 .. 1/512).  One CTA (MG_GM_T threads) per
// system, every grid of the system in a per-CTA slice of global scratch: binary64 [p | cE | cN | r | q],
// then the binary32 levels exactly as on chip.  The passes are the on-chip ones (same arithmetic, same
// order per node), each a coalesced sweep over the grid through L1/L2; __syncthreads orders them.
#ifndef MG_GM_T
#define MG_GM_T 512
#endif
template <int N>
struct MgGm {
    static constexpr int T = MG_GM_T;
    static constexpr int G = N + 1;
    static constexpr size_t GG = (size_t)G * G;
    static constexpr size_t D_END = 5 * GG;                                          // doubles
    static constexpr size_t F_END = (MgCfg<N, 32, 1>::F_END + 31) / 32 * 32;           // floats
    static constexpr size_t SYS = ((D_END * 8 + F_END * 4) + 255) / 256 * 256;       // bytes per CTA
};

template <int N>
__global__ void __launch_bounds__(MG_GM_T, 1)
mgcg_gm_kernel(const double* __restrict__ a_all, int nb, double tol, int max_iter, double* __restrict__ out, int slot,
               unsigned* __restrict__ job_counter, const int* __restrict__ order, unsigned char* __restrict__ scratch,
               const int* __restrict__ nb_dev, int ok_status) {
    if (nb_dev) nb = *nb_dev;
    using K = MgGm<N>;
    constexpr int T = K::T, G = K::G, C = N - 1, n = C * C, P = 2 * N * N;
    __shared__ double red[2 * (T / 32)];
    __shared__ int jobslot;
    const int tg = threadIdx.x;
    double* dg = reinterpret_cast<double*>(scratch + (size_t)blockIdx.x * K::SYS);
    double* pg = dg;
    double* cE = dg + K::GG;
    double* cN = dg + 2 * K::GG;
    double* rg = dg + 3 * K::GG;
    double* qg = dg + 4 * K::GG;
    float* fb = reinterpret_cast<float*>(dg + K::D_END);
    const double h = 1.0 / N, h2 = h * h;
    auto cix = [](int e) { return (e / C + 1) * G + (e % C + 1); };

    for (;;) {
        if (tg == 0) jobslot = (int)atomicAdd(job_counter, 1u);
        __syncthreads();
        const int job = jobslot;
        __syncthreads();
        if (job >= nb) break;
        const int sj = order ? __ldg(order + job) : job;
        const double* a = a_all + (size_t)sj * P;
        mg_setup<N, T, 1>(a, cE, cN, pg, fb, tg, 0);
        const Lvl L0 = level_rt<N>(fb, 0);

        double rr = 0.0;
        for (int e = tg; e < n; e += T) {
            const int c = cix(e);
            rg[c] = h2;
            L0.f[c] = (float)h2;
            rr = fma(h2, h2, rr);
        }
        __syncthreads();
        vcyc<N, N, T, 1>(fb, tg, 0);
        double rz = 0.0;
#pragma unroll 4
        for (int e = tg; e < n; e += T) {
            const int c = cix(e);
            const double z = (double)L0.u[c];
            pg[c] = z;
            rz = fma(rg[c], z, rz);
        }
        double2 S = gsum2<T, 1>(rz, rr, red, tg, 0);
        rz = S.x;
        const double bnorm = sqrt(S.y);
        const double tol_b = tol * bnorm;
        double Xq = 0.0, rnorm = bnorm;
        int it = 0, status = 1;
        if (bnorm == 0.0) status = 0;
        while (status == 1 && it < max_iter) {
            double pq = 0.0, sp = 0.0;
#pragma unroll 4
            for (int e = tg; e < n; e += T) {
                const int c = cix(e);
                const double ce = cE[c], cw = cE[c - 1], cn = cN[c], cs = cN[c - G];
                const double pv = pg[c];
                double Ap = ((ce + cw) + (cn + cs)) * pv;
                Ap = fma(-ce, pg[c + 1], Ap);
                Ap = fma(-cw, pg[c - 1], Ap);
                Ap = fma(-cn, pg[c + G], Ap);
                Ap = fma(-cs, pg[c - G], Ap);
                qg[c] = Ap;
                pq = fma(pv, Ap, pq);
                sp += pv;
            }
            S = gsum2<T, 1>(pq, sp, red, tg, 0);
            const double alpha = rz / S.x;
            Xq = fma(alpha, S.y, Xq);
            rr = 0.0;
#pragma unroll 4
            for (int e = tg; e < n; e += T) {                  // own nodes only: no barrier needed on q
                const int c = cix(e);
                const double rv = fma(-alpha, qg[c], rg[c]);
                rg[c] = rv;
                L0.f[c] = (float)rv;
                rr = fma(rv, rv, rr);
            }
            ++it;
            __syncthreads();
            vcyc<N, N, T, 1>(fb, tg, 0);
            double rz_new = 0.0;
#pragma unroll 4
            for (int e = tg; e < n; e += T) {
                const int c = cix(e);
                rz_new = fma(rg[c], (double)L0.u[c], rz_new);
            }
            S = gsum2<T, 1>(rz_new, rr, red, tg, 0);
            rnorm = sqrt(S.y);
            if (!(rnorm == rnorm)) { status = 3; break; }
            if (rnorm <= tol_b) { status = 0; break; }
            const double beta = S.x / rz;
            rz = S.x;
#pragma unroll 4
            for (int e = tg; e < n; e += T) {
                const int c = cix(e);
                pg[c] = fma(beta, pg[c], (double)L0.u[c]);
            }
            __syncthreads();
        }
        if (tg == 0) {
            double* o = out + (size_t)sj * kRecLen;
            o[0 + slot] = h2 * Xq;
            o[2 + slot] = (double)it;
            o[4 + slot] = bnorm > 0.0 ? rnorm / bnorm : 0.0;
            o[6 + slot] = (double)(status == 0 ? ok_status : status);
        }
        __syncthreads();
    }
}

// ---- K3m-t: the streamed-mesh MG-PCG with temporal blocking (default for h = 1/128 .. 1/512).
// The fine level's ten grid passes per CG step become three:
//   A (tiles): r_k = r_{k-1} - alpha q, f = r_k in binary32, first red sweep, black sweep, residual
//      t = f - A u and restriction P^T t -- on a 64 x 32 tile with a 4-node halo (recomputed, never
//      exchanged); stores r_k, u and the coarse right-hand side;
//   B (tiles): u += P u_c, black sweep, red sweep -> z, r^T z -- 2-node halo; stores z;
//   C (tiles): p_{k+1} = z + beta p_k and q = A p_{k+1} formed together (p_{k+1} at the four
//      neighbours recomputed from p_k and z), p^T q, 1^T p.
// The tiles' inputs arrive as TMA boxes (72 x 40, zero-filled outside the grid) in two shared-memory
// stages, so the next tile streams in while this one is computed (as K3c).  r and p are ping-pong
// planes (a tile's halo must read the previous iterate where the neighbouring tile has already
// written the new one); z has its own plane.  Per node and step every value is the on-chip kernel's,
// with the same operations in the same order; only the partial-sum order of the dot products
// differs.  Coarser levels: vcyc from h = 2/N in the on-chip layout.
//
// Per-CTA scratch: binary64 planes [7][N+1][GP] (p0 p1 cE cN r0 r1 q), binary32 planes [4][N+1][GP]
// (ce cn u z), GP = N + 4 with grid column i stored at i + 3 (so every box starts 16-byte aligned),
// then the on-chip level layout (level 0 only as set-up temporaries).
namespace tl {
constexpr int T = 512;
constexpr int TX = 64, TY = 32, H = 4;
constexpr int BX = TX + 2 * H, BY = TY + 2 * H, BN = BX * BY;          // 72 x 40 box
constexpr int B64 = BN * 8, B32 = BN * 4;                               // box bytes (multiples of 128)
constexpr int STAGE = 2 * B64 + 3 * B32;     // A: R, Q | CE, CN; B: R | CE, CN, U; C: P, CE64, CN64 | Z
static_assert(3 * B64 + B32 == STAGE, "pass C's boxes fill the same stage");
constexpr int CWX = TX / 2 + 4, CWY = TY / 2 + 4;                       // coarse window of a tile
constexpr size_t SMEM = 2 * (size_t)STAGE + 2 * (size_t)B32 + (CWX * CWY * 4 + 7) / 8 * 8 + 2 * (T / 32) * 8 + 2 * 8 + 16;
enum { P0, P1, DCE, DCN, R0, R1, DQ, ND };                               // binary64 planes
enum { FCE, FCN, FU, FZ, NF };                                           // binary32 planes
__host__ __device__ constexpr int gp(int N) { return N + 4; }
}  // namespace tl

template <int N>
struct MgTl {
    static constexpr int GP = tl::gp(N);
    static constexpr size_t PL = (size_t)GP * (N + 1);                   // elements per plane
    static constexpr size_t D_BYTES = tl::ND * PL * 8;
    static constexpr size_t F_BYTES = tl::NF * PL * 4;
    static constexpr size_t F_END = (MgCfg<N, 32, 1>::F_END + 31) / 32 * 32;   // on-chip level layout
    static constexpr size_t SYS = (D_BYTES + F_BYTES + F_END * 4 + 255) / 256 * 256;
    static constexpr int NTX = (N - 1 + tl::TX - 1) / tl::TX, NTY = (N - 1 + tl::TY - 1) / tl::TY;
    static constexpr int NT = NTX * NTY;
};

__device__ __forceinline__ uint32_t mg_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mg_mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mg_tma(uint32_t dst, const CUtensorMap* map, int x, int y, int plane, int cta,
                                       uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
            "r"(dst), "l"(map), "r"(x), "r"(y), "r"(plane), "r"(cta), "r"(bar)
        : "memory");
}

// issue tile t of pass A (mode 0: r_old = plane v, q | ce, cn), B (mode 1: r_new = plane v | ce, cn, u) or
// C (mode 2: p_old = plane v, cE, cN | z) into stage s
template <int N>
__device__ __forceinline__ void mg_issue(const CUtensorMap* m64, const CUtensorMap* m32, unsigned char* stage0,
                                         uint32_t bar0, int cta, int t, int s, int mode, int v) {
    using K = MgTl<N>;
    const int x = (t % K::NTX) * tl::TX;                          // stored column of node x0 - H
    const int y = 1 + (t / K::NTX) * tl::TY - tl::H;
    const uint32_t dst = mg_smem_u32(stage0 + (size_t)s * tl::STAGE), bar = bar0 + 8 * s;
    const uint32_t bytes = mode == 0 ? 2 * tl::B64 + 2 * tl::B32 : mode == 1 ? tl::B64 + 3 * tl::B32 : 3 * tl::B64 + tl::B32;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    mg_tma(dst, m64, x, y, v, cta, bar);
    if (mode == 2) {
        mg_tma(dst + tl::B64, m64, x, y, tl::DCE, cta, bar);
        mg_tma(dst + 2 * tl::B64, m64, x, y, tl::DCN, cta, bar);
        mg_tma(dst + 3 * tl::B64, m32, x, y, tl::FZ, cta, bar);
        return;
    }
    if (mode == 0) mg_tma(dst + tl::B64, m64, x, y, tl::DQ, cta, bar);
    mg_tma(dst + 2 * tl::B64, m32, x, y, tl::FCE, cta, bar);
    mg_tma(dst + 2 * tl::B64 + tl::B32, m32, x, y, tl::FCN, cta, bar);
    if (mode == 1) mg_tma(dst + 2 * tl::B64 + 2 * tl::B32, m32, x, y, tl::FU, cta, bar);
}

template <int N>
__global__ void __launch_bounds__(tl::T, 1)
mgcg_tile_kernel(const __grid_constant__ CUtensorMap m64, const __grid_constant__ CUtensorMap m32,
                 const double* __restrict__ a_all, int nb, double tol, int max_iter, double* __restrict__ out,
                 int slot, unsigned* __restrict__ job_counter, const int* __restrict__ order,
                 unsigned char* __restrict__ scratch,
                 const int* __restrict__ nb_dev, int ok_status) {
    if (nb_dev) nb = *nb_dev;
    using K = MgTl<N>;
    constexpr int T = tl::T, GP = K::GP, C = N - 1, P = 2 * N * N;
    constexpr int BX = tl::BX, BN = tl::BN, H = tl::H, TX = tl::TX, TY = tl::TY, NT = K::NT;
    constexpr int NC = N / 2, GC = NC + 1;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* stage0 = smem;
    float* sf = reinterpret_cast<float*>(smem + 2 * tl::STAGE);     // f, then t (pass A)
    float* su = sf + BN;
    float* scu = su + BN;                                          // coarse u of the tile (pass B)
    double* red = reinterpret_cast<double*>(scu + tl::CWX * tl::CWY);
    uint64_t* bars = reinterpret_cast<uint64_t*>(red + 2 * (T / 32));
    int* jobslot = reinterpret_cast<int*>(bars + 2);
    const int tg = threadIdx.x, cta = blockIdx.x;
    unsigned char* base = scratch + (size_t)cta * K::SYS;
    double* D = reinterpret_cast<double*>(base);
    float* F = reinterpret_cast<float*>(base + K::D_BYTES);
    float* fb = reinterpret_cast<float*>(base + K::D_BYTES + K::F_BYTES);    // on-chip level layout
    auto dpl = [&](int pl) { return D + (size_t)pl * K::PL; };
    auto fpl = [&](int pl) { return F + (size_t)pl * K::PL; };
    double* cE = dpl(tl::DCE);
    double* cN = dpl(tl::DCN);
    double* qg = dpl(tl::DQ);
    float* ug = fpl(tl::FU);
    float* zg = fpl(tl::FZ);
    const double h = 1.0 / N, h2 = h * h;
    const uint32_t bar0 = mg_smem_u32(&bars[0]);
    if (tg == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t phase = 0;
    constexpr int MS = (BN + T - 1) / T;
    int kxy[MS];                                                   // box coordinates of this thread's slots
#pragma unroll
    for (int m = 0; m < MS; ++m) {
        const int k = tg + m * T;
        kxy[m] = (k % BX) | ((k / BX) << 16);
    }
    auto gix = [](int i, int j) { return j * GP + i + 3; };
    auto interior = [](int i, int j) { return i >= 1 && i <= C && j >= 1 && j <= C; };

    for (;;) {
        if (tg == 0) *jobslot = (int)atomicAdd(job_counter, 1u);
        __syncthreads();
        const int job = *jobslot;
        __syncthreads();
        if (job >= nb) break;
        const int sj = order ? __ldg(order + job) : job;
        const double* a = a_all + (size_t)sj * P;
        // on-chip-layout levels (coarse levels; level 0 as temporaries); its binary64 outputs go to
        // planes that are re-initialised below
        mg_setup<N, T, 1>(a, dpl(tl::R1), dpl(tl::DQ), dpl(tl::P1), fb, tg, 0);
        for (int e = tg; e < (int)K::PL; e += T) {
            const int i = e % GP - 3, j = e / GP;
            double ce = 0.0, cn = 0.0;
            if (i >= 0 && i < N && j >= 1 && j < N)
                ce = 0.5 * (__ldg(a + 2 * (j * N + i)) + __ldg(a + 2 * ((j - 1) * N + i) + 1));
            if (i >= 1 && i < N && j < N) cn = 0.5 * (__ldg(a + 2 * (j * N + i) + 1) + __ldg(a + 2 * (j * N + i - 1)));
            D[e] = 0.0;                                     // p0
            D[K::PL + e] = 0.0;                             // p1
            cE[e] = ce;
            cN[e] = cn;
            D[tl::R0 * K::PL + e] = interior(i, j) ? h2 : 0.0;
            D[tl::R1 * K::PL + e] = 0.0;
            qg[e] = 0.0;
            F[e] = (float)ce;
            F[K::PL + e] = (float)cn;
            ug[e] = 0.0f;
            zg[e] = 0.0f;
        }
        const Lvl L1 = level_rt<N>(fb, 1);
        int cr = 0, cp = 0;            // current r / p planes (R0 + cr, P0 + cp)

        // ---- tile loop of one pass (TMA double buffer; the first two tiles are issued here).
        // mode 0 = pass A (coef = alpha, acc = r^T r), 1 = pass B (acc = r^T z), 2 = pass C (coef = beta,
        // acc = p^T q, acc2 = 1^T p).  Thread tg owns box slots k = tg + m T (coordinates in kxy[m]); a
        // stage touches the slots whose box coordinates fall in a per-tile window (span()).
        auto run_pass = [&](int mode, double coef, double& acc, double& acc2) {
            const int ro = mode == 2 ? tl::P0 + cp : tl::R0 + cr;      // A: r_old; B: r_new; C: p_old
            double* rn = dpl(tl::R0 + (cr ^ 1));
            double* pn = dpl(tl::P0 + (cp ^ 1));
            asm volatile("fence.proxy.async.global;" ::: "memory");   // generic stores -> TMA reads
            __syncthreads();
            if (tg == 0) {
                mg_issue<N>(&m64, &m32, stage0, bar0, cta, 0, 0, mode, ro);
                if (NT > 1) mg_issue<N>(&m64, &m32, stage0, bar0, cta, 1, 1, mode, ro);
            }
            const float* U = L1.u;
            for (int t = 0; t < NT; ++t) {
                const int s = t & 1;
                const int x0 = 1 + (t % K::NTX) * TX, y0 = 1 + (t / K::NTX) * TY;
                const int ox = x0 - H, oy = y0 - H;                     // grid node of box slot (0, 0)
                const int wx = min(x0 + TX, N) - x0, wy = min(y0 + TY, N) - y0;   // owned extent
                const int par = (ox + oy) & 1;                          // colour of slot (lx, ly): (lx + ly + par) & 1
                // window of the interior nodes within hh of the owned region, in box coordinates
                auto span = [&](int hh) {
                    return make_int4(max(H - hh, 1 - ox), min(wx + H + hh - 1, C - ox), max(H - hh, 1 - oy),
                                     min(wy + H + hh - 1, C - oy));
                };
                auto in = [](int4 w, int lx, int ly) { return lx >= w.x && lx <= w.y && ly >= w.z && ly <= w.w; };
                const int cx0 = max(0, (x0 - 2) >> 1), cy0 = max(0, (y0 - 2) >> 1);
                if (mode == 1) {                                        // coarse u of the tile -> smem
                    for (int e = tg; e < tl::CWX * tl::CWY; e += T) {
                        const int I = cx0 + e % tl::CWX, J = cy0 + e / tl::CWX;
                        scu[e] = (I <= NC && J <= NC) ? U[J * GC + I] : 0.0f;
                    }
                }
                mg_mbar_wait(bar0 + 8 * s, (phase >> s) & 1u);
                phase ^= 1u << s;
                const unsigned char* st = stage0 + (size_t)s * tl::STAGE;
                const double* R = reinterpret_cast<const double*>(st);
                const double* Q = reinterpret_cast<const double*>(st + tl::B64);
                const float* CE = reinterpret_cast<const float*>(st + 2 * tl::B64);
                const float* CN = CE + BN;
                const float* UU = CN + BN;
                auto sweep = [&](int4 w, int colour) {                  // Gauss-Seidel on one colour
#pragma unroll
                    for (int m = 0; m < MS; ++m) {
                        const int k = tg + m * T, lx = kxy[m] & 0xffff, ly = kxy[m] >> 16;
                        if (k < BN && in(w, lx, ly) && ((lx + ly + par) & 1) == colour) {
                            const float ce = CE[k], cw = CE[k - 1], cn = CN[k], cs = CN[k - BX];
                            float sv = sf[k];
                            sv = fmaf(ce, su[k + 1], sv);
                            sv = fmaf(cw, su[k - 1], sv);
                            sv = fmaf(cn, su[k + BX], sv);
                            sv = fmaf(cs, su[k - BX], sv);
                            su[k] = __fdividef(sv, (ce + cw) + (cn + cs));
                        }
                    }
                };
                if (mode == 2) {
                    // p_new = z + beta p_old and q = A p_new on the owned nodes (p_new at the neighbours
                    // recomputed from the box)
                    const double* PB = R;
                    const double* E64 = PB + BN;
                    const double* N64 = E64 + BN;
                    const float* ZB = reinterpret_cast<const float*>(N64 + BN);
                    auto pnew = [&](int kk) { return fma(coef, PB[kk], (double)ZB[kk]); };
                    const int4 w0 = span(0);
#pragma unroll
                    for (int m = 0; m < MS; ++m) {
                        const int k = tg + m * T, lx = kxy[m] & 0xffff, ly = kxy[m] >> 16;
                        if (k < BN && in(w0, lx, ly)) {
                            const double ce = E64[k], cw = E64[k - 1], cn = N64[k], cs = N64[k - BX];
                            const double pv = pnew(k);
                            double Ap = ((ce + cw) + (cn + cs)) * pv;
                            Ap = fma(-ce, pnew(k + 1), Ap);
                            Ap = fma(-cw, pnew(k - 1), Ap);
                            Ap = fma(-cn, pnew(k + BX), Ap);
                            Ap = fma(-cs, pnew(k - BX), Ap);
                            const int c = gix(ox + lx, oy + ly);
                            qg[c] = Ap;
                            pn[c] = pv;
                            acc = fma(pv, Ap, acc);
                            acc2 += pv;
                        }
                    }
                } else if (mode == 0) {
                    const int4 wH = span(H), w3 = span(H - 1), w0 = span(0), w1 = span(1);
#pragma unroll
                    for (int m = 0; m < MS; ++m) {                      // r_k, f = (float) r_k; first red sweep
                        const int k = tg + m * T, lx = kxy[m] & 0xffff, ly = kxy[m] >> 16;
                        if (k >= BN) continue;
                        float f = 0.0f, u = 0.0f;
                        if (in(wH, lx, ly)) {
                            const double r = fma(-coef, Q[k], R[k]);
                            f = (float)r;
                            if (in(w0, lx, ly)) {
                                rn[gix(ox + lx, oy + ly)] = r;
                                acc = fma(r, r, acc);
                            }
                            if (in(w3, lx, ly) && !((lx + ly + par) & 1))
                                u = __fdividef(f, (CE[k] + CE[k - 1]) + (CN[k] + CN[k - BX]));
                        }
                        sf[k] = f;
                        su[k] = u;
                    }
                    __syncthreads();
                    sweep(span(H - 2), 1);
                    __syncthreads();
#pragma unroll
                    for (int m = 0; m < MS; ++m) {                      // t = f - A u (in place of f); store u
                        const int k = tg + m * T, lx = kxy[m] & 0xffff, ly = kxy[m] >> 16;
                        if (k < BN && in(w1, lx, ly)) {
                            const float ce = CE[k], cw = CE[k - 1], cn = CN[k], cs = CN[k - BX];
                            float Au = ((ce + cw) + (cn + cs)) * su[k];
                            Au = fmaf(-ce, su[k + 1], Au);
                            Au = fmaf(-cw, su[k - 1], Au);
                            Au = fmaf(-cn, su[k + BX], Au);
                            Au = fmaf(-cs, su[k - BX], Au);
                            sf[k] = sf[k] - Au;
                            if (in(w0, lx, ly)) ug[gix(ox + lx, oy + ly)] = su[k];
                        }
                    }
                    __syncthreads();
                    // f_c = P^T t for the coarse nodes whose centre (2I, 2J) this tile owns
                    const int Ilo = max(1, (x0 + 1) / 2), Ihi = min(NC - 1, (x0 + wx - 1) / 2);
                    const int Jlo = max(1, (y0 + 1) / 2), Jhi = min(NC - 1, (y0 + wy - 1) / 2);
                    const int nI = Ihi - Ilo + 1, nJ = Jhi - Jlo + 1;
                    if (nI > 0 && nJ > 0)
                        for (int e = tg; e < nI * nJ; e += T) {
                            const int I = Ilo + e % nI, J = Jlo + e / nI;
                            const int k = (2 * J - oy) * BX + (2 * I - ox);
                            L1.f[J * GC + I] = sf[k] + 0.5f * ((sf[k + 1] + sf[k - 1]) + (sf[k + BX] + sf[k - BX]) +
                                                               (sf[k + BX + 1] + sf[k - BX - 1]));
                        }
                } else {
                    __syncthreads();                                    // scu written
                    const int4 w2 = span(2), w0 = span(0);
#pragma unroll
                    for (int m = 0; m < MS; ++m) {                      // f = (float) r_k, u = u_pre + P u_c
                        const int k = tg + m * T, lx = kxy[m] & 0xffff, ly = kxy[m] >> 16;
                        if (k >= BN) continue;
                        float f = 0.0f, u = 0.0f;
                        if (in(w2, lx, ly)) {
                            const int i = ox + lx, j = oy + ly;
                            f = (float)R[k];
                            const int I = (i >> 1) - cx0, J = (j >> 1) - cy0;
                            const float* Uc = scu + J * tl::CWX + I;
                            float v;
                            if (!(i & 1) && !(j & 1)) v = Uc[0];
                            else if ((i & 1) && !(j & 1)) v = 0.5f * (Uc[0] + Uc[1]);
                            else if (!(i & 1) && (j & 1)) v = 0.5f * (Uc[0] + Uc[tl::CWX]);
                            else v = 0.5f * (Uc[0] + Uc[tl::CWX + 1]);
                            u = UU[k] + v;
                        }
                        sf[k] = f;
                        su[k] = u;
                    }
                    __syncthreads();
                    sweep(span(1), 1);
                    __syncthreads();
#pragma unroll
                    for (int m = 0; m < MS; ++m) {                      // red sweep on the owned nodes; z out
                        const int k = tg + m * T, lx = kxy[m] & 0xffff, ly = kxy[m] >> 16;
                        if (k < BN && in(w0, lx, ly)) {
                            float z = su[k];
                            if (!((lx + ly + par) & 1)) {
                                const float ce = CE[k], cw = CE[k - 1], cn = CN[k], cs = CN[k - BX];
                                float sv = sf[k];
                                sv = fmaf(ce, su[k + 1], sv);
                                sv = fmaf(cw, su[k - 1], sv);
                                sv = fmaf(cn, su[k + BX], sv);
                                sv = fmaf(cs, su[k - BX], sv);
                                z = __fdividef(sv, (ce + cw) + (cn + cs));
                            }
                            zg[gix(ox + lx, oy + ly)] = z;
                            acc = fma(R[k], (double)z, acc);
                        }
                    }
                }
                __syncthreads();                            // stage s, sf, su, scu free
                if (tg == 0 && t + 2 < NT) mg_issue<N>(&m64, &m32, stage0, bar0, cta, t + 2, s, mode, ro);
            }
            if (mode == 0) cr ^= 1;
            if (mode == 2) cp ^= 1;
        };

        // ---- PCG from x0 = 0 (r_0 = b, q = 0, p = 0, alpha = beta = 0 for the first passes)
        double rr = 0.0, rz = 0.0, dummy = 0.0;
        run_pass(0, 0.0, rr, dummy);
        __syncthreads();
        vcyc<N, NC, T, 1>(fb, tg, 0);
        run_pass(1, 0.0, rz, dummy);
        double2 S = gsum2<T, 1>(rz, rr, red, tg, 0);
        rz = S.x;
        const double bnorm = sqrt(S.y);
        const double tol_b = tol * bnorm;
        double Xq = 0.0, rnorm = bnorm, beta = 0.0;
        int it = 0, status = 1;
        if (bnorm == 0.0) status = 0;
        while (status == 1 && it < max_iter) {
            double pq = 0.0, sp = 0.0;
            run_pass(2, beta, pq, sp);
            S = gsum2<T, 1>(pq, sp, red, tg, 0);
            const double alpha = rz / S.x;
            Xq = fma(alpha, S.y, Xq);
            rr = 0.0;
            run_pass(0, alpha, rr, dummy);
            ++it;
            __syncthreads();
            vcyc<N, NC, T, 1>(fb, tg, 0);
            double rz_new = 0.0;
            run_pass(1, 0.0, rz_new, dummy);
            S = gsum2<T, 1>(rz_new, rr, red, tg, 0);
            rnorm = sqrt(S.y);
            if (!(rnorm == rnorm)) { status = 3; break; }
            if (rnorm <= tol_b) { status = 0; break; }
            beta = S.x / rz;
            rz = S.x;
        }
        if (tg == 0) {
            double* o = out + (size_t)sj * kRecLen;
            o[0 + slot] = h2 * Xq;
            o[2 + slot] = (double)it;
            o[4 + slot] = bnorm > 0.0 ? rnorm / bnorm : 0.0;
            o[6 + slot] = (double)(status == 0 ? ok_status : status);
        }
        __syncthreads();
    }
}

template <int N>
cudaError_t run_mg_tile(const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot, unsigned* ctr,
                        const int* order, void* scratch, int nctas, cudaStream_t s, const int* nb_dev, int ok_status) {
    using K = MgTl<N>;
    if (!scratch || nctas < 1) return cudaErrorInvalidValue;
    static PerDevice<cudaError_t> attr;              // the attribute is per device
    cudaError_t de = cudaSuccess;
    const cudaError_t ae = attr.get([] {
        return cudaFuncSetAttribute(mgcg_tile_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tl::SMEM);
    }, &de);
    if (de != cudaSuccess) return de;
    if (ae != cudaSuccess) return ae;
    const uint64_t grid = std::min<uint64_t>(nb, (uint64_t)nctas);
    if (grid == 0) return cudaSuccess;
    CUtensorMap m64, m32;
    const uint64_t d64[4] = {(uint64_t)K::GP, (uint64_t)N + 1, (uint64_t)tl::ND, grid};
    const uint64_t s64[3] = {(uint64_t)K::GP * 8, K::PL * 8, K::SYS};
    const uint64_t d32[4] = {(uint64_t)K::GP, (uint64_t)N + 1, (uint64_t)tl::NF, grid};
    const uint64_t s32[3] = {(uint64_t)K::GP * 4, K::PL * 4, K::SYS};
    const uint32_t box[4] = {(uint32_t)tl::BX, (uint32_t)tl::BY, 1, 1};
    unsigned char* sc = static_cast<unsigned char*>(scratch);
    if (!encode_tensor_map(&m64, true, 4, sc, d64, s64, box) ||
        !encode_tensor_map(&m32, false, 4, sc + K::D_BYTES, d32, s32, box))
        return cudaErrorInvalidValue;
    mgcg_tile_kernel<N><<<(unsigned)grid, tl::T, tl::SMEM, s>>>(m64, m32, a, (int)nb, tol, max_iter, out, slot, ctr,
                                                               order, sc, nb_dev, ok_status);
    return cudaGetLastError();
}

// MLMC_MG_GM=plain selects the ten-pass global-memory kernel (A/B runs).
bool use_mg_plain() {
#ifndef MLMC_TUNING
    return false;      // production build: the tiled kernel (K3m-t) only
#endif
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("MLMC_MG_GM");
        v = (e && std::strcmp(e, "plain") == 0) ? 1 : 0;
    }
    return v == 1;
}

template <int N, int T, int GROUPS, bool PC = true>
cudaError_t run_mg(const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot, unsigned* ctr,
                   const int* order, cudaStream_t s, const int* nb_dev, int ok_status) {
    using K = MgCfg<N, T, GROUPS, PC>;
    auto kern = mgcg_kernel<N, T, GROUPS, PC>;
    static PerDevice<KernelOcc> occ_cache;
    const KernelOcc occ = occ_of(occ_cache, kern, K::BLOCK, K::SMEM);
    if (occ.err != cudaSuccess) return occ.err;
    const uint64_t grid = std::min<uint64_t>((nb + GROUPS - 1) / GROUPS, (uint64_t)occ.per_sm * occ.sms);
    if (grid == 0) return cudaSuccess;
    kern<<<(unsigned)grid, K::BLOCK, K::SMEM, s>>>(a, (int)nb, tol, max_iter, out, slot, ctr, order, nb_dev,
                                                 ok_status);
    return cudaGetLastError();
}

template <int N>
cudaError_t run_mg_gm(const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot, unsigned* ctr,
                      const int* order, void* scratch, int nctas, cudaStream_t s, const int* nb_dev, int ok_status) {
    if (!scratch || nctas < 1) return cudaErrorInvalidValue;
    const uint64_t grid = std::min<uint64_t>(nb, (uint64_t)nctas);
    if (grid == 0) return cudaSuccess;
    mgcg_gm_kernel<N><<<(unsigned)grid, MgGm<N>::T, 0, s>>>(a, (int)nb, tol, max_iter, out, slot, ctr, order,
                                                           static_cast<unsigned char*>(scratch), nb_dev, ok_status);
    return cudaGetLastError();
}

}  // namespace

bool mgcg_supported(int N) { return N == 8 || N == 16 || N == 32 || N == 64 || N == 128 || N == 256 || N == 512; }

size_t mgcg_scratch_per_cta(int N) {
    const bool plain = use_mg_plain();
    switch (N) {
        case 128: return plain ? (size_t)MgGm<128>::SYS : (size_t)MgTl<128>::SYS;
        case 256: return plain ? (size_t)MgGm<256>::SYS : (size_t)MgTl<256>::SYS;
        case 512: return plain ? (size_t)MgGm<512>::SYS : (size_t)MgTl<512>::SYS;
        default: return 0;
    }
}

int mgcg_ctas_per_sm(int N) { (void)N; return 1; }

#ifdef MLMC_TUNING
#define MG_GM(n) run_mg_gm<n>(a, nb, tol, max_iter, out, slot, ctr, order, scratch, nctas, s, nb_dev, ok_status)
#else
#define MG_GM(n) cudaErrorNotSupported
#endif
cudaError_t launch_mgcg(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                        unsigned* ctr, const int* order, void* scratch, int nctas, cudaStream_t s, const int* nb_dev,
                        int ok_status) {
    const bool plain = use_mg_plain();
    switch (N) {
        case 8: return run_mg<8, 32, 4>(a, nb, tol, max_iter, out, slot, ctr, order, s, nb_dev, ok_status);
        case 16: return run_mg<16, 32, 4>(a, nb, tol, max_iter, out, slot, ctr, order, s, nb_dev, ok_status);
        case 32: return run_mg<32, 128, 1>(a, nb, tol, max_iter, out, slot, ctr, order, s, nb_dev, ok_status);
        case 64: return run_mg<64, 256, 1>(a, nb, tol, max_iter, out, slot, ctr, order, s, nb_dev, ok_status);
        case 128:
            return plain ? MG_GM(128)
                         : run_mg_tile<128>(a, nb, tol, max_iter, out, slot, ctr, order, scratch, nctas, s, nb_dev, ok_status);
        case 256:
            return plain ? MG_GM(256)
                         : run_mg_tile<256>(a, nb, tol, max_iter, out, slot, ctr, order, scratch, nctas, s, nb_dev, ok_status);
        case 512:
            return plain ? MG_GM(512)
                         : run_mg_tile<512>(a, nb, tol, max_iter, out, slot, ctr, order, scratch, nctas, s, nb_dev, ok_status);
        default: return cudaErrorNotSupported;
    }
}

bool cg_supported(int N) { return N == 8 || N == 16 || N == 32 || N == 64; }

cudaError_t launch_cg(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                      unsigned* ctr, const int* order, cudaStream_t s) {
    switch (N) {
        case 8: return run_mg<8, 32, 4, false>(a, nb, tol, max_iter, out, slot, ctr, order, s, nullptr, 0);
        case 16: return run_mg<16, 32, 4, false>(a, nb, tol, max_iter, out, slot, ctr, order, s, nullptr, 0);
        case 32: return run_mg<32, 128, 1, false>(a, nb, tol, max_iter, out, slot, ctr, order, s, nullptr, 0);
        case 64: return run_mg<64, 256, 1, false>(a, nb, tol, max_iter, out, slot, ctr, order, s, nullptr, 0);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace mlmc
