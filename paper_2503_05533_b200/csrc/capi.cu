// capi.cu -- the C-ABI of include/mlmc.h: plan, workspace, per-level sampling and Algorithm 2.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <mutex>
#include <vector>

#include "internal.h"

using namespace mlmc;

struct mlmc_ctx {
    mlmc_problem pr{};
    KLModes kl;
    int device = 0;
    int sms = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t single_c = nullptr;     // mlmc_sample_level: the coarse solve's stream (forked off ctx->stream)
    cudaEvent_t single_fork = nullptr, single_join = nullptr;
    cudaStream_t stream = nullptr;
    std::vector<double*> phi_dev;        // per level, lazily built (P x m synthesis, MLMC_FIELD_KERNEL=dense)
    SepModes sep;                        // separable synthesis (default): modes by x-function ...
    int* sep_i = nullptr;                // ... on the device: the K x K mode map (k of the pair (a, b), or -1)
    double* sep_c = nullptr;             //     and its c_k (0 where no mode)
    std::vector<double*> tab_dev;        // per level: the four 1D tables [4][N][K], lazily built
    unsigned char* ws = nullptr;         // borrowed workspace
    size_t ws_bytes = 0;
    double* sums_dev = nullptr;          // owned: MLMC_MAX_LEVELS * kSumsLen
    double* adapt_dev = nullptr;         // owned: mlmc_adaptive_run's per-round level sums (MLMC_MAX_LEVELS * kSumsLen)
    unsigned long long* xsums_dev = nullptr;   // owned: MLMC_MAX_LEVELS * kXLen exact sums of the last call
    bool want_xsums = false;             // form them (inside mlmc_adaptive_run only)
    std::string err;
    struct AutoChoice { int N, cls; mlmc_precision p; double ms; };
    std::vector<AutoChoice> auto_choice;   // policy 3: per mesh, the solver the pilot chose
    // per-kernel accounting
    bool prof_on = false;
    std::vector<mlmc_kernel_stat> stats;
    struct Pending { int idx; cudaEvent_t a, b; };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> ev_pool;
    // concurrent levels (mlmc_sample_levels_async): priority streams + fork/join events
    std::vector<cudaStream_t> aux;
    std::vector<cudaEvent_t> join_ev;
    cudaEvent_t fork_ev = nullptr;
    // per level slot: a second stream for the coarse solve, its fork/join events, and the
    // "fields ready" event that gates the other levels' solves behind the largest level's
    std::vector<cudaStream_t> aux_c;
    std::vector<cudaEvent_t> cfork_ev, cjoin_ev, prep_ev;
};

namespace {

thread_local std::string g_err;

int fail(mlmc_ctx* c, int code, const std::string& msg) {
    if (c) c->err = msg;
    g_err = msg;
    return code;
}

#define CU(call)                                                                                        \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess) return fail(ctx, MLMC_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

int level_N(const mlmc_ctx* c, int level) { return c->pr.h0_inv << level; }

int stat_index(mlmc_ctx* c, int kind, int N) {
    for (size_t i = 0; i < c->stats.size(); ++i)
        if (c->stats[i].kind == kind && c->stats[i].N == N) return (int)i;
    c->stats.push_back(mlmc_kernel_stat{kind, N, 0, 0.0});
    return (int)c->stats.size() - 1;
}

cudaEvent_t take_event(mlmc_ctx* c) {
    if (!c->ev_pool.empty()) { cudaEvent_t e = c->ev_pool.back(); c->ev_pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

void drain_pending(mlmc_ctx* c) {
    for (auto& p : c->pending) {
        float ms = 0.f;
        if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess)
            c->stats[p.idx].ms += ms;
        c->ev_pool.push_back(p.a);
        c->ev_pool.push_back(p.b);
    }
    c->pending.clear();
}

// Launch through f(), counting it and (profiling on) timing it with events on its stream.
template <class F>
cudaError_t counted(mlmc_ctx* c, cudaStream_t st, int kind, int N, F&& f) {
    int idx = stat_index(c, kind, N);
    c->stats[idx].launches++;
    if (!c->prof_on) return f();
    cudaEvent_t a = take_event(c), b = take_event(c);
    cudaEventRecord(a, st);
    cudaError_t e = f();
    cudaEventRecord(b, st);
    c->pending.push_back({idx, a, b});
    if (c->pending.size() > 4096) drain_pending(c);
    return e;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Workspace layout for one pass of `batch` samples of `level`.
struct WsLayout {
    size_t xi, a_f, a_c, rec, chunks, ctr, keys_f, keys_c, ord_f, ord_c, esc_f, esc_c, gm, ch_f, ch_c, ch_f_bytes,
        ch_c_bytes, xc, total;
    int gm_ctas;
};
// Cholesky factor scratch of one solve (0 for MINRES / unsupported combinations)
size_t chol_bytes(const mlmc_precision* p, int N, uint64_t batch) {
    if (!p || p->solver != MLMC_SOLVER_CHOL_IR || N < 2) return 0;
    return chol_scratch_bytes(N, p->u_f, p->u_s, batch, p->u);
}
WsLayout ws_layout(const mlmc_ctx* c, int level, uint64_t batch, const mlmc_precision* pf = nullptr,
                   const mlmc_precision* pc = nullptr) {
    WsLayout L{};
    int Nf = level_N(c, level), Nc = level > 0 ? level_N(c, level - 1) : 0;
    size_t off = 0;
    L.xi = off;     off += align256(sizeof(double) * batch * c->pr.m);
    L.a_f = off;    off += align256(sizeof(double) * batch * 2 * (size_t)Nf * Nf);
    L.a_c = off;    off += align256(sizeof(double) * batch * 2 * (size_t)Nc * Nc);
    L.rec = off;    off += align256(sizeof(double) * batch * kRecLen);
    L.chunks = off; off += align256(sizeof(double) * (kSumsLen + kXLen) * ((batch + kChunk - 1) / kChunk + 1));
    L.ctr = off;    off += align256(sizeof(unsigned) * 32);   // job counters (0 / 4 fine / coarse, 8 / 12 escalation), 16 / 17 order
    // contrast keys and longest-first orders of the fine / coarse MINRES solves (order_kernel)
    L.keys_f = off; off += align256(sizeof(unsigned long long) * 2 * batch);
    L.keys_c = off; off += align256(sizeof(unsigned long long) * 2 * batch);
    L.ord_f = off;  off += align256(sizeof(int) * batch);
    L.ord_c = off;  off += align256(sizeof(int) * batch);
    // escalation lists of the fine / coarse solves: [count | indices]
    L.esc_f = off;  off += align256(sizeof(int) * (batch + 4));
    L.esc_c = off;  off += align256(sizeof(int) * (batch + 4));
    L.gm = off;
    L.gm_ctas = 0;
    if (Nf >= kGmMinN) {   // per-CTA scratch of the streamed-mesh solvers (fine and coarse share it)
        auto uses_mg = [](const mlmc_precision* p) {
            return p && (p->solver == MLMC_SOLVER_MGCG || (p->flags & MLMC_FLAG_ESCALATE));
        };
        const bool mg = uses_mg(pf) || uses_mg(pc);
        const int per_sm = mg ? mgcg_ctas_per_sm(Nf) : 1;
        L.gm_ctas = (int)std::min<uint64_t>(batch, (uint64_t)std::max(c->sms, 1) * per_sm);
        size_t per_cta = std::max(minres_gm_scratch_per_cta(Nf), minres_stream_scratch_per_cta(Nf));
        if (mg) per_cta = std::max(per_cta, mgcg_scratch_per_cta(Nf));
        off += align256(per_cta * L.gm_ctas);
    }
    // factor scratch of the Cholesky-IR solves (fine and coarse may run concurrently: two regions)
    L.ch_f_bytes = chol_bytes(pf, Nf, batch);
    L.ch_c_bytes = level > 0 ? chol_bytes(pc, Nc, batch) : 0;
    L.ch_f = off;   off += align256(L.ch_f_bytes);
    L.ch_c = off;   off += align256(L.ch_c_bytes);
    // coarse solutions of a coarse-to-fine pair (MLMC_FLAG_C2F): [batch][(Nc - 1)^2]
    L.xc = off;
    if (pf && (pf->flags & MLMC_FLAG_C2F) && level > 0) off += align256(sizeof(double) * batch * (size_t)(Nc - 1) * (Nc - 1));
    L.total = off;
    return L;
}

uint64_t max_batch(const mlmc_ctx* c, int level, size_t bytes, const mlmc_precision* pf = nullptr,
                   const mlmc_precision* pc = nullptr) {
    uint64_t lo = 0, hi = 1;
    while (ws_layout(c, level, hi, pf, pc).total <= bytes && hi < (1ull << 40)) { lo = hi; hi *= 2; }
    while (hi - lo > 1) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (ws_layout(c, level, mid, pf, pc).total <= bytes) lo = mid; else hi = mid;
    }
    return lo;
}

// Where one level's pipeline runs: a slice of the workspace and a stream.
struct Exec {
    unsigned char* ws;
    size_t bytes;
    cudaStream_t st;
};

// Optional scheduling of a single-pass level inside mlmc_sample_levels_async: the coarse solve
// forks onto st_c (fine and coarse solves are independent), `prep` is recorded once the fields
// are on HBM, and the solves wait for `gate` (the largest level's prep) so that the longest
// solve is the first one eligible for the SMs.
struct LevelSched {
    cudaStream_t st_c = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr, prep = nullptr, gate = nullptr;
};

// Scheduling knobs of the concurrent-levels step, for A/B runs of the tuning build only (MLMC_SCHED_GATE=0:
// no gate behind the largest level's fields; MLMC_SCHED_FORK=0: coarse halves after the fine ones on one
// stream; MLMC_SCHED_PRIO=0: every level stream at the same priority, =2: the largest level's coarse stream one
// step below its fine one).  The production build uses the defaults, which measured fastest on configs[1]
// (tools/gpu_call_r02ac.sh: 2.341 ms; no gate 2.472, no fork 2.376, flat priorities 2.379, coarse one step
// lower 2.348).
int sched_knob(const char* name) {
#ifdef MLMC_TUNING
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : 1;
#else
    (void)name;
    return 1;
#endif
}

// Which synthesis a mesh uses (a function of N, m and K only, so results never depend on the batch):
// the separable one (K1s) where the kernel supports the mesh and K, unless N = 8 and K > 16 (there the
// per-sample K x K gather outweighs the 2N^2 x m contraction: measured on configs[4] level 0), or where
// Phi would not be small (> 256 MB); the P x m one (K1) otherwise.  MLMC_FIELD_KERNEL=dense|ffma forces
// the P x m one, =sep the separable one wherever it is supported.
bool field_sep(const mlmc_ctx* ctx, int N) {
    if (field_use_dense()) return false;
    const int K = ctx->sep.K;
    if (!field_sep_supported(N, K)) return false;
    if (field_force_sep()) return true;
    const double phi_bytes = 8.0 * 2.0 * N * N * ctx->pr.m;
    return N >= 16 || K <= 16 || phi_bytes > 256.0 * (1 << 20);
}

// Plan data of a level's field synthesis, built on first use: the separable tables (a few KB per level)
// or the P x m matrix Phi (1.07 GB at h = 1/512, m = 256).
int ensure_phi(mlmc_ctx* ctx, int level) {
    const int N = level_N(ctx, level);
    if (!field_use_dense() && !ctx->sep_i) build_sep_modes(ctx->pr, ctx->kl, ctx->sep);
    if (field_sep(ctx, N)) {
        if (!ctx->sep_i) {
            const int m = ctx->pr.m, K = ctx->sep.K;
            std::vector<int32_t> kmap((size_t)K * K, -1);
            std::vector<double> cmap((size_t)K * K, 0.0);
            for (int a = 0; a < K; ++a)
                for (int c = ctx->sep.aoff[a]; c < ctx->sep.aoff[a + 1]; ++c) {
                    const size_t e = (size_t)a * K + ctx->sep.mb[c];
                    if (kmap[e] >= 0) return fail(ctx, MLMC_EINVAL, "two KL modes share a pair of 1D functions");
                    kmap[e] = ctx->sep.mk[c];
                    cmap[e] = ctx->sep.mc[c];
                }
            (void)m;
            CU(cudaMalloc(&ctx->sep_i, sizeof(int32_t) * kmap.size()));
            CU(cudaMemcpy(ctx->sep_i, kmap.data(), sizeof(int32_t) * kmap.size(), cudaMemcpyHostToDevice));
            CU(cudaMalloc(&ctx->sep_c, sizeof(double) * cmap.size()));
            CU(cudaMemcpy(ctx->sep_c, cmap.data(), sizeof(double) * cmap.size(), cudaMemcpyHostToDevice));
        }
        if (ctx->tab_dev[level]) return MLMC_OK;
        std::vector<double> tab;
        build_sep_tables(ctx->pr, ctx->kl, ctx->sep, N, tab);
        double* d = nullptr;
        CU(cudaMalloc(&d, tab.size() * sizeof(double)));
        CU(cudaMemcpy(d, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice));
        ctx->tab_dev[level] = d;
        return MLMC_OK;
    }
    if (ctx->phi_dev[level]) return MLMC_OK;
    std::vector<double> phi;
    build_phi(ctx->pr, ctx->kl, N, phi);
    double* d = nullptr;
    CU(cudaMalloc(&d, phi.size() * sizeof(double)));
    CU(cudaMemcpy(d, phi.data(), phi.size() * sizeof(double), cudaMemcpyHostToDevice));
    ctx->phi_dev[level] = d;
    return MLMC_OK;
}

// K1 + K2 of mesh level `mesh` for nb samples (xi -> a), on stream st
// (order / done: see launch_field_sep -- only on the separable path; the caller orders the P x m one itself)
cudaError_t field(const mlmc_ctx* ctx, int mesh, const double* xi, double* a, uint64_t nb, unsigned long long* keys,
                  cudaStream_t st, int* order = nullptr, unsigned* done = nullptr) {
    const int N = level_N(ctx, mesh), m = ctx->pr.m;
    if (!field_sep(ctx, N)) return launch_field(ctx->phi_dev[mesh], xi, a, 2 * N * N, m, nb, keys, st);
    return launch_field_sep(ctx->tab_dev[mesh], ctx->sep_i, ctx->sep_c, ctx->sep.K, xi, a, N, m, nb, keys, st, order,
                            done);
}

int check_prec(mlmc_ctx* ctx, const mlmc_precision* p, int N, double tol) {
    if (!p) return fail(ctx, MLMC_EINVAL, "precision is NULL");
    if (!(tol > 0.0) || !std::isfinite(tol)) return fail(ctx, MLMC_EINVAL, "tolerance must be > 0");
    if (p->solver == MLMC_SOLVER_MINRES) {
        if (!minres_supported(N)) return fail(ctx, MLMC_EINVAL, "MINRES kernel not built for N=" + std::to_string(N));
        if ((p->flags & MLMC_FLAG_VERIFY) && N >= kGmMinN)   // x_k is carried by the on-chip tile kernels only
            return fail(ctx, MLMC_EINVAL, "MLMC_FLAG_VERIFY needs h >= 1/64 (N <= 64), got N=" + std::to_string(N));
        return MLMC_OK;
    }
    if (p->solver == MLMC_SOLVER_MGCG) {
        if (!mgcg_supported(N)) return fail(ctx, MLMC_EINVAL, "MG-PCG kernel not built for N=" + std::to_string(N));
        return MLMC_OK;
    }
    if (p->solver == MLMC_SOLVER_CG) {
        if (!cg_supported(N)) return fail(ctx, MLMC_EINVAL, "CG kernel not built for N=" + std::to_string(N));
        return MLMC_OK;
    }
    if (p->solver == MLMC_SOLVER_CHOL_IR) {
        if (p->u != p->u_r || (p->u != MLMC_FMT_F64 && p->u != MLMC_FMT_F32 && p->u != MLMC_FMT_F16))
            return fail(ctx, MLMC_EINVAL, "IR supports u = u_r in binary64, binary32 or binary16");
        if (!chol_supported(N, p->u_f, p->u_s, p->u))
            return fail(ctx, MLMC_EINVAL, "Cholesky-IR (u_f, u_s) not supported for N=" + std::to_string(N));
        return MLMC_OK;
    }
    return fail(ctx, MLMC_EINVAL, "unknown solver");
}

double fmt_bits(int f) { return f == MLMC_FMT_F16 ? 16 : f == MLMC_FMT_F32 ? 32 : f == MLMC_FMT_E4M3 ? 8 : 64; }

// Cost model R5 of one solve on mesh N: fixed + step x iterations, in one commensurate unit across solvers --
// the device time of one MINRES node-step (one unknown, one MINRES iteration) on the same mesh class.  MINRES
// itself costs n per step: the paper's cost measure (PETSc FLOPs of MINRES, proportional to
// iterations x unknowns), so policy 0 is exactly the paper's model.  The other solvers' weights were measured
// once on B200 (round 1) and are frozen here, so a run's N_l decisions never depend on
// the box or on timing noise:
//   MG-PCG step       on chip (N <= 64): ~20 MINRES steps of the same system (profiles/r01p_cg_vs_minres.jsonl,
//                     DESIGN.md K3m); streamed (N >= 128): 162 vs 40 B per node-step at 2.56 vs 5.04 TB/s -> 8
//   CG step           1.5 (the MG kernel's layout, 1.2-2.9x slower passes than K3, profiles/r01p_*)
//   Cholesky-IR       factorisation 2.5 n bw (binary32 factor; 3.6 binary16 / E4M3, 5 binary64), each
//                     substitution pair + residual 0.7 n bw (K4 launch times of profiles/r01c_ncu_k4.md against
//                     the K3 node-step time at h = 1/32)
void cost_model(const mlmc_precision* p, int N, double& fixed, double& step) {
    const double n = (double)(N - 1) * (N - 1), bw = N - 1;
    if (p->solver == MLMC_SOLVER_MINRES) { fixed = 0.0; step = n; }
    else if (p->solver == MLMC_SOLVER_CG) { fixed = 0.0; step = 1.5 * n; }
    else if (p->solver == MLMC_SOLVER_MGCG) { const double w = N <= 64 ? 20.0 : 8.0; fixed = w * n; step = w * n; }
    else {
        const double cf = p->u_f == MLMC_FMT_F32 ? 2.5 : p->u_f == MLMC_FMT_F64 ? 5.0 : 3.6;
        fixed = (cf + 0.7) * n * bw;                   // factor + the initial solve x0
        step = 0.7 * n * bw;
    }
}

// cost of an escalated half (status 4): the failed attempt (run to its iteration cap) + MG-PCG's fixed part,
// then MG-PCG's per-step cost times the recorded MG-PCG steps
void escalation_cost(const mlmc_precision* p, int N, double& fixed, double& step) {
    double f0, s0;
    cost_model(p, N, f0, s0);
    const int n = (N - 1) * (N - 1);
    const double cap = p->max_iter > 0 ? p->max_iter : (p->solver == MLMC_SOLVER_CHOL_IR ? 50.0 : 16.0 * n + 1000.0);
    const mlmc_precision mg{MLMC_SOLVER_MGCG, MLMC_FMT_F64, MLMC_FMT_F64, MLMC_FMT_F64, MLMC_FMT_F64, 0, 0};
    double fm, sm;
    cost_model(&mg, N, fm, sm);
    fixed = f0 + s0 * cap + fm;
    step = sm;
}

// MLMC_MINRES_GM=1 selects the three-phase global-memory MINRES instead of the streamed one (A/B).
bool use_gm_kernel() {
#ifndef MLMC_TUNING
    return false;      // production build: K3c only
#endif
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("MLMC_MINRES_GM");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

// Longest-first job order for a MINRES solve (LPT scheduling of the persistent CTAs): worth it where
// a launch is a few waves of long solves (h >= 1/16: the tile and streamed kernels, nb <= kOrderMax).  MLMC_ORDER=0
// switches it off (A/B runs).  (h = 1/16 since round 2, kOrderMax 8192 for configs[1] level 1's 5000 systems: C2 step
// 2.339 / 2.342 / 2.341 vs 2.343 / 2.346 / 2.346 ms from h = 1/32 on, alternating runs; identical sums)
bool use_order(const mlmc_precision* p, int N, uint64_t nb) {
    static int env = -1;
    if (env < 0) {
        const char* e = std::getenv("MLMC_ORDER");
        env = (e && e[0] == '0') ? 0 : 1;
    }
    int min_n = kOrderMinN;
#ifdef MLMC_TUNING
    static int env_n = -1;
    if (env_n < 0) {
        const char* e = std::getenv("MLMC_ORDER_MIN_N");
        env_n = e ? std::atoi(e) : kOrderMinN;
    }
    min_n = env_n;
#endif
    if (!env || p->solver != MLMC_SOLVER_MINRES || N < min_n || nb < 2 || nb > (uint64_t)kOrderMax) return false;
    if (N >= kGmMinN) return minres_stream_supported(N) && !use_gm_kernel();   // streamed kernel (K3c)
    return minres_tile_variant(N) >= 0;
}


int solve_mesh(mlmc_ctx* ctx, const Exec& ex, int N, const mlmc_precision* p, double tol, const double* a, uint64_t nb,
               double* rec, int slot, unsigned* ctr, double* gm_scratch, int gm_ctas, void* ch_scratch,
               size_t ch_bytes, const unsigned long long* keys = nullptr, int* order = nullptr, int* esc = nullptr,
               int xmode = 0, double* xio = nullptr) {
    int n = (N - 1) * (N - 1);
    if (p->solver == MLMC_SOLVER_MINRES) {
        int mi = p->max_iter > 0 ? p->max_iter : 16 * n + 1000;   // finite-precision Lanczos at contrast ~1e7 (Eq. (20), sigma = 2) needs > n
        bool verify = (p->flags & MLMC_FLAG_VERIFY) != 0;
        // (the longest-first order, `order`, is formed by run_level right after the fields)
        if (N >= kGmMinN && minres_cluster_supported(N) && !use_gm_kernel())
            CU(counted(ctx, ex.st, MLMC_K_MINRES, N, [&] {
                return launch_minres_cluster(N, a, nb, tol, mi, rec, slot, ctr, keys ? order : nullptr, ex.st);
            }));
        else if (N >= kGmMinN && minres_stream_supported(N) && !use_gm_kernel())
            CU(counted(ctx, ex.st, MLMC_K_MINRES, N, [&] {
                return launch_minres_stream(N, a, nb, tol, mi, rec, slot, ctr, gm_scratch, gm_ctas, ex.st,
                                            keys ? order : nullptr);
            }));
        else if (N >= kGmMinN)
            CU(counted(ctx, ex.st, MLMC_K_MINRES, N, [&] {
                return launch_minres_gm(N, a, nb, tol, mi, rec, slot, ctr, gm_scratch, gm_ctas, ex.st);
            }));
        else
            CU(counted(ctx, ex.st, MLMC_K_MINRES, N,
                       [&] {
                           return launch_minres(N, a, nb, tol, mi, rec, slot, ctr, verify, keys ? order : nullptr, ex.st,
                                                xmode, xio);
                       }));

    } else if (p->solver == MLMC_SOLVER_CG) {
        int mi = p->max_iter > 0 ? p->max_iter : 16 * n + 1000;
        CU(counted(ctx, ex.st, MLMC_K_MINRES, N,
                   [&] { return launch_cg(N, a, nb, tol, mi, rec, slot, ctr, nullptr, ex.st); }));
    } else if (p->solver == MLMC_SOLVER_MGCG) {
        int mi = p->max_iter > 0 ? p->max_iter : 1000;
        CU(counted(ctx, ex.st, MLMC_K_MINRES, N,
                   [&] { return launch_mgcg(N, a, nb, tol, mi, rec, slot, ctr, nullptr, gm_scratch, gm_ctas, ex.st); }));
    } else {
        int mi = p->max_iter > 0 ? p->max_iter : 50;
        CU(counted(ctx, ex.st, MLMC_K_CHOL_IR, N,
                   [&] {
                       return launch_chol_ir(N, a, nb, p->u_f, p->u_s, tol, mi, rec, slot, ctr, ch_scratch, ch_bytes,
                                             ex.st, p->u);
                   }));
    }
    // escalation (on_fail = 2): the failed MINRES / Cholesky-IR solves of this launch (max_iter,
    // breakdown, limiting accuracy) are solved again by MG-PCG to the same tolerance; converged ones are
    // recorded with status 4 and counted apart
    if (p->solver != MLMC_SOLVER_MGCG && (p->flags & MLMC_FLAG_ESCALATE) && esc && mgcg_supported(N)) {
        CU(cudaMemsetAsync(esc, 0, sizeof(int), ex.st));
        CU(launch_escalate_collect(rec, nb, slot, esc + 4, esc, ex.st));
        CU(counted(ctx, ex.st, MLMC_K_MINRES, N, [&] {
            return launch_mgcg(N, a, nb, tol, 1000, rec, slot, ctr + 8, esc + 4, gm_scratch, gm_ctas, ex.st, esc, 4);
        }));
    }
    return MLMC_OK;
}

int validate_level(mlmc_ctx* ctx, int level, const mlmc_precision* pf, const mlmc_precision* pc, double tol_f,
                   double tol_c) {
    if (level < 0 || level > ctx->pr.L_max) return fail(ctx, MLMC_EINVAL, "level out of range");
    const int Nf = level_N(ctx, level), Nc = level > 0 ? level_N(ctx, level - 1) : 0;
    int rc = check_prec(ctx, pf, Nf, tol_f);
    if (rc) return rc;
    if (level > 0 && (rc = check_prec(ctx, pc, Nc, tol_c))) return rc;
    if ((rc = ensure_phi(ctx, level))) return rc;
    if (level > 0 && (rc = ensure_phi(ctx, level - 1))) return rc;
    if (pf->flags & MLMC_FLAG_C2F) {   // coarse-to-fine initial guess: both halves MINRES on tile meshes
        if (level == 0 || pf->solver != MLMC_SOLVER_MINRES || !pc || pc->solver != MLMC_SOLVER_MINRES ||
            !(Nf == 16 || Nf == 32 || Nf == 64) || minres_tile_variant(Nf) < 0 || minres_tile_variant(Nc) < 0)
            return fail(ctx, MLMC_EINVAL, "MLMC_FLAG_C2F needs level >= 1, MINRES on both halves and h = 1/16..1/64");
    }
    return MLMC_OK;
}

// One level's pipeline (K0 -> K1 -> K3/K4 fine + coarse -> K5) in passes that fit ex.ws, on ex.st.
int run_level(mlmc_ctx* ctx, const Exec& ex, int level, uint64_t n, uint64_t seed, uint64_t first_index,
              const mlmc_precision* pf, const mlmc_precision* pc, double tol_f, double tol_c, double* sums_dev,
              double* per_sample, bool per_sample_is_dev, const double* xi_in, bool xi_in_is_dev,
              const LevelSched* sch = nullptr, unsigned long long* xsums = nullptr) {
    const int Nf = level_N(ctx, level), Nc = level > 0 ? level_N(ctx, level - 1) : 0;
    uint64_t B = max_batch(ctx, level, ex.bytes, pf, pc);
    if (B == 0 && n > 0) return fail(ctx, MLMC_ENOMEM, "workspace too small for one sample");
    // passes made of whole 4096-sample chunks: the chunked sums then do not depend on the pass size
    if (B > kChunk && B < n) B = (B / kChunk) * kChunk;
    const WsLayout L = ws_layout(ctx, level, std::max<uint64_t>(B, 1), pf, pc);
    double* xi = reinterpret_cast<double*>(ex.ws + L.xi);
    double* af = reinterpret_cast<double*>(ex.ws + L.a_f);
    double* ac = reinterpret_cast<double*>(ex.ws + L.a_c);
    double* rec = reinterpret_cast<double*>(ex.ws + L.rec);
    double* chunks = reinterpret_cast<double*>(ex.ws + L.chunks);
    unsigned* ctr = reinterpret_cast<unsigned*>(ex.ws + L.ctr);
    double* gm = reinterpret_cast<double*>(ex.ws + L.gm);
    CostParams cp{};
    cost_model(pf, Nf, cp.f_fixed, cp.f_step);
    escalation_cost(pf, Nf, cp.f_esc, cp.f_esc_step);
    if (level > 0) {
        cost_model(pc, Nc, cp.c_fixed, cp.c_step);
        escalation_cost(pc, Nc, cp.c_esc, cp.c_esc_step);
    }
    const int m = ctx->pr.m;
    const cudaStream_t st = ex.st;
    int rc;
    CU(cudaMemsetAsync(sums_dev, 0, sizeof(double) * kSumsLen, st));
    if (xsums) CU(cudaMemsetAsync(xsums, 0, sizeof(unsigned long long) * kXLen, st));
    struct NvtxRange {   // Nsight / NVTX range of the level's passes (a no-op without a tool attached)
        explicit NvtxRange(int l) { char b[48]; std::snprintf(b, sizeof(b), "mlmc level %d", l); nvtxRangePushA(b); }
        ~NvtxRange() { nvtxRangePop(); }
    } nvtx_range(level);
    for (uint64_t done = 0; done < n;) {
        const uint64_t nb = std::min<uint64_t>(B, n - done);
        CU(cudaMemsetAsync(ctr, 0, sizeof(unsigned) * 32, st));
        if (xi_in) {
            CU(cudaMemcpyAsync(xi, xi_in + done * m, sizeof(double) * m * nb,
                               xi_in_is_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
        } else {
            CU(counted(ctx, st, MLMC_K_RNG, 0,
                       [&] { return launch_rng(xi, m, nb, seed, level, first_index + done, st); }));
        }
        const bool ord_f = use_order(pf, Nf, nb), ord_c = level > 0 && use_order(pc, Nc, nb);
        unsigned long long* kf = ord_f ? reinterpret_cast<unsigned long long*>(ex.ws + L.keys_f) : nullptr;
        unsigned long long* kc = ord_c ? reinterpret_cast<unsigned long long*>(ex.ws + L.keys_c) : nullptr;
        if (kf) CU(cudaMemsetAsync(kf, 0, sizeof(unsigned long long) * 2 * nb, st));
        if (kc) CU(cudaMemsetAsync(kc, 0, sizeof(unsigned long long) * 2 * nb, st));
        int* of = reinterpret_cast<int*>(ex.ws + L.ord_f);
        int* oc = reinterpret_cast<int*>(ex.ws + L.ord_c);
        // longest-first orders with the fields: on the separable path the field kernel's last CTA forms the order
        // (ctr[16], ctr[17] count the CTAs done); otherwise one order kernel right after the field, before the
        // gate.  A separate one-CTA kernel that waits for a whole free SM sat behind the other levels' solves
        // (the job trace showed level 2's fine solves starting only at 1.86 ms of a 2.4 ms step).
        const bool fuse_f = kf && field_sep(ctx, Nf), fuse_c = kc && field_sep(ctx, Nc);
        CU(counted(ctx, st, MLMC_K_FIELD, Nf, [&] {
            return field(ctx, level, xi, af, nb, kf, st, fuse_f ? of : nullptr, fuse_f ? ctr + 16 : nullptr);
        }));
        if (level > 0)
            CU(counted(ctx, st, MLMC_K_FIELD, Nc, [&] {
                return field(ctx, level - 1, xi, ac, nb, kc, st, fuse_c ? oc : nullptr, fuse_c ? ctr + 17 : nullptr);
            }));
        if (kf && !fuse_f) CU(counted(ctx, st, MLMC_K_ORDER, Nf, [&] { return launch_order(kf, (int)nb, of, st); }));
        if (kc && !fuse_c) CU(counted(ctx, st, MLMC_K_ORDER, Nc, [&] { return launch_order(kc, (int)nb, oc, st); }));
        if (level == 0) CU(cudaMemsetAsync(rec, 0, sizeof(double) * kRecLen * nb, st));
        const bool sched = sch && nb == n;               // single pass only
        if (sched && sch->prep) CU(cudaEventRecord(sch->prep, st));
        if (sched && sch->gate) CU(cudaStreamWaitEvent(st, sch->gate, 0));
        // the global-memory MINRES shares one scratch between the fine and coarse solves: no fork then; a
        // coarse-to-fine pair (MLMC_FLAG_C2F) runs the coarse half first, the fine half from its solution
        const bool c2f = level > 0 && (pf->flags & MLMC_FLAG_C2F);
        double* xc = reinterpret_cast<double*>(ex.ws + L.xc);
        // (the fork is per pass: the join below orders the next pass's field writes after this coarse solve);
        // with per-kernel profiling on, the solves stay serialised so that every launch's event time is its own
        // (K3b keeps its system on chip, so a fine half on it may fork as well -- its coarse half then runs on the
        // SMs its clusters leave free -- unless that coarse half uses the shared scratch: configs[4] level 4 pass
        // 24.1 -> 21.4 ms, level 5 329 -> 308 ms for 148 samples, tools/fork_probe.py)
        const auto on_chip = [&](int Nm, const mlmc_precision* pm) {
            return Nm < kGmMinN || (pm->solver == MLMC_SOLVER_MINRES && minres_cluster_supported(Nm) && !use_gm_kernel());
        };
        const bool fork = sch && level > 0 && sch->st_c && on_chip(Nf, pf) && on_chip(Nc, pc) && !c2f && !ctx->prof_on &&
                          sched_knob("MLMC_SCHED_FORK");
        if (fork) {
            CU(cudaEventRecord(sch->fork, st));
            CU(cudaStreamWaitEvent(sch->st_c, sch->fork, 0));
        }
        void* chf = ex.ws + L.ch_f;
        void* chc = ex.ws + L.ch_c;
        int* ef = reinterpret_cast<int*>(ex.ws + L.esc_f);
        int* ec = reinterpret_cast<int*>(ex.ws + L.esc_c);
        if (c2f) {
            if ((rc = solve_mesh(ctx, ex, Nc, pc, tol_c, ac, nb, rec, 1, ctr + 4, gm, L.gm_ctas, chc, L.ch_c_bytes, kc,
                                 oc, ec, 1, xc)))
                return rc;
            if ((rc = solve_mesh(ctx, ex, Nf, pf, tol_f, af, nb, rec, 0, ctr, gm, L.gm_ctas, chf, L.ch_f_bytes, kf, of,
                                 ef, 2, xc)))
                return rc;
        } else if ((rc = solve_mesh(ctx, ex, Nf, pf, tol_f, af, nb, rec, 0, ctr, gm, L.gm_ctas, chf, L.ch_f_bytes, kf,
                                    of, ef)))
            return rc;
        if (fork) {
            const Exec exc{ex.ws, ex.bytes, sch->st_c};
            if ((rc = solve_mesh(ctx, exc, Nc, pc, tol_c, ac, nb, rec, 1, ctr + 4, gm, L.gm_ctas, chc, L.ch_c_bytes, kc,
                                 oc, ec)))
                return rc;
            CU(cudaEventRecord(sch->join, sch->st_c));
            CU(cudaStreamWaitEvent(st, sch->join, 0));
        } else if (level > 0 && !c2f && (rc = solve_mesh(ctx, ex, Nc, pc, tol_c, ac, nb, rec, 1, ctr + 4, gm,
                                                         L.gm_ctas, chc, L.ch_c_bytes, kc, oc, ec))) {
            return rc;
        }
        CU(counted(ctx, st, MLMC_K_SUMS, Nf, [&] {
            return launch_level_sums(rec, nb, level, cp, chunks, sums_dev, true, st, xsums);
        }));
        if (per_sample) {
            double* dst = per_sample + done * kRecLen;
            CU(cudaMemcpyAsync(dst, rec, sizeof(double) * kRecLen * nb,
                               per_sample_is_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
        }
        done += nb;
    }
    return MLMC_OK;
}

int sample_level_impl(mlmc_ctx* ctx, int level, uint64_t n, uint64_t seed, uint64_t first_index,
                      const mlmc_precision* pf, const mlmc_precision* pc, double tol_f, double tol_c, double* sums_dev,
                      double* per_sample, bool per_sample_is_dev, const double* xi_in = nullptr,
                      bool xi_in_is_dev = false) {
    if (!ctx) return MLMC_EINVAL;
    int rc = validate_level(ctx, level, pf, pc, tol_f, tol_c);
    if (rc) return rc;
    if (!ctx->ws) return fail(ctx, MLMC_ENOMEM, "no workspace bound");
    // the fine and coarse solves of a pass are independent: the coarse one runs on a forked stream
    LevelSched sch;
    sch.st_c = ctx->single_c;
    sch.fork = ctx->single_fork;
    sch.join = ctx->single_join;
    return run_level(ctx, Exec{ctx->ws, ctx->ws_bytes, ctx->stream}, level, n, seed, first_index, pf, pc, tol_f, tol_c,
                     sums_dev, per_sample, per_sample_is_dev, xi_in, xi_in_is_dev, &sch,
                     ctx->want_xsums ? ctx->xsums_dev : nullptr);
}

}  // namespace

void mlmc::ctx_note_auto_choice(mlmc_ctx* ctx, int N, int cls, const mlmc_precision& p, double ms_per_sample) {
    for (auto& e : ctx->auto_choice)
        if (e.N == N && e.cls == cls) { e.p = p; e.ms = ms_per_sample; return; }
    ctx->auto_choice.push_back({N, cls, p, ms_per_sample});
}

bool mlmc::ctx_find_auto_choice(const mlmc_ctx* ctx, int N, int cls, mlmc_precision* p) {
    for (const auto& e : ctx->auto_choice)
        if (e.N == N && e.cls == cls) { *p = e.p; return true; }
    return false;
}

int mlmc::copy_sums_to_host(mlmc_ctx* ctx, const double* dev, int nlev, double* host) {
    CU(cudaMemcpyAsync(host, dev, sizeof(double) * kSumsLen * nlev, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return MLMC_OK;
}

void mlmc::ctx_want_xsums(mlmc_ctx* ctx, bool on) { ctx->want_xsums = on; }
double* mlmc::ctx_adaptive_sums(mlmc_ctx* ctx) { return ctx->adapt_dev; }

int mlmc::copy_xsums_to_host(mlmc_ctx* ctx, int nlev, unsigned long long* host) {
    CU(cudaMemcpyAsync(host, ctx->xsums_dev, sizeof(unsigned long long) * kXLen * nlev, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return MLMC_OK;
}

namespace {

bool is_device_ptr(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace

extern "C" {

const char* mlmc_strerror(int code) {
    switch (code) {
        case MLMC_OK: return "ok";
        case MLMC_EINVAL: return "invalid argument";
        case MLMC_ESOLVER: return "solver failure";
        case MLMC_ELMAX: return "L_max reached with the bias test failing";
        case MLMC_ECUDA: return "CUDA error";
        case MLMC_ENOMEM: return "insufficient workspace / memory";
        default: return "unknown error";
    }
}

const char* mlmc_last_error(const mlmc_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

int mlmc_plan_levels(const mlmc_problem* problem, mlmc_ctx** out) {
    mlmc_ctx* ctx = nullptr;
    if (!problem || !out) return fail(nullptr, MLMC_EINVAL, "NULL argument");
    const mlmc_problem& p = *problem;
    if (p.field != MLMC_FIELD_EXPCOV_KL && p.field != MLMC_FIELD_PAPER_EQ20) return fail(nullptr, MLMC_EINVAL, "bad field");
    if (p.m < 1 || p.m > 1024) return fail(nullptr, MLMC_EINVAL, "m out of range");
    if (p.refine != 2) return fail(nullptr, MLMC_EINVAL, "only refine = 2 is supported");
    if (p.h0_inv < 2 || p.L_max < 0 || p.L_max >= MLMC_MAX_LEVELS || ((long)p.h0_inv << p.L_max) > 512)
        return fail(nullptr, MLMC_EINVAL, "mesh hierarchy out of range (h0_inv * 2^L_max <= 512)");
    if (!(p.sigma2 > 0.0)) return fail(nullptr, MLMC_EINVAL, "sigma2 must be > 0");
    if (p.field == MLMC_FIELD_EXPCOV_KL && !(p.corr_len > 0.0)) return fail(nullptr, MLMC_EINVAL, "corr_len must be > 0");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(nullptr, MLMC_ECUDA, "no CUDA device");
    }
    if (p.device < 0 || p.device >= ndev) return fail(nullptr, MLMC_EINVAL, "bad device ordinal");
    ctx = new mlmc_ctx();
    ctx->pr = p;
    ctx->device = p.device;
    if (p.field == MLMC_FIELD_EXPCOV_KL) {
        int rc = kl_modes(p.sigma2, p.corr_len, p.m, ctx->kl);
        if (rc) { delete ctx; return fail(nullptr, rc, "KL eigenpairs failed"); }
    }
    ctx->phi_dev.assign(p.L_max + 1, nullptr);
    ctx->tab_dev.assign(p.L_max + 1, nullptr);
    cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, p.device);
    cudaError_t e = cudaSetDevice(p.device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->sums_dev, sizeof(double) * kSumsLen * MLMC_MAX_LEVELS);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->xsums_dev, sizeof(unsigned long long) * kXLen * MLMC_MAX_LEVELS);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->adapt_dev, sizeof(double) * kSumsLen * MLMC_MAX_LEVELS);
    if (e == cudaSuccess) {   // the coarse-solve stream of single-level calls, created here, not in a timed call
        int least = 0, greatest = 0;
        cudaDeviceGetStreamPriorityRange(&least, &greatest);
        e = cudaStreamCreateWithPriority(&ctx->single_c, cudaStreamNonBlocking, least);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->single_fork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->single_join, cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        std::string msg = cudaGetErrorString(e);
        mlmc_destroy(ctx);
        return fail(nullptr, MLMC_ECUDA, msg);
    }
    ctx->stream = ctx->own_stream;
    *out = ctx;
    return MLMC_OK;
}

void mlmc_destroy(mlmc_ctx* ctx) {
    if (!ctx) return;
    cudaStreamSynchronize(ctx->stream);
    for (cudaStream_t s : ctx->aux) { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
    for (cudaStream_t s : ctx->aux_c) { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
    for (auto* v : {&ctx->cfork_ev, &ctx->cjoin_ev, &ctx->prep_ev})
        for (cudaEvent_t e : *v) cudaEventDestroy(e);
    for (cudaEvent_t e : ctx->join_ev) cudaEventDestroy(e);
    if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
    drain_pending(ctx);
    for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
    for (double* d : ctx->phi_dev) if (d) cudaFree(d);
    for (double* d : ctx->tab_dev) if (d) cudaFree(d);
    if (ctx->sep_i) cudaFree(ctx->sep_i);
    if (ctx->sep_c) cudaFree(ctx->sep_c);
    if (ctx->sums_dev) cudaFree(ctx->sums_dev);
    if (ctx->xsums_dev) cudaFree(ctx->xsums_dev);
    if (ctx->adapt_dev) cudaFree(ctx->adapt_dev);
    if (ctx->single_c) { cudaStreamSynchronize(ctx->single_c); cudaStreamDestroy(ctx->single_c); }
    if (ctx->single_fork) cudaEventDestroy(ctx->single_fork);
    if (ctx->single_join) cudaEventDestroy(ctx->single_join);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

int mlmc_level_info_get(const mlmc_ctx* ctx, int level, mlmc_level_info* out) {
    if (!ctx || !out || level < 0 || level > ctx->pr.L_max) return MLMC_EINVAL;
    int N = level_N(ctx, level);
    out->N = N; out->n = (N - 1) * (N - 1); out->P = 2 * N * N; out->bw = N - 1; out->h = 1.0 / N;
    return MLMC_OK;
}

int mlmc_workspace_bytes(const mlmc_ctx* ctx, int level, uint64_t batch, size_t* out) {
    if (!ctx || !out || level < 0 || level > ctx->pr.L_max) return MLMC_EINVAL;
    *out = ws_layout(ctx, level, std::max<uint64_t>(batch, 1)).total;
    return MLMC_OK;
}

int mlmc_workspace_bytes_prec(const mlmc_ctx* ctx, int level, uint64_t batch, const mlmc_precision* prec_fine,
                              const mlmc_precision* prec_coarse, size_t* out) {
    if (!ctx || !out || level < 0 || level > ctx->pr.L_max) return MLMC_EINVAL;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return MLMC_ECUDA;
    *out = ws_layout(ctx, level, std::max<uint64_t>(batch, 1), prec_fine, prec_coarse).total;
    return MLMC_OK;
}

int mlmc_bind_workspace(mlmc_ctx* ctx, void* dev_ptr, size_t bytes, void* cuda_stream) {
    if (!ctx) return MLMC_EINVAL;
    if (!dev_ptr || (reinterpret_cast<uintptr_t>(dev_ptr) & 255)) return fail(ctx, MLMC_EINVAL, "workspace NULL or not 256-byte aligned");
    ctx->ws = static_cast<unsigned char*>(dev_ptr);
    ctx->ws_bytes = bytes;
    ctx->stream = static_cast<cudaStream_t>(cuda_stream);   // NULL = the legacy default stream
    return MLMC_OK;
}

int mlmc_sample_level_async(mlmc_ctx* ctx, int level, uint64_t n, uint64_t seed, uint64_t first_index,
                            const mlmc_precision* prec_fine, const mlmc_precision* prec_coarse, double tol_fine,
                            double tol_coarse, double* sums_dev, double* per_sample_dev) {
    if (!ctx || !sums_dev) return fail(ctx, MLMC_EINVAL, "NULL argument");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, MLMC_ECUDA, "cudaSetDevice");
    return sample_level_impl(ctx, level, n, seed, first_index, prec_fine, prec_coarse, tol_fine, tol_coarse, sums_dev,
                             per_sample_dev, true);
}

int mlmc_sample_level(mlmc_ctx* ctx, int level, uint64_t n, uint64_t seed, uint64_t first_index,
                      const mlmc_precision* prec_fine, const mlmc_precision* prec_coarse, double tol_fine,
                      double tol_coarse, mlmc_level_sums* out_sums, double* per_sample) {
    if (!ctx || !out_sums) return fail(ctx, MLMC_EINVAL, "NULL argument");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, MLMC_ECUDA, "cudaSetDevice");
    bool dev = per_sample ? is_device_ptr(per_sample) : false;
    int rc = sample_level_impl(ctx, level, n, seed, first_index, prec_fine, prec_coarse, tol_fine, tol_coarse,
                               ctx->sums_dev, per_sample, dev);
    if (rc) return rc;
    CU(cudaMemcpyAsync(out_sums, ctx->sums_dev, sizeof(double) * kSumsLen, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return MLMC_OK;
}

}  // extern "C"

namespace {

// Several levels concurrently (shared by mlmc_sample_levels_async and mlmc_sample_levels_xi): xi_in[q]
// (optional, host or device) replaces the Philox draw of entry q, per_sample[q] (optional, host or
// device) receives its records.
int sample_levels_impl(mlmc_ctx* ctx, int nlev, const int* levels, const uint64_t* n, uint64_t seed,
                       const uint64_t* first_index, const mlmc_precision* prec_fine, const mlmc_precision* prec_coarse,
                       const double* tol_fine, const double* tol_coarse, double* sums_dev,
                       const double* const* xi_in = nullptr, double* const* per_sample = nullptr) {
    if (!ctx || nlev < 1 || nlev > MLMC_MAX_LEVELS || !levels || !n || !first_index || !prec_fine || !prec_coarse ||
        !tol_fine || !tol_coarse || !sums_dev)
        return fail(ctx, MLMC_EINVAL, "NULL / bad argument");
    if (!ctx->ws) return fail(ctx, MLMC_ENOMEM, "no workspace bound");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, MLMC_ECUDA, "cudaSetDevice");
    for (int q = 0; q < nlev; ++q) {
        int rc = validate_level(ctx, levels[q], &prec_fine[q], &prec_coarse[q], tol_fine[q], tol_coarse[q]);
        if (rc) return rc;
    }
    // largest work first (proxy: samples x unknowns x N, i.e. ~ iterations x unknowns)
    std::vector<int> order(nlev);
    std::vector<double> cost(nlev);
    for (int q = 0; q < nlev; ++q) {
        order[q] = q;
        const double N = (double)level_N(ctx, levels[q]);
        cost[q] = (double)n[q] * (N - 1) * (N - 1) * N;
    }
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
    // workspace slices: each level's single-pass need if everything fits, else proportional
    std::vector<size_t> need(nlev);
    size_t total = 0;
    for (int q = 0; q < nlev; ++q) {
        need[q] = ws_layout(ctx, levels[q], std::max<uint64_t>(n[q], 1), &prec_fine[q], &prec_coarse[q]).total;
        total += need[q];
    }
    std::vector<size_t> slice(nlev);
    for (int q = 0; q < nlev; ++q)
        slice[q] = total <= ctx->ws_bytes ? need[q]
                                          : (size_t)((double)ctx->ws_bytes * ((double)need[q] / (double)total)) & ~(size_t)255;
    // streams: one per level, highest priority for the largest level
    if ((int)ctx->aux.size() < nlev) {
        int least = 0, greatest = 0;
        cudaDeviceGetStreamPriorityRange(&least, &greatest);
        while ((int)ctx->aux.size() < nlev) {
            const int k = (int)ctx->aux.size();
            const int pk = sched_knob("MLMC_SCHED_PRIO");
            int prio = pk ? std::max(greatest, least - (least - greatest) * (MLMC_MAX_LEVELS - k) / MLMC_MAX_LEVELS)
                          : greatest;
            // (tuning: =3 the two largest levels on top, =4 by size, =5 the small levels above the middle ones:
            // C2 step 2.40 / 2.41 / 2.41 vs 2.37 ms default on the same box; B200 has 4 priorities, 0 .. -3)
            if (pk == 3 && k == 1) prio = greatest;
            if (pk == 4 && k >= 1) prio = std::min(least, greatest + k);
            if (pk == 5 && k >= 1) prio = std::min(least, greatest + 1 + (MLMC_MAX_LEVELS - k) % 3);
            // (tuning: =6 the two smallest of four levels on top, then the largest, then the second: C2 step 2.38 with
            // the gate, 2.42-2.43 without, vs 2.35 ms default on the same box)
            if (pk == 6) prio = k >= 2 ? greatest : std::min(least, greatest + 1 + k);
            cudaStream_t s;
            CU(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, k == 0 && pk != 6 ? greatest : prio));
            ctx->aux.push_back(s);
            const int prio_c = k == 0 && sched_knob("MLMC_SCHED_PRIO") == 2 ? std::min(least, greatest + 1) : prio;
            CU(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking,
                                            k == 0 && prio_c == prio && pk != 6 ? greatest : prio_c));
            ctx->aux_c.push_back(s);
            cudaEvent_t e;
            CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ctx->join_ev.push_back(e);
            for (auto* v : {&ctx->cfork_ev, &ctx->cjoin_ev, &ctx->prep_ev}) {
                CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                v->push_back(e);
            }
        }
        if (!ctx->fork_ev) CU(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
    }
    CU(cudaEventRecord(ctx->fork_ev, ctx->stream));
    size_t off = 0;
    std::vector<size_t> offs(nlev);
    for (int q = 0; q < nlev; ++q) { offs[q] = off; off += slice[q]; }
    for (int k = 0; k < nlev; ++k) {
        const int q = order[k];
        cudaStream_t st = ctx->aux[k];
        CU(cudaStreamWaitEvent(st, ctx->fork_ev, 0));
        LevelSched sch;
        sch.st_c = ctx->aux_c[k];
        sch.fork = ctx->cfork_ev[k];
        sch.join = ctx->cjoin_ev[k];
        sch.prep = k == 0 && sched_knob("MLMC_SCHED_GATE") ? ctx->prep_ev[0] : nullptr;
        sch.gate = k == 0 || !sched_knob("MLMC_SCHED_GATE") ? nullptr : ctx->prep_ev[0];
        const bool top_single =
            max_batch(ctx, levels[order[0]], slice[order[0]], &prec_fine[order[0]], &prec_coarse[order[0]]) >= n[order[0]];
        if (!top_single) sch.prep = sch.gate = nullptr;   // the largest level runs in passes: no gate
        const double* xq = xi_in ? xi_in[q] : nullptr;
        double* pq = per_sample ? per_sample[q] : nullptr;
        int rc = run_level(ctx, Exec{ctx->ws + offs[q], slice[q], st}, levels[q], n[q], seed, first_index[q],
                           &prec_fine[q], &prec_coarse[q], tol_fine[q], tol_coarse[q], sums_dev + (size_t)q * kSumsLen,
                           pq, pq && is_device_ptr(pq), xq, xq && is_device_ptr(xq), &sch,
                           ctx->want_xsums ? ctx->xsums_dev + (size_t)q * kXLen : nullptr);
        if (rc) return rc;
        CU(cudaEventRecord(ctx->join_ev[k], st));
    }
    for (int k = 0; k < nlev; ++k) CU(cudaStreamWaitEvent(ctx->stream, ctx->join_ev[k], 0));
    return MLMC_OK;
}

}  // namespace

extern "C" {

int mlmc_sample_levels_async(mlmc_ctx* ctx, int nlev, const int* levels, const uint64_t* n, uint64_t seed,
                             const uint64_t* first_index, const mlmc_precision* prec_fine,
                             const mlmc_precision* prec_coarse, const double* tol_fine, const double* tol_coarse,
                             double* sums_dev) {
    return sample_levels_impl(ctx, nlev, levels, n, seed, first_index, prec_fine, prec_coarse, tol_fine, tol_coarse,
                              sums_dev);
}

int mlmc_sample_levels_xi(mlmc_ctx* ctx, int nlev, const int* levels, const uint64_t* n, const double* const* xi,
                          const mlmc_precision* prec_fine, const mlmc_precision* prec_coarse, const double* tol_fine,
                          const double* tol_coarse, mlmc_level_sums* out_sums, double* const* per_sample) {
    if (!ctx || !xi || !out_sums || nlev < 1 || nlev > MLMC_MAX_LEVELS) return fail(ctx, MLMC_EINVAL, "NULL / bad argument");
    for (int q = 0; q < nlev; ++q)
        if (!xi[q] && n && n[q] > 0) return fail(ctx, MLMC_EINVAL, "xi[q] is NULL");
    std::vector<uint64_t> first(nlev, 0);
    int rc = sample_levels_impl(ctx, nlev, levels, n, 0, first.data(), prec_fine, prec_coarse, tol_fine, tol_coarse,
                                ctx->sums_dev, xi, per_sample);
    if (rc) return rc;
    CU(cudaMemcpyAsync(out_sums, ctx->sums_dev, sizeof(double) * kSumsLen * nlev, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return MLMC_OK;
}

int mlmc_sample_level_xi(mlmc_ctx* ctx, int level, uint64_t n, const double* xi, const mlmc_precision* prec_fine,
                         const mlmc_precision* prec_coarse, double tol_fine, double tol_coarse, mlmc_level_sums* out_sums,
                         double* per_sample) {
    if (!ctx || !out_sums || (!xi && n > 0)) return fail(ctx, MLMC_EINVAL, "NULL argument");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, MLMC_ECUDA, "cudaSetDevice");
    bool dev = per_sample ? is_device_ptr(per_sample) : false;
    bool xdev = xi ? is_device_ptr(xi) : false;
    int rc = sample_level_impl(ctx, level, n, 0, 0, prec_fine, prec_coarse, tol_fine, tol_coarse, ctx->sums_dev,
                               per_sample, dev, xi, xdev);
    if (rc) return rc;
    CU(cudaMemcpyAsync(out_sums, ctx->sums_dev, sizeof(double) * kSumsLen, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return MLMC_OK;
}

int mlmc_auto_choice(const mlmc_ctx* ctx, int N, mlmc_precision* out, double* ms_per_sample) {
    if (!ctx || !out) return MLMC_EINVAL;
    for (auto it = ctx->auto_choice.rbegin(); it != ctx->auto_choice.rend(); ++it)   // the latest for N
        if (it->N == N) {
            *out = it->p;
            if (ms_per_sample) *ms_per_sample = it->ms;
            return MLMC_OK;
        }
    return MLMC_EINVAL;
}

int mlmc_auto_choice_set(mlmc_ctx* ctx, int N, int tol_class, const mlmc_precision* p) {
    if (!ctx || !p || tol_class < 0 || tol_class > 2) return MLMC_EINVAL;
    int level = -1;
    for (int l = 0; l <= ctx->pr.L_max; ++l)
        if (level_N(ctx, l) == N) level = l;
    if (level < 0) return fail(ctx, MLMC_EINVAL, "mlmc_auto_choice_set: N is not a mesh of the plan");
    const double tol = tol_class == 0 ? 1e-3 : tol_class == 1 ? 1e-5 : 1e-8;
    int rc = check_prec(ctx, p, N, tol);
    if (rc) return rc;
    mlmc_precision q = *p;
    q.max_iter = 0;
    mlmc::ctx_note_auto_choice(ctx, N, tol_class, q, -1.0);   // recorded, not measured
    return MLMC_OK;
}

int mlmc_profile_enable(mlmc_ctx* ctx, int on) {
    if (!ctx) return MLMC_EINVAL;
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    drain_pending(ctx);
    ctx->stats.clear();
    ctx->prof_on = on != 0;
    return MLMC_OK;
}

int mlmc_profile_read(mlmc_ctx* ctx, mlmc_kernel_stat* stats, int max, int* count) {
    if (!ctx || !count) return MLMC_EINVAL;
    CU(cudaStreamSynchronize(ctx->stream));
    drain_pending(ctx);
    *count = (int)ctx->stats.size();
    for (int i = 0; i < max && i < (int)ctx->stats.size(); ++i) stats[i] = ctx->stats[i];
    return MLMC_OK;
}

int mlmc_debug_trace(mlmc_ctx* ctx, void* dev_buf, uint32_t cap, uint32_t* count) {
    if (!ctx) return MLMC_EINVAL;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, MLMC_ECUDA, "cudaSetDevice");
    const cudaError_t e = minres_trace(static_cast<unsigned long long*>(dev_buf), cap, count);
    if (e == cudaErrorNotSupported) return fail(ctx, MLMC_EINVAL, "the job trace needs the MLMC_TUNING build");
    if (e != cudaSuccess) return fail(ctx, MLMC_ECUDA, cudaGetErrorString(e));
    return MLMC_OK;
}

int mlmc_debug_field(mlmc_ctx* ctx, int level, int mesh_level, uint64_t n, uint64_t seed, uint64_t first_index,
                     double* xi_dev, double* a_dev) {
    if (!ctx) return MLMC_EINVAL;
    if (level < 0 || level > ctx->pr.L_max || mesh_level < 0 || mesh_level > level || mesh_level < level - 1)
        return fail(ctx, MLMC_EINVAL, "bad level / mesh_level");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, MLMC_ECUDA, "cudaSetDevice");
    int rc = ensure_phi(ctx, mesh_level);
    if (rc) return rc;
    double* xi = xi_dev;
    if (!xi) CU(cudaMalloc(&xi, sizeof(double) * std::max<uint64_t>(n, 1) * ctx->pr.m));
    CU(launch_rng(xi, ctx->pr.m, n, seed, level, first_index, ctx->stream));
    int N = level_N(ctx, mesh_level);
    (void)N;
    if (a_dev) CU(field(ctx, mesh_level, xi, a_dev, n, nullptr, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (!xi_dev) cudaFree(xi);
    return MLMC_OK;
}

// ---------------------------------------------------------------- host helpers
int mlmc_eps_schedule(int L, double h0, double k_p, double* eps_out) {
    if (L < 0 || !(h0 > 0) || !(k_p > 0) || !eps_out) return MLMC_EINVAL;
    for (int l = 0; l <= L; ++l) {
        double hl = h0 / std::ldexp(1.0, l);
        eps_out[l] = (l < L) ? std::sqrt(k_p) * hl * hl : k_p * hl * hl;   // Eq. (16)
    }
    return MLMC_OK;
}

int mlmc_optimal_samples(int nlev, const double* V, const double* C, double tol, double* N_out) {
    if (nlev < 1 || !V || !C || !N_out || !(tol > 0)) return MLMC_EINVAL;
    double S = 0.0;
    for (int l = 0; l < nlev; ++l) {
        if (!(C[l] > 0) || V[l] < 0) return MLMC_EINVAL;
        S += std::sqrt(V[l] * C[l]);
    }
    for (int l = 0; l < nlev; ++l) N_out[l] = std::sqrt(V[l] / C[l]) * (2.0 / (tol * tol)) * S;
    return MLMC_OK;
}

int mlmc_kl_modes(double sigma2, double corr_len, int m, int32_t* ik, int32_t* jk, double* lam, double* w, int nroots) {
    KLModes kl;
    int rc = kl_modes(sigma2, corr_len, m, kl);
    if (rc) return rc;
    for (int k = 0; k < m; ++k) {
        if (ik) ik[k] = kl.ik[k];
        if (jk) jk[k] = kl.jk[k];
        if (lam) lam[k] = kl.lam[k];
    }
    if (w) for (int k = 0; k < nroots && k < (int)kl.w.size(); ++k) w[k] = kl.w[k];
    return MLMC_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- K3d: one sample over row slabs (NEXT-3)
int mlmc_dd_layout_get(int N, int m, int rank, int world, mlmc_dd_layout* out) {
    if (!out || N < 4 || world < 1 || rank < 0 || rank >= world || m < 1) return MLMC_EINVAL;
    const int C = N - 1;
    const int j0 = 1 + (int)((int64_t)rank * C / world), j1 = 1 + (int)((int64_t)(rank + 1) * C / world);
    if (j1 - j0 < 2) return MLMC_EINVAL;                  // a slab sends its second row: >= 2 rows each
    mlmc_dd_layout L{};
    L.N = N; L.rank = rank; L.world = world; L.j0 = j0; L.j1 = j1;
    L.rows = j1 - j0 + 4;                                 // rows j0-2 .. j1+1
    L.pitch = N + 2;                                      // columns i = -1 .. N at i + 1
    L.tiles = dd_tiles(N, j0, j1);
    const size_t plane = align256(sizeof(double) * (size_t)L.rows * L.pitch);
    size_t off = 0;
    for (int q = 0; q < 5; ++q) { L.plane_off[q] = off; off += plane; }
    L.sums_off = off;  off += align256(sizeof(double) * 4);
    L.state_off = off; off += align256(sizeof(DDState));
    // CTA partials, double-buffered ([2][CTAs][3]): a persistent grid has at most min(tiles, resident slots) CTAs
    // per rank, the fused-exchange grid up to the largest rank's tile count (+1 row of tiles)
    L.partials_off = off; off += align256(sizeof(double) * 6 * (size_t)(L.tiles + 64));
    L.counter_off = off; off += align256(sizeof(unsigned) * 4);     // [0] CTA arrivals, [1] rank arrivals
    L.rpart_off = off; off += align256(sizeof(double) * 2 * kDDMaxRanks * 3);
    L.xi_off = off;    off += align256(sizeof(double) * (size_t)m);
    L.a_off = off;     off += align256(sizeof(double) * 2 * (size_t)N * N);
    L.bytes = off;
    *out = L;
    return MLMC_OK;
}

int mlmc_dd_exchange_rows(const mlmc_dd_layout* L, int step, int64_t offs[4]) {
    if (!L || !offs || step < 0) return MLMC_EINVAL;
    const uint64_t plane = L->plane_off[(step + 2) % 3];   // p_{j+1} formed by pass `step`
    const uint64_t row = sizeof(double) * (uint64_t)L->pitch;
    auto at = [&](int j) { return (int64_t)(plane + row * (uint64_t)(j - (L->j0 - 2))); };
    const bool lo = L->rank > 0, hi = L->rank + 1 < L->world;
    offs[0] = lo ? at(L->j0 + 1) : -1;   // send to rank-1: its ghost row j1' + 1 = j0 + 1
    offs[1] = lo ? at(L->j0 - 2) : -1;   // receive rank-1's row j0 - 2
    offs[2] = hi ? at(L->j1 - 2) : -1;   // send to rank+1: its ghost row j0' - 2 = j1 - 2
    offs[3] = hi ? at(L->j1 + 1) : -1;   // receive rank+1's row j1 + 1
    return MLMC_OK;
}

struct mlmc_dd {
    mlmc_ctx* ctx = nullptr;
    int mesh_level = 0;
    mlmc_dd_layout L{};
    unsigned char* ws = nullptr;
    cudaGraphExec_t chunk = nullptr;      // mlmc_dd_run_local: kDDChunk steps (pass + scalar) as one graph
};

namespace {
constexpr int kDDChunk = 32;
int dd_check(mlmc_dd* dd) {
    if (!dd || !dd->ctx || !dd->ws) return MLMC_EINVAL;
    return cudaSetDevice(dd->ctx->device) == cudaSuccess ? MLMC_OK : fail(dd->ctx, MLMC_ECUDA, "cudaSetDevice");
}
cudaError_t dd_pass(mlmc_dd* dd, cudaStream_t s, bool fuse_scalar = false) {
    const mlmc_dd_layout& L = dd->L;
    return launch_dd_pass(L.N, L.j0, L.j1, L.rows, L.pitch, reinterpret_cast<double*>(dd->ws + L.plane_off[0]),
                          (L.plane_off[1] - L.plane_off[0]) / sizeof(double),
                          reinterpret_cast<DDState*>(dd->ws + L.state_off),
                          reinterpret_cast<double*>(dd->ws + L.partials_off),
                          reinterpret_cast<unsigned*>(dd->ws + L.counter_off),
                          reinterpret_cast<double*>(dd->ws + L.sums_off), fuse_scalar, s);
}
cudaError_t dd_scalar(mlmc_dd* dd, cudaStream_t s) {
    return launch_dd_scalar(reinterpret_cast<DDState*>(dd->ws + dd->L.state_off),
                            reinterpret_cast<const double*>(dd->ws + dd->L.sums_off), dd->L.N, s);
}
}  // namespace

int mlmc_dd_create(mlmc_ctx* ctx, int mesh_level, int rank, int world, void* dev_ws, size_t bytes, mlmc_dd** out) {
    if (!ctx || !out) return MLMC_EINVAL;
    if (mesh_level < 0 || mesh_level > ctx->pr.L_max) return fail(ctx, MLMC_EINVAL, "bad mesh level");
    mlmc_dd_layout L{};
    if (mlmc_dd_layout_get(level_N(ctx, mesh_level), ctx->pr.m, rank, world, &L) != MLMC_OK)
        return fail(ctx, MLMC_EINVAL, "slab partition: world too large for the mesh (>= 2 rows per rank)");
    if (!dev_ws || bytes < L.bytes) return fail(ctx, MLMC_ENOMEM, "dd workspace smaller than mlmc_dd_layout.bytes");
    auto* dd = new mlmc_dd;
    dd->ctx = ctx;
    dd->mesh_level = mesh_level;
    dd->L = L;
    dd->ws = static_cast<unsigned char*>(dev_ws);
    *out = dd;
    return MLMC_OK;
}

int mlmc_dd_begin(mlmc_dd* dd, uint64_t seed, int level, uint64_t index, double tol, int max_iter) {
    int rc = dd_check(dd);
    if (rc) return rc;
    mlmc_ctx* ctx = dd->ctx;
    if (!(level == dd->mesh_level || level == dd->mesh_level + 1) || level > ctx->pr.L_max)
        return fail(ctx, MLMC_EINVAL, "mlmc_dd_begin: level must be mesh_level or mesh_level + 1");
    if (!(tol > 0.0) || !std::isfinite(tol)) return fail(ctx, MLMC_EINVAL, "tolerance must be > 0");
    rc = ensure_phi(ctx, dd->mesh_level);
    if (rc) return rc;
    const mlmc_dd_layout& L = dd->L;
    const int n = (L.N - 1) * (L.N - 1);
    if (max_iter <= 0) max_iter = 16 * n + 1000;           // the MINRES default cap
    double* xi = reinterpret_cast<double*>(dd->ws + L.xi_off);
    double* a = reinterpret_cast<double*>(dd->ws + L.a_off);
    cudaStream_t s = ctx->stream;
    CU(counted(ctx, s, 0, L.N, [&] { return launch_rng(xi, ctx->pr.m, 1, seed, level, index, s); }));
    CU(counted(ctx, s, 1, L.N, [&] { return field(ctx, dd->mesh_level, xi, a, 1, nullptr, s); }));
    CU(cudaMemsetAsync(dd->ws + L.counter_off, 0, sizeof(unsigned) * 4, s));
    CU(counted(ctx, s, 2, L.N, [&] {
        return launch_dd_init(a, L.N, L.j0, L.rows, L.pitch, reinterpret_cast<double*>(dd->ws + L.plane_off[0]),
                              (L.plane_off[1] - L.plane_off[0]) / sizeof(double),
                              reinterpret_cast<DDState*>(dd->ws + L.state_off), tol, max_iter, s);
    }));
    return MLMC_OK;
}

int mlmc_dd_pass(mlmc_dd* dd) {
    int rc = dd_check(dd);
    if (rc) return rc;
    mlmc_ctx* ctx = dd->ctx;
    CU(counted(ctx, ctx->stream, 2, dd->L.N, [&] { return dd_pass(dd, ctx->stream); }));
    return MLMC_OK;
}

int mlmc_dd_scalar(mlmc_dd* dd) {
    int rc = dd_check(dd);
    if (rc) return rc;
    mlmc_ctx* ctx = dd->ctx;
    CU(counted(ctx, ctx->stream, 2, dd->L.N, [&] { return dd_scalar(dd, ctx->stream); }));
    return MLMC_OK;
}

int mlmc_dd_result(mlmc_dd* dd, double out[5]) {
    int rc = dd_check(dd);
    if (rc) return rc;
    if (!out) return MLMC_EINVAL;
    mlmc_ctx* ctx = dd->ctx;
    DDState st{};
    CU(cudaMemcpyAsync(&st, dd->ws + dd->L.state_off, sizeof(DDState), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    out[0] = st.done ? st.Q : 0.0;
    out[1] = st.k;
    out[2] = st.done ? st.relres : (st.beta1 > 0 ? st.phibar * st.inv_beta1 : 1.0);
    out[3] = st.status;
    out[4] = st.done;
    return MLMC_OK;
}

int mlmc_dd_run_local(mlmc_dd* dd, double out[5]) {
    int rc = dd_check(dd);
    if (rc) return rc;
    mlmc_ctx* ctx = dd->ctx;
    if (dd->L.world != 1) return fail(ctx, MLMC_EINVAL, "mlmc_dd_run_local needs world = 1 (no exchange)");
    cudaStream_t s = ctx->stream;
    {   // one cooperative launch for the whole solve (one grid barrier per step); per-step graphs otherwise
        const mlmc_dd_layout& L = dd->L;
        cudaError_t e = counted(ctx, s, 2, L.N, [&] {
            return launch_dd_persistent(L.N, L.j0, L.j1, L.rows, L.pitch,
                                        reinterpret_cast<double*>(dd->ws + L.plane_off[0]),
                                        (L.plane_off[1] - L.plane_off[0]) / sizeof(double),
                                        reinterpret_cast<DDState*>(dd->ws + L.state_off),
                                        reinterpret_cast<double*>(dd->ws + L.partials_off),
                                        reinterpret_cast<unsigned*>(dd->ws + L.counter_off),
                                        reinterpret_cast<double*>(dd->ws + L.sums_off), s);
        });
        if (e == cudaSuccess) return mlmc_dd_result(dd, out);
        cudaGetLastError();                          // not co-schedulable here: fall back to the graph chunks
    }
    if (!dd->chunk) {
        // kDDChunk steps as one graph: every launch takes its step-dependent values from the device state
        cudaStream_t cs = nullptr;
        CU(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        cudaGraph_t g = nullptr;
        CU(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        cudaError_t e = cudaSuccess;
        for (int k = 0; k < kDDChunk && e == cudaSuccess; ++k) e = dd_pass(dd, cs, true);   // scalar step fused
        cudaError_t e2 = cudaStreamEndCapture(cs, &g);
        cudaStreamDestroy(cs);
        if (e != cudaSuccess || e2 != cudaSuccess) return fail(ctx, MLMC_ECUDA, "dd graph capture failed");
        CU(cudaGraphInstantiate(&dd->chunk, g, 0));
        cudaGraphDestroy(g);
    }
    DDState* st_dev = reinterpret_cast<DDState*>(dd->ws + dd->L.state_off);
    int done = 0;
    const int max_chunks = (int)(((int64_t)16 * (dd->L.N - 1) * (dd->L.N - 1) + 1000) / kDDChunk + 2);
    const int idx = stat_index(ctx, 2, dd->L.N);
    for (int c = 0; c < max_chunks && !done; ++c) {
        CU(cudaGraphLaunch(dd->chunk, s));
        ctx->stats[idx].launches += kDDChunk;                // the graph's kernels
        CU(cudaMemcpyAsync(&done, &st_dev->done, sizeof(int), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
    }
    return mlmc_dd_result(dd, out);
}

namespace {
// the fused-exchange launch description of ranks 0..world-1 whose workspaces are at ws[q] (device-accessible)
DDPeerLaunch dd_peer_desc(int N, int m, int world, void* const* ws) {
    DDPeerLaunch D{};
    D.N = N;
    D.world = world;
    for (int q = 0; q < world; ++q) {
        mlmc_dd_layout L{};
        mlmc_dd_layout_get(N, m, q, world, &L);
        unsigned char* b = static_cast<unsigned char*>(ws[q]);
        D.j0[q] = L.j0; D.j1[q] = L.j1; D.rows[q] = L.rows;
        D.planes[q] = reinterpret_cast<double*>(b + L.plane_off[0]);
        D.plane_stride[q] = (L.plane_off[1] - L.plane_off[0]) / sizeof(double);
        D.st[q] = reinterpret_cast<DDState*>(b + L.state_off);
        D.partials[q] = reinterpret_cast<double*>(b + L.partials_off);
        D.counter[q] = reinterpret_cast<unsigned*>(b + L.counter_off);
        D.xcounter[q] = reinterpret_cast<unsigned*>(b + L.counter_off) + 1;
        D.rpart[q] = reinterpret_cast<double*>(b + L.rpart_off);
        D.sums[q] = reinterpret_cast<double*>(b + L.sums_off);
    }
    return D;
}
}  // namespace

int mlmc_dd_run_emulated(mlmc_dd* const* dds, int world, double out[5]) {
    if (!dds || world < 1 || world > kDDMaxRanks || !dds[0]) return MLMC_EINVAL;
    int rc = dd_check(dds[0]);
    if (rc) return rc;
    mlmc_ctx* ctx = dds[0]->ctx;
    std::vector<void*> ws(world);
    for (int q = 0; q < world; ++q) {
        if (!dds[q] || dds[q]->ctx != ctx || dds[q]->L.rank != q || dds[q]->L.world != world ||
            dds[q]->L.N != dds[0]->L.N)
            return fail(ctx, MLMC_EINVAL, "mlmc_dd_run_emulated: dds[q] must be rank q of `world` on one ctx / mesh");
        ws[q] = dds[q]->ws;
    }
    DDPeerLaunch D = dd_peer_desc(dds[0]->L.N, ctx->pr.m, world, ws.data());
    D.rank0 = 0;
    D.nranks = world;
    cudaStream_t s = ctx->stream;
    for (int q = 0; q < world; ++q) CU(cudaMemsetAsync(D.counter[q], 0, sizeof(unsigned) * 2, s));
    CU(counted(ctx, s, 2, D.N, [&] { return launch_dd_peer(D, s); }));
    for (int q = 0; q < world; ++q) CU(cudaMemsetAsync(D.counter[q], 0, sizeof(unsigned) * 2, s));
    return mlmc_dd_result(dds[0], out);
}

int mlmc_dd_run_peer(mlmc_dd* dd, void* const* peer_ws, double out[5]) {
    int rc = dd_check(dd);
    if (rc) return rc;
    mlmc_ctx* ctx = dd->ctx;
    const int world = dd->L.world;
    if (world > kDDMaxRanks) return fail(ctx, MLMC_EINVAL, "mlmc_dd_run_peer: at most 8 ranks (one NVLink node)");
    if (!peer_ws) return fail(ctx, MLMC_EINVAL, "mlmc_dd_run_peer: peer_ws is NULL");
    for (int q = 0; q < world; ++q)
        if (!peer_ws[q]) return fail(ctx, MLMC_EINVAL, "mlmc_dd_run_peer: a peer workspace is NULL");
    DDPeerLaunch D = dd_peer_desc(dd->L.N, ctx->pr.m, world, peer_ws);
    D.rank0 = dd->L.rank;
    D.nranks = 1;
    cudaStream_t s = ctx->stream;
    // the counters were zeroed by mlmc_dd_begin on every rank (the caller synchronises the ranks between
    // mlmc_dd_begin and this call, e.g. with a barrier)
    CU(counted(ctx, s, 2, D.N, [&] { return launch_dd_peer(D, s); }));
    CU(cudaStreamSynchronize(s));
    CU(cudaMemsetAsync(D.counter[dd->L.rank], 0, sizeof(unsigned) * 2, s));
    return mlmc_dd_result(dd, out);
}

// ---- peer mapping of the slab workspaces (CUDA IPC; one process per GPU on an NVLink node)
namespace {
using PFN_getAddressRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
PFN_getAddressRange address_range_fn() {
    static PFN_getAddressRange fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_getAddressRange>(p);
    });
    return fn;
}
}  // namespace

int mlmc_dd_ipc_handle(mlmc_dd* dd, void* handle, uint64_t* offset) {
    int rc = dd_check(dd);
    if (rc) return rc;
    mlmc_ctx* ctx = dd->ctx;
    if (!handle || !offset) return fail(ctx, MLMC_EINVAL, "mlmc_dd_ipc_handle: NULL output");
    auto range = address_range_fn();
    if (!range) return fail(ctx, MLMC_ECUDA, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dd->ws)) != CUDA_SUCCESS)
        return fail(ctx, MLMC_ECUDA, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));   // the allocation holding the workspace
    std::memcpy(handle, &h, sizeof(h));
    *offset = (uint64_t)(reinterpret_cast<CUdeviceptr>(dd->ws) - base);
    return MLMC_OK;
}

int mlmc_dd_ipc_open(mlmc_ctx* ctx, const void* handle, uint64_t offset, void** ptr, void** base_out) {
    if (!ctx || !handle || !ptr || !base_out) return MLMC_EINVAL;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, MLMC_ECUDA, "cudaSetDevice");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    CU(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *base_out = base;
    *ptr = static_cast<unsigned char*>(base) + offset;
    return MLMC_OK;
}

int mlmc_dd_ipc_close(mlmc_ctx* ctx, void* base) {
    if (!ctx || !base) return MLMC_EINVAL;
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, MLMC_ECUDA, "cudaSetDevice");
    CU(cudaIpcCloseMemHandle(base));
    return MLMC_OK;
}

void mlmc_dd_destroy(mlmc_dd* dd) {
    if (!dd) return;
    if (dd->chunk) cudaGraphExecDestroy(dd->chunk);
    delete dd;
}
