// controller.cpp -- Algorithm 2 (adaptive MPML) on top of the per-level sampler.
//
// Readings: R1 bias constant (r m^alpha - 1)/sqrt(2) with
// r = 1; R2 stop when both tests pass, ELMAX if the bias test still fails at
// L_max once the variance test passes; R3 draw max(0, ceil(N_l) - N_l^done)
// new samples, N_l never decreases; R4 V_l = s_l^2 with 1/N_l; R5/R21 C_l =
// mean deterministic work of one coupled sample; R6 N_init = 100; R8 coarse
// half at eps_{l-1}; R20 samples already drawn keep their tolerance; R23 the
// global per-level index counts all rounds, ranks take contiguous slices; R25
// the variance test uses the N_l drawn so far.  Every rank runs this loop on
// identical all-reduced sums, so every rank takes the same decisions without a
// broadcast.  The same loop runs over the GPU (mlmc_adaptive_run: every level
// of a round in one mlmc_sample_levels_async call) or over a caller-supplied
// host sampler (mlmc_adaptive_run_host: CPU tests of the controller and of the
// multi-rank exchange).
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <cmath>
#include <cstring>
#include <functional>
#include <vector>

#include "internal.h"

namespace {

using u64 = unsigned long long;
using mlmc::kXFields;
using mlmc::kXLen;
using mlmc::kXScale;
using mlmc::kXWords;

struct LevelAcc {
    double s[MLMC_SUMS_LEN] = {0};
    u64 x[kXLen] = {0};   // exact fixed-point Y, Y^2, Q_f, Q_c, cost sums (internal.h kX*)
    uint64_t drawn = 0;
};

// 256-bit two's-complement addition (mod 2^256) of field f's limbs
void x_add(u64* a, const u64* b) {
    u64 c = 0;
    for (int i = 0; i < 4; ++i) {
        const u64 s = a[i] + b[i];
        const u64 c1 = s < a[i];
        a[i] = s + c;
        c = c1 | (a[i] < s);
    }
}

// x rounded once (nearest even) to a multiple of 2^-kXScale as 4 limbs + overflow word (the host twin of
// k_reduce.cu's x_acc, for the host runner's per-rank sums)
void x_from_double(double x, u64* w) {
    for (int i = 0; i < kXWords; ++i) w[i] = 0;
    if (x == 0.0) return;
    if (!(std::fabs(x) < 0x1p62)) { w[4] = 1; return; }
    const double X = std::ldexp(x, kXScale);
    u64 v[4] = {0, 0, 0, 0};
    if (std::fabs(X) < 0x1p62) {
        const long long i = std::llrint(X);   // default rounding: to nearest even
        v[0] = (u64)i;
        v[1] = v[2] = v[3] = i < 0 ? ~0ull : 0ull;
    } else {
        int e;
        const double f = std::frexp(std::fabs(X), &e);
        const u64 m = (u64)(f * 0x1p53);
        const int k = e - 53, q = k >> 6, r = k & 63;
        v[q] = m << r;
        if (r && q + 1 < 4) v[q + 1] = m >> (64 - r);
        if (x < 0.0) {
            for (int i = 0; i < 4; ++i) v[i] = ~v[i];
            const u64 one[4] = {1, 0, 0, 0};
            x_add(v, one);
        }
    }
    for (int i = 0; i < 4; ++i) w[i] = v[i];
}

// The exact fixed-point value (4 limbs, units of 2^-kXScale) rounded to the nearest double, ties to even.
// A function of the integer alone, so every rank converts an identical total to identical bits.
double x_to_double(const u64* w) {
    u64 a[4] = {w[0], w[1], w[2], w[3]};
    const bool neg = a[3] >> 63;
    if (neg) {   // |value|
        for (int i = 0; i < 4; ++i) a[i] = ~a[i];
        const u64 one[4] = {1, 0, 0, 0};
        x_add(a, one);
    }
    int msb = -1;
    for (int i = 3; i >= 0 && msb < 0; --i)
        if (a[i]) msb = 64 * i + 63 - __builtin_clzll(a[i]);
    if (msb < 0) return 0.0;
    auto bit = [&](int i) -> u64 { return (i >= 0 && i < 256) ? (a[i >> 6] >> (i & 63)) & 1ull : 0ull; };
    u64 mant = 0;   // bits msb .. msb-52
    for (int b = 0; b < 53; ++b) mant |= bit(msb - 52 + b) << b;
    const u64 guard = bit(msb - 53);
    bool sticky = false;
    for (int i = msb - 54; i >= 0 && !sticky; --i) sticky = bit(i) != 0;
    int e = msb - 52 - kXScale;
    if (guard && (sticky || (mant & 1ull))) {
        if (++mant == (1ull << 53)) { mant >>= 1; ++e; }
    }
    const double v = std::ldexp((double)mant, e);
    return neg ? -v : v;
}

mlmc_precision minres_prec() {
    return mlmc_precision{MLMC_SOLVER_MINRES, MLMC_FMT_F64, MLMC_FMT_F64, MLMC_FMT_F64, MLMC_FMT_F64, 0, 0};
}

// Table 1 (right) quads on the levels where the shared-memory banded factor exists (N <= 32):
// level 0 hhss, level 1 ssss, levels 2+ ssdd, as written -- where the level's tolerance is one the reduced
// precisions can certify (binary16 substitutions for tol >= 1e-3, binary32 vectors for tol >= 1e-5;
// otherwise the next wider format), MINRES beyond (R14).
mlmc_precision policy_prec(int policy, int level, int N, double tol) {
    if (policy == 2 && N >= 32)   // NEXT-4: MG-PCG where it beats MINRES, h <= 1/32
        return mlmc_precision{MLMC_SOLVER_MGCG, MLMC_FMT_F64, MLMC_FMT_F64, MLMC_FMT_F64, MLMC_FMT_F64, 0, 0};
    if (policy == 1 && N <= 32) {
        const int vec = tol >= 1e-5 ? MLMC_FMT_F32 : MLMC_FMT_F64;
        if (level == 0)
            return mlmc_precision{MLMC_SOLVER_CHOL_IR, MLMC_FMT_F16, tol >= 1e-3 ? MLMC_FMT_F16 : MLMC_FMT_F32, vec, vec,
                                  0, 0};
        if (level == 1)
            return mlmc_precision{MLMC_SOLVER_CHOL_IR, MLMC_FMT_F32, MLMC_FMT_F32, vec, vec, 0, 0};
        return mlmc_precision{MLMC_SOLVER_CHOL_IR, MLMC_FMT_F32, MLMC_FMT_F64, MLMC_FMT_F64, MLMC_FMT_F64, 0, 0};
    }
    return minres_prec();
}

// Draw one round: for each q, n[q] samples of levels[q] from first[q]; write
// MLMC_SUMS_LEN sums per entry to sums (host).
// xs (exact runners only): nlev x kXLen fixed-point words of the same sums.
using RoundSampler = std::function<int(int nlev, const int* levels, const uint64_t* n, const uint64_t* first,
                                       const mlmc_precision* pf, const mlmc_precision* pc, const double* tf,
                                       const double* tc, double* sums, u64* xs)>;

// precision of the solves on mesh N of level `level` at tolerance tol
using PrecChooser = std::function<int(int level, int N, double tol, mlmc_precision* out)>;

// exact: the sampler also returns the fixed-point sums; they are what the ranks exchange and what the
// statistics use (bit-identical sums and decisions for any number of ranks).
int adaptive_core(int h0_inv, int L_max, double eps, const mlmc_adaptive_opts& o, const RoundSampler& sampler,
                  const PrecChooser& choose, mlmc_allreduce_fn allreduce, void* user, mlmc_result* out,
                  bool exact = false) {
    if (!(eps > 0.0) || o.world < 1 || o.rank < 0 || o.rank >= o.world || L_max < 1 || h0_inv < 2)
        return MLMC_EINVAL;
    if (o.world > 1 && !allreduce) return MLMC_EINVAL;
    const double h0 = 1.0 / h0_inv, TOL = eps;
    const int N_init = o.N_init > 0 ? o.N_init : 100;
    const int max_rounds = o.max_rounds > 0 ? o.max_rounds : 100;
    const double r_bias = o.r_bias > 0 ? o.r_bias : 1.0;
    const double alpha = 2.0, mref = 2.0;
    const double bias_c = (r_bias * std::pow(mref, alpha) - 1.0) / std::sqrt(2.0);

    std::vector<LevelAcc> acc(2);
    std::vector<double> target(2, (double)N_init);
    std::vector<double> epsl;
    int L = 1, rounds = 0, code = MLMC_OK;
    double solve_s = 0.0;
    int64_t n_fail = 0;

    // field f (0 Y, 1 Y^2, 2 Q_f, 3 Q_c, 4 cost) of level l: the exact sum rounded once where it exists
    auto sum = [&](int l, int f) {
        const u64* x = acc[l].x + f * kXWords;
        return exact && x[4] == 0 ? x_to_double(x) : acc[l].s[f];
    };
    auto stats = [&](int l, double& mean, double& var, double& cost) {
        const double n = acc[l].s[5];
        mean = n > 0 ? sum(l, 0) / n : 0.0;
        var = n > 0 ? std::max(0.0, sum(l, 1) / n - mean * mean) : 0.0;   // Eq. (4) with 1/N_l (R4)
        cost = n > 0 ? sum(l, 4) / n : 0.0;
    };

    // MLMC_ROUND_LOG=<path>: rank 0 appends one JSON line per round (round, L, N_l, level statistics, eps_l,
    // the two tests) -- the run's trace, for long runs and post-mortems
    const char* log_path = o.rank == 0 ? std::getenv("MLMC_ROUND_LOG") : nullptr;
    while (L <= L_max && rounds < max_rounds) {
        ++rounds;
        epsl.assign(L + 1, o.fixed_tol > 0 ? o.fixed_tol : 1e-10);
        if (o.k_p > 0.0) mlmc_eps_schedule(L, h0, o.k_p, epsl.data());   // step 2, Eq. (16)
        std::vector<double> round_sums((size_t)(L + 1) * MLMC_SUMS_LEN, 0.0);
        std::vector<u64> round_x((size_t)(L + 1) * kXLen, 0);
        std::vector<uint64_t> dN(L + 1, 0);
        // steps 3-4: this rank's slice of every level's new indices, all levels in one call
        std::vector<int> lv;
        std::vector<uint64_t> cnt, first;
        std::vector<mlmc_precision> pf, pc;
        std::vector<double> tf, tc;
        for (int l = 0; l <= L; ++l) {
            const double want = std::ceil(target[l]);
            dN[l] = want > (double)acc[l].drawn ? (uint64_t)(want - (double)acc[l].drawn) : 0;
            if (dN[l] == 0) continue;
            const uint64_t lo = acc[l].drawn + dN[l] * (uint64_t)o.rank / (uint64_t)o.world;
            const uint64_t hi = acc[l].drawn + dN[l] * (uint64_t)(o.rank + 1) / (uint64_t)o.world;
            lv.push_back(l);
            cnt.push_back(hi - lo);
            first.push_back(lo);
            mlmc_precision qf, qc;
            int rcp = choose(l, h0_inv << l, epsl[l], &qf);
            if (!rcp && l > 0) rcp = choose(l - 1, h0_inv << (l - 1), epsl[l - 1], &qc);
            if (rcp) return rcp;   // the chooser has already agreed its outcome across the ranks
            if (o.on_fail == 2) {   // escalation of failed MINRES / IR solves to MG-PCG (MLMC_FLAG_ESCALATE)
                if (qf.solver != MLMC_SOLVER_MGCG) qf.flags |= MLMC_FLAG_ESCALATE;
                if (l > 0 && qc.solver != MLMC_SOLVER_MGCG) qc.flags |= MLMC_FLAG_ESCALATE;
            }
            pf.push_back(qf);
            pc.push_back(l > 0 ? qc : qf);
            tf.push_back(epsl[l]);
            tc.push_back(l > 0 ? epsl[l - 1] : epsl[l]);
        }
        int local_rc = MLMC_OK;
        if (!lv.empty()) {
            std::vector<double> s(lv.size() * MLMC_SUMS_LEN, 0.0);
            std::vector<u64> xs(exact ? lv.size() * kXLen : 0, 0);
            auto t0 = std::chrono::steady_clock::now();
            nvtxRangePushA("mlmc adaptive round: sampling");
            local_rc = sampler((int)lv.size(), lv.data(), cnt.data(), first.data(), pf.data(), pc.data(), tf.data(),
                               tc.data(), s.data(), exact ? xs.data() : nullptr);
            nvtxRangePop();
            solve_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            // a rank-local failure must not leave the other ranks waiting in the exchange: the error
            // travels in the round's all-reduce and every rank returns together
            if (local_rc && o.world == 1) return local_rc;
            if (local_rc) { std::fill(s.begin(), s.end(), 0.0); std::fill(xs.begin(), xs.end(), 0ull); }
            for (size_t q = 0; q < lv.size(); ++q) {
                std::memcpy(&round_sums[(size_t)lv[q] * MLMC_SUMS_LEN], &s[q * MLMC_SUMS_LEN],
                            sizeof(double) * MLMC_SUMS_LEN);
                if (exact) std::memcpy(&round_x[(size_t)lv[q] * kXLen], &xs[q * kXLen], sizeof(u64) * kXLen);
            }
        }
        // ONE exchange per round: a SUM all-reduce of the additive fields (the per-rank iteration maxima, fields
        // 9/10, are diagnostics the controller never uses: they are not exchanged), the exact sums' 32-bit
        // pieces and an error flag
        if (o.world > 1) {
            for (int l = 0; l <= L; ++l) {
                round_sums[(size_t)l * MLMC_SUMS_LEN + 9] = 0.0;
                round_sums[(size_t)l * MLMC_SUMS_LEN + 10] = 0.0;
            }
            // exact sums: each field's 256-bit integer as eight 32-bit pieces (doubles, so the SUM over up to
            // 2^21 ranks stays exact), then the carries are propagated; the overflow counts are plain sums
            constexpr int XD = kXFields * 9;
            const size_t base = round_sums.size();
            if (exact) {
                round_sums.resize(base + (size_t)(L + 1) * XD, 0.0);
                for (int l = 0; l <= L; ++l)
                    for (int f = 0; f < kXFields; ++f) {
                        const u64* x = &round_x[(size_t)l * kXLen + f * kXWords];
                        double* d = &round_sums[base + (size_t)l * XD + f * 9];
                        for (int i = 0; i < 8; ++i) d[i] = (double)((x[i / 2] >> (32 * (i % 2))) & 0xffffffffull);
                        d[8] = (double)x[4];
                    }
            }
            round_sums.push_back(local_rc ? 1.0 : 0.0);                  // ranks that failed this round
            if (allreduce(round_sums.data(), (int)round_sums.size(), 0, user) != 0) return MLMC_ECUDA;
            const bool any_err = round_sums.back() > 0.0;
            round_sums.pop_back();
            if (any_err) return local_rc ? local_rc : MLMC_ESOLVER;
            if (exact) {
                for (int l = 0; l <= L; ++l)
                    for (int f = 0; f < kXFields; ++f) {
                        u64* x = &round_x[(size_t)l * kXLen + f * kXWords];
                        const double* d = &round_sums[base + (size_t)l * XD + f * 9];
                        u64 carry = 0;
                        for (int i = 0; i < 4; ++i) x[i] = 0;
                        for (int i = 0; i < 8; ++i) {
                            const u64 t = (u64)d[i] + carry;
                            x[i / 2] |= (t & 0xffffffffull) << (32 * (i % 2));
                            carry = t >> 32;
                        }
                        x[4] = (u64)d[8];
                    }
                round_sums.resize(base);
            }
        }
        bool failed = false;
        for (int l = 0; l <= L; ++l) {
            const double* rs = &round_sums[(size_t)l * MLMC_SUMS_LEN];
            for (int k = 0; k < MLMC_SUMS_LEN; ++k)
                acc[l].s[k] = (k == 9 || k == 10) ? std::max(acc[l].s[k], rs[k]) : acc[l].s[k] + rs[k];
            if (exact)
                for (int f = 0; f < kXFields; ++f) {
                    const u64* rx = &round_x[(size_t)l * kXLen + f * kXWords];
                    x_add(acc[l].x + f * kXWords, rx);
                    acc[l].x[f * kXWords + 4] += rx[4];
                }
            acc[l].drawn += dN[l];
            if (rs[6] > 0) failed = true;
            n_fail += (int64_t)rs[6];
        }
        // a failed solve is never resampled (R15): stop, or keep it and count it (on_fail = 1)
        if (failed && o.on_fail == 0) { code = MLMC_ESOLVER; break; }
        // steps 5-7
        std::vector<double> mean(L + 1), V(L + 1), C(L + 1), Nopt(L + 1);
        for (int l = 0; l <= L; ++l) stats(l, mean[l], V[l], C[l]);
        mlmc_optimal_samples(L + 1, V.data(), C.data(), TOL, Nopt.data());
        for (int l = 0; l <= L; ++l) target[l] = std::max((double)acc[l].drawn, Nopt[l]);   // R3
        const bool bias_fail = std::fabs(mean[L]) > bias_c * TOL;                          // step 8
        double vsum = 0.0;
        for (int l = 0; l <= L; ++l) vsum += V[l] / (double)acc[l].drawn;                 // R25
        const bool var_ok = vsum <= TOL * TOL / 2.0;
        if (log_path) {
            if (FILE* f = std::fopen(log_path, "a")) {
                std::fprintf(f, "{\"round\": %d, \"L\": %d, \"eps\": %.17g, \"bias_fail\": %s, \"var_ok\": %s, "
                                "\"solve_seconds\": %.6g, \"levels\": [", rounds, L, TOL, bias_fail ? "true" : "false",
                             var_ok ? "true" : "false", solve_s);
                for (int l = 0; l <= L; ++l)
                    std::fprintf(f, "%s{\"N\": %llu, \"mean\": %.17g, \"var\": %.17g, \"cost\": %.17g, "
                                    "\"eps_l\": %.17g, \"target\": %.17g}", l ? ", " : "",
                                 (unsigned long long)acc[l].drawn, mean[l], V[l], C[l], epsl[l], target[l]);
                std::fprintf(f, "]}\n");
                std::fclose(f);
            }
        }
        if (!bias_fail && var_ok) { code = MLMC_OK; break; }                                // steps 12-13
        if (bias_fail) {
            if (L == L_max) {
                code = MLMC_ELMAX;
                if (var_ok) break;
                continue;
            }
            ++L;                                                                            // steps 9-10
            acc.emplace_back();
            target.push_back((double)N_init);
        }
        if (rounds == max_rounds) code = MLMC_ELMAX;
    }
    std::memset(out, 0, sizeof(*out));
    out->L = L;
    out->rounds = rounds;
    out->code = code;
    out->n_fail = (int32_t)std::min<int64_t>(n_fail, INT32_MAX);
    out->solve_seconds = solve_s;
    double est = 0.0;
    for (int l = 0; l <= L && l < MLMC_MAX_LEVELS; ++l) {
        double m_, v_, c_;
        stats(l, m_, v_, c_);
        out->N[l] = acc[l].drawn;
        out->mean[l] = m_;
        out->var[l] = v_;
        out->cost[l] = c_;
        out->eps[l] = l < (int)epsl.size() ? epsl[l] : 0.0;
        est += m_;   // Eq. (3)
    }
    out->estimate = est;
    return code;
}

}  // namespace

// Policy 3 (auto): on first use of a mesh, every admissible solver / precision is
// timed on a pilot batch (its own seed, never part of the estimator; kernel device time from the library's
// per-launch events) and the fastest per sample is kept for that mesh.  Admissibility is empirical: a
// candidate with a failed pilot solve (breakdown, no convergence within the pilot's iteration cap:
// Corollary 3.3's kappa u_f < 1/2 violated in practice) is out.  With several ranks the pilot times are
// summed across them first, so every rank keeps the same choice.
struct AutoChooser {
    mlmc_ctx* ctx;
    uint64_t seed;
    mlmc_allreduce_fn allreduce;
    void* user;
    int world;

    static mlmc_precision q(int solver, int uf, int us, int u, int max_iter = 0) {
        return mlmc_precision{solver, uf, us, u, u, max_iter, 0};
    }
    // (MINRES last: its pilot is screened against the best time of the others, see choose)
    std::vector<mlmc_precision> candidates(int N, double tol) const {
        std::vector<mlmc_precision> c;
        c.push_back(q(MLMC_SOLVER_MGCG, MLMC_FMT_F64, MLMC_FMT_F64, MLMC_FMT_F64));
        if (N <= 32) {   // the banded factors (K4)
            if (tol >= 1e-3) c.push_back(q(MLMC_SOLVER_CHOL_IR, MLMC_FMT_F16, MLMC_FMT_F16, MLMC_FMT_F32));
            if (tol >= 1e-5) {
                c.push_back(q(MLMC_SOLVER_CHOL_IR, MLMC_FMT_E4M3, MLMC_FMT_F32, MLMC_FMT_F32));
                c.push_back(q(MLMC_SOLVER_CHOL_IR, MLMC_FMT_F16, MLMC_FMT_F32, MLMC_FMT_F32));
                c.push_back(q(MLMC_SOLVER_CHOL_IR, MLMC_FMT_F32, MLMC_FMT_F32, MLMC_FMT_F32));
            }
            c.push_back(q(MLMC_SOLVER_CHOL_IR, MLMC_FMT_F16, MLMC_FMT_F32, MLMC_FMT_F64));
            c.push_back(q(MLMC_SOLVER_CHOL_IR, MLMC_FMT_F32, MLMC_FMT_F64, MLMC_FMT_F64));
        }
        c.push_back(q(MLMC_SOLVER_MINRES, MLMC_FMT_F64, MLMC_FMT_F64, MLMC_FMT_F64));
        return c;
    }
    // device ms of the pilot's solves on mesh N (the library's per-launch events)
    double pilot_ms(int N) const {
        mlmc_kernel_stat st[64];
        int cnt = 0;
        mlmc_profile_read(ctx, st, 64, &cnt);
        double t = 0.0;
        for (int i = 0; i < std::min(cnt, 64); ++i)
            if (st[i].N == N && (st[i].kind == MLMC_K_MINRES || st[i].kind == MLMC_K_CHOL_IR)) t += st[i].ms;
        return t;
    }
    int choose(int level, int N, double tol, mlmc_precision* out) {
        // the admissible candidates change at tol = 1e-3 and 1e-5: one choice per (mesh, tolerance class),
        // kept in the context across runs
        const int cls = tol >= 1e-3 ? 0 : tol >= 1e-5 ? 1 : 2;
        if (mlmc::ctx_find_auto_choice(ctx, N, cls, out)) return MLMC_OK;
        const int n_unk = (N - 1) * (N - 1);
        const uint64_t npilot = (uint64_t)std::min(512, std::max(8, (1 << 20) / n_unk));
        std::vector<mlmc_precision> cand = candidates(N, tol);
        std::vector<double> ms(cand.size(), 0.0);
        // the coarse half of a pilot sample is a loose MINRES solve (it only has to converge, not to be timed)
        const mlmc_precision cheap = q(MLMC_SOLVER_MINRES, MLMC_FMT_F64, MLMC_FMT_F64, MLMC_FMT_F64, 4 * n_unk + 400);
        const uint64_t pseed = seed ^ 0x9e3779b97f4a7c15ull;
        for (size_t c = 0; c < cand.size(); ++c) {
            mlmc_precision p = cand[c];
            p.max_iter = p.solver == MLMC_SOLVER_CHOL_IR ? 50 : 4 * n_unk + 400;   // the pilot's budget
            double best = -1.0;
            for (size_t b = 0; b < c; ++b)
                if (ms[b] >= 0 && (best < 0 || ms[b] < best)) best = ms[b];
            if (p.solver == MLMC_SOLVER_MINRES && best > 0.0) {
                // screening: kScreen MINRES steps on the same pilot batch; if they already cost more than the best
                // candidate's whole solve, or the residual decay they show extrapolates (log-linearly) to a
                // solve slower than it, MINRES is dominated and its full pilot (thousands of steps on the fine
                // meshes: ~2.5 s of the first configs[4] run at eps = 1e-5) is skipped
                constexpr int kScreen = 200;
                mlmc_precision ps = p;
                ps.max_iter = kScreen;
                std::vector<double> rec((size_t)npilot * MLMC_SAMPLE_LEN, 0.0);
                mlmc_level_sums ss;
                int rs = mlmc_profile_enable(ctx, 1);
                if (!rs) rs = mlmc_sample_level(ctx, level, npilot, pseed, 0, &ps, &cheap, tol, 0.5, &ss, rec.data());
                const double t_screen = rs ? -1.0 : pilot_ms(N);
                mlmc_profile_enable(ctx, 0);
                if (!rs && ss.n_fail > 0) {                   // not converged within kScreen steps
                    double worst = 0.0;                       // steps the slowest sample would need
                    for (uint64_t k = 0; k < npilot; ++k) {
                        const double rr = rec[k * MLMC_SAMPLE_LEN + 4];
                        const double need = (rr > 0.0 && rr < 1.0) ? kScreen * std::log(tol) / std::log(rr)
                                                                   : 1e300;
                        worst = std::max(worst, need);
                    }
                    const double est = t_screen * worst / kScreen;
                    if (t_screen >= best || est >= 1.5 * best) { ms[c] = -1.0; continue; }
                } else if (!rs) {                             // converged within the screen: that is its pilot
                    ms[c] = t_screen;
                    continue;
                }
            }
            mlmc_level_sums sums;
            int rc = mlmc_profile_enable(ctx, 1);
            if (!rc) rc = mlmc_sample_level(ctx, level, npilot, pseed, 0, &p, &cheap, tol, 0.5, &sums, nullptr);
            if (rc == MLMC_EINVAL) { mlmc_profile_enable(ctx, 0); ms[c] = -1.0; continue; }   // not built here
            if (rc) {                            // agree on the failure before leaving
                mlmc_profile_enable(ctx, 0);
                if (world > 1 && allreduce) {
                    std::vector<double> buf(2 * ms.size() + 1, 0.0);
                    buf.back() = 1.0;
                    allreduce(buf.data(), (int)buf.size(), 0, user);
                }
                return rc;
            }
            const double t = pilot_ms(N);
            mlmc_profile_enable(ctx, 0);
            ms[c] = sums.n_fail > 0 ? -1.0 : t;     // a failed pilot solve: inadmissible
        }
        if (world > 1 && allreduce) {   // one SUM all-reduce: pilot times, failure counts, error flag
            const size_t C = ms.size();
            std::vector<double> buf(2 * C + 1, 0.0);
            for (size_t c = 0; c < C; ++c) { buf[c] = ms[c] < 0 ? 0.0 : ms[c]; buf[C + c] = ms[c] < 0 ? 1.0 : 0.0; }
            if (allreduce(buf.data(), (int)buf.size(), 0, user) != 0) return MLMC_ECUDA;
            if (buf[2 * C] > 0.0) return MLMC_ECUDA;          // another rank's pilot failed
            for (size_t c = 0; c < C; ++c) ms[c] = buf[C + c] > 0 ? -1.0 : buf[c];
        }
        size_t best = 0;
        for (size_t c = 1; c < ms.size(); ++c)
            if (ms[c] >= 0 && (ms[best] < 0 || ms[c] < ms[best])) best = c;
        mlmc_precision p = cand[best];
        p.max_iter = 0;
        mlmc::ctx_note_auto_choice(ctx, N, cls, p, ms[best] / (double)npilot);
        *out = p;
        return MLMC_OK;
    }
};

extern "C" int mlmc_adaptive_run(mlmc_ctx* ctx, double eps, const mlmc_adaptive_opts* opts,
                                 mlmc_allreduce_fn allreduce, void* user, mlmc_result* out) {
    if (!ctx || !opts || !out) return MLMC_EINVAL;
    mlmc_level_info li0;
    if (mlmc_level_info_get(ctx, 0, &li0) != MLMC_OK) return MLMC_EINVAL;
    int L_max = 0;
    mlmc_level_info li;
    while (L_max + 1 < MLMC_MAX_LEVELS && mlmc_level_info_get(ctx, L_max + 1, &li) == MLMC_OK) ++L_max;
    double* dev = mlmc::ctx_adaptive_sums(ctx);     // persistent (no allocation inside a timed run)
    if (!dev) return MLMC_ECUDA;
    const uint64_t seed = opts->seed;
    RoundSampler gpu = [&](int nlev, const int* lv, const uint64_t* n, const uint64_t* first, const mlmc_precision* pf,
                           const mlmc_precision* pc, const double* tf, const double* tc, double* sums,
                           u64* xs) -> int {
        int rc = mlmc_sample_levels_async(ctx, nlev, lv, n, seed, first, pf, pc, tf, tc, dev);
        if (rc) return rc;
        rc = mlmc::copy_sums_to_host(ctx, dev, nlev, sums);
        return rc || !xs ? rc : mlmc::copy_xsums_to_host(ctx, nlev, xs);
    };
    AutoChooser ac{ctx, seed, allreduce, user, opts->world};
    const int policy = opts->policy;
    PrecChooser choose = [&](int level, int N, double tol, mlmc_precision* p) -> int {
        if (policy == 3) return ac.choose(level, N, tol, p);
        *p = policy_prec(policy, level, N, tol);
        return MLMC_OK;
    };
    mlmc::ctx_want_xsums(ctx, true);
    int rc = adaptive_core(li0.N, L_max, eps, *opts, gpu, choose, allreduce, user, out, true);
    mlmc::ctx_want_xsums(ctx, false);
    return rc;
}

extern "C" int mlmc_adaptive_run_host(int h0_inv, int L_max, double eps, const mlmc_adaptive_opts* opts,
                                      mlmc_level_sampler_fn sampler, void* sampler_user, mlmc_allreduce_fn allreduce,
                                      void* user, mlmc_result* out) {
    if (!opts || !out || !sampler) return MLMC_EINVAL;
    RoundSampler host = [&](int nlev, const int* lv, const uint64_t* n, const uint64_t* first, const mlmc_precision* pf,
                            const mlmc_precision* pc, const double* tf, const double* tc, double* sums,
                            u64* xs) -> int {
        for (int q = 0; q < nlev; ++q) {
            double* s = sums + (size_t)q * MLMC_SUMS_LEN;
            int rc = sampler(lv[q], n[q], first[q], &pf[q], &pc[q], tf[q], tc[q], s, sampler_user);
            if (rc) return rc;
            // a host sampler returns its slice's sums already rounded: they enter the exact exchange as they
            // are (so the ranks still agree bit for bit; independence of the slicing needs per-sample values)
            if (xs)
                for (int f = 0; f < kXFields; ++f) x_from_double(s[f], xs + (size_t)q * kXLen + f * kXWords);
        }
        return MLMC_OK;
    };
    const int policy = opts->policy == 3 ? 0 : opts->policy;   // no pilot timing over a host sampler
    PrecChooser choose = [&](int level, int N, double tol, mlmc_precision* p) -> int {
        *p = policy_prec(policy, level, N, tol);
        return MLMC_OK;
    };
    return adaptive_core(h0_inv, L_max, eps, *opts, host, choose, allreduce, user, out, true);
}
