// host_kl.cpp -- plan-time Karhunen-Loeve data (runs once per plan, not per sample).
//
// BASELINE field (R11): covariance sigma2 exp(-|x1-y1|/l - |x2-y2|/l) on (0,1)^2
// is the product of two 1D exponential kernels exp(-c|s-t|), c = 1/l, on [0,1].
// The 1D eigenpairs solve the transcendental equation
//     tan w = 2 c w / (w^2 - c^2)   <=>   (w^2 - c^2) sin w = 2 c w cos w,
// eigenvalue theta = 2c / (w^2 + c^2), eigenfunction N (cos w s + (c/w) sin w s).
// Exactly one root lies in each ((k-1) pi, k pi): the function changes sign at
// the ends of every such interval, so plain bisection inside it is safe.
// 2D eigenvalues lambda_ij = sigma2 (theta_i theta_j), kept m largest, ties
// (i,j)/(j,i) broken by ascending i then j (R11).  Truncation per P:564.
// Paper field Eq. (20): Phi[p][j-1] = sqrt(sigma2) j^-q sin(2 pi j x1) cos(2 pi j x2).
#include <algorithm>
#include <cmath>
#include <thread>

#include "internal.h"

namespace mlmc {

static double tr_residual(double w, double c) { return (w * w - c * c) * std::sin(w) - 2.0 * c * w * std::cos(w); }

static double root_in_interval(double lo, double hi, double c) {
    double flo = tr_residual(lo, c);
    for (int it = 0; it < 2000; ++it) {
        double mid = lo + 0.5 * (hi - lo);
        if (!(mid > lo && mid < hi)) break;
        double fm = tr_residual(mid, c);
        if (fm == 0.0) return mid;
        if ((fm > 0.0) == (flo > 0.0)) { lo = mid; flo = fm; } else { hi = mid; }
    }
    return lo + 0.5 * (hi - lo);
}

int kl_modes(double sigma2, double corr_len, int m, KLModes& out) {
    if (!(corr_len > 0.0) || m < 1 || !(sigma2 > 0.0)) return MLMC_EINVAL;
    const double pi = 3.141592653589793238462643383279502884;
    const double c = 1.0 / corr_len;
    out.c = c;
    const int K = m + 1;   // 1D modes beyond m can never reach the top m (theta strictly decreasing)
    out.w.resize(K);
    out.nrm.resize(K);
    std::vector<double> theta(K);
    for (int k = 1; k <= K; ++k) {
        double lo = (k - 1) * pi, hi = k * pi;
        if (k == 1) lo = 1e-9 * pi;   // f(0) = 0 is the trivial root
        double w = root_in_interval(lo, hi, c);
        out.w[k - 1] = w;
        theta[k - 1] = 2.0 * c / (w * w + c * c);
        // ||cos(w s) + r sin(w s)||^2_{L2(0,1)} with r = c / w
        double r = c / w;
        double s2 = std::sin(2.0 * w), c2 = std::cos(2.0 * w);
        double nn = 0.5 * (1.0 + r * r) + 0.25 * (1.0 - r * r) * s2 / w + 0.5 * r * (1.0 - c2) / w;
        out.nrm[k - 1] = 1.0 / std::sqrt(nn);
    }
    struct Cand { double lam; int32_t i, j; };
    std::vector<Cand> cand;
    cand.reserve((size_t)K * K);
    for (int i = 1; i <= K; ++i)
        for (int j = 1; j <= K; ++j) cand.push_back({sigma2 * (theta[i - 1] * theta[j - 1]), i, j});
    std::stable_sort(cand.begin(), cand.end(), [](const Cand& a, const Cand& b) {
        if (a.lam != b.lam) return a.lam > b.lam;
        if (a.i != b.i) return a.i < b.i;
        return a.j < b.j;
    });
    out.ik.resize(m); out.jk.resize(m); out.lam.resize(m);
    for (int k = 0; k < m; ++k) { out.ik[k] = cand[k].i; out.jk[k] = cand[k].j; out.lam[k] = cand[k].lam; }
    return MLMC_OK;
}

void build_phi(const mlmc_problem& pr, const KLModes& kl, int N, std::vector<double>& phi) {
    const int P = 2 * N * N, m = pr.m;
    const double h = 1.0 / N;
    const double pi = 3.141592653589793238462643383279502884;
    phi.assign((size_t)P * m, 0.0);
    // distinct centroid coordinates per axis: (i + 1/3) h and (i + 2/3) h
    int Kused = 0;
    if (pr.field == MLMC_FIELD_EXPCOV_KL)
        for (int k = 0; k < m; ++k) Kused = std::max(Kused, std::max(kl.ik[k], kl.jk[k]));
    std::vector<double> sq(m);
    if (pr.field == MLMC_FIELD_EXPCOV_KL)
        for (int k = 0; k < m; ++k) sq[k] = std::sqrt(kl.lam[k]);
    // rows j of the mesh in parallel (the h = 1/512 table at m = 256 is 1.07 GB); each entry is
    // computed by the same expression whichever thread writes it
    auto rows = [&](int j_begin, int j_end) {
        std::vector<double> e1(Kused + 1), e2(Kused + 1);
        for (int j = j_begin; j < j_end; ++j)
            for (int i = 0; i < N; ++i)
                for (int up = 0; up < 2; ++up) {
                    // lower triangle {(i,j),(i+1,j),(i+1,j+1)}: centroid (i+2/3, j+1/3) h
                    // upper triangle {(i,j),(i+1,j+1),(i,j+1)}: centroid (i+1/3, j+2/3) h
                    double x1 = (i + (up ? 1.0 : 2.0) / 3.0) * h;
                    double x2 = (j + (up ? 2.0 : 1.0) / 3.0) * h;
                    double* row = &phi[((size_t)2 * (j * N + i) + up) * m];
                    if (pr.field == MLMC_FIELD_EXPCOV_KL) {
                        for (int q = 1; q <= Kused; ++q) {
                            double w = kl.w[q - 1], r = kl.c / w;
                            e1[q] = kl.nrm[q - 1] * (std::cos(w * x1) + r * std::sin(w * x1));
                            e2[q] = kl.nrm[q - 1] * (std::cos(w * x2) + r * std::sin(w * x2));
                        }
                        for (int k = 0; k < m; ++k) row[k] = sq[k] * e1[kl.ik[k]] * e2[kl.jk[k]];
                    } else {
                        double sd = std::sqrt(pr.sigma2);
                        for (int jj = 1; jj <= m; ++jj)
                            row[jj - 1] = sd * std::pow((double)jj, -pr.q_decay) * std::sin(2.0 * pi * jj * x1) *
                                          std::cos(2.0 * pi * jj * x2);
                    }
                }
    };
    const size_t work = (size_t)P * m;
    const int nt = work < (1u << 20) ? 1 : (int)std::min<unsigned>(std::max(1u, std::thread::hardware_concurrency()), 32u);
    if (nt == 1) {
        rows(0, N);
        return;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) {
        const int jb = (int)((long long)N * t / nt), je = (int)((long long)N * (t + 1) / nt);
        if (jb < je) pool.emplace_back(rows, jb, je);
    }
    for (auto& th : pool) th.join();
}

void build_sep_modes(const mlmc_problem& pr, const KLModes& kl, SepModes& out) {
    const int m = pr.m;
    std::vector<int32_t> a(m), b(m);
    std::vector<double> c(m);
    int K = 0;
    for (int k = 0; k < m; ++k) {
        if (pr.field == MLMC_FIELD_EXPCOV_KL) {     // sqrt(lambda_k) e_{ik}(x1) e_{jk}(x2)
            a[k] = kl.ik[k] - 1;
            b[k] = kl.jk[k] - 1;
            c[k] = std::sqrt(kl.lam[k]);
        } else {                                    // sqrt(sigma2) j^-q sin(2 pi j x1) cos(2 pi j x2), j = k + 1
            a[k] = b[k] = k;
            c[k] = std::sqrt(pr.sigma2) * std::pow((double)(k + 1), -pr.q_decay);
        }
        K = std::max(K, std::max(a[k], b[k]) + 1);
    }
    out.K = K;
    out.aoff.assign(K + 1, 0);
    for (int k = 0; k < m; ++k) ++out.aoff[a[k] + 1];
    for (int i = 0; i < K; ++i) out.aoff[i + 1] += out.aoff[i];
    std::vector<int32_t> pos(out.aoff.begin(), out.aoff.end() - 1);
    out.mk.assign(m, 0);
    out.mb.assign(m, 0);
    out.mc.assign(m, 0.0);
    for (int k = 0; k < m; ++k) {                   // stable: modes of one a keep their KL order
        const int e = pos[a[k]]++;
        out.mk[e] = k;
        out.mb[e] = b[k];
        out.mc[e] = c[k];
    }
}

void build_sep_tables(const mlmc_problem& pr, const KLModes& kl, const SepModes& sm, int N, std::vector<double>& tab) {
    const int K = sm.K;
    const double h = 1.0 / N;
    const double pi = 3.141592653589793238462643383279502884;
    tab.assign((size_t)4 * N * K, 0.0);
    for (int i = 0; i < N; ++i)
        for (int t = 0; t < 2; ++t) {
            const double x = (i + (t ? 2.0 : 1.0) / 3.0) * h;
            for (int q = 0; q < K; ++q) {
                double f, g;
                if (pr.field == MLMC_FIELD_EXPCOV_KL) {   // the same 1D function in both directions
                    const double w = kl.w[q], r = kl.c / w;
                    f = g = kl.nrm[q] * (std::cos(w * x) + r * std::sin(w * x));
                } else {
                    f = std::sin(2.0 * pi * (q + 1) * x);
                    g = std::cos(2.0 * pi * (q + 1) * x);
                }
                tab[((size_t)t * N + i) * K + q] = f;
                tab[((size_t)(2 + t) * N + i) * K + q] = g;
            }
        }
}

}  // namespace mlmc
