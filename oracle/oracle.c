/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU reference for the per-sample hot path of
 * the MPML method of arXiv 2503.05533 ("Exploiting Inexact Computations in
 * Multilevel Monte Carlo ...").  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with the CUDA product in
 * paper_2503_05533_b200/ and the product never loads it.
 *
 * Citation keys: "P:n" = /root/reference/PAPER.md line n (the paper's LaTeX);
 * "Rk" = reading k of DESIGN.md section 3 (where the paper is silent).
 *
 * Everything is IEEE binary64 unless a function says it emulates a lower
 * precision (Algorithm 1), in which case every operation is rounded
 * to the target format with round-to-nearest-even (standard model).
 *
 * Parity pins (tests/test_oracle_*.py) tie every function below to something
 * other than itself: Philox KAT vectors, KL eigen-relation by Nystrom
 * quadrature, closed-form Poisson QoI, manufactured solution O(h^2),
 * brute-force dense solves, the paper's Table 1, Corollary 4.4, etc.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>

#define OR_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------- */
/* 1. Counter-based RNG: Philox4x32-10 + Box-Muller (R12).                     */
/*    The paper only says omega_j ~ N(0, sigma^2); the generator is a  */
/*    reading: key = (seed_lo, seed_hi), counter = (t, k_lo, k_hi, level).     */
/* ------------------------------------------------------------------------- */
OR_EXPORT void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                                uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {            /* key schedule: Weyl increments between rounds */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* xi[0..m) ~ N(0,1) for sample `index` of level `level` (R12). */
OR_EXPORT void or_normals(uint64_t seed, int level, uint64_t index, int m, double* xi) {
    const double two_pi = 6.283185307179586476925286766559;
    for (int t = 0; 2 * t < m; ++t) {
        uint32_t ctr[4] = {(uint32_t)t, (uint32_t)(index & 0xffffffffu),
                           (uint32_t)(index >> 32), (uint32_t)level};
        uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
        uint32_t r[4];
        or_philox4x32_10(ctr, key, r);
        double u1 = ((double)(r[0] >> 5) * 67108864.0 + (double)(r[1] >> 6) + 0.5)
                    * (1.0 / 9007199254740992.0);
        double u2 = ((double)(r[2] >> 5) * 67108864.0 + (double)(r[3] >> 6) + 0.5)
                    * (1.0 / 9007199254740992.0);
        double rad = sqrt(-2.0 * log(u1));
        xi[2 * t] = rad * cos(two_pi * u2);
        if (2 * t + 1 < m) xi[2 * t + 1] = rad * sin(two_pi * u2);
    }
}

/* ------------------------------------------------------------------------- */
/* 2. KL expansion of the separable exponential covariance (BASELINE field,   */
/*    R11): C(x,y) = sigma2 * exp(-|x1-y1|/l - |x2-y2|/l) on (0,1)^2.          */
/*    1D kernel exp(-c|x-y|), c = 1/l, on [0,1]:                              */
/*      roots w_k > 0 of f(w) = (w^2 - c^2) sin w - 2 c w cos w,              */
/*      theta_k = 2c / (w_k^2 + c^2),                                         */
/*      e_k(x) = N_k (cos w_k x + (c/w_k) sin w_k x).                          */
/*    The truncation at m terms is the "truncated Karhunen-Loeve expansion"   */
/*    of P:564.                                                               */
/* ------------------------------------------------------------------------- */
static double kl_f(double w, double c) {
    return (w * w - c * c) * sin(w) - 2.0 * c * w * cos(w);
}

/* First K positive roots by sign-change scan on a fine grid, then bisection to
 * the last representable bracket. */
OR_EXPORT int or_kl_roots_1d(double corr_len, int K, double* w_out) {
    const double c = 1.0 / corr_len;
    const double step = 1e-3;
    int found = 0;
    double a = step, fa = kl_f(a, c);
    while (found < K) {
        double b = a + step, fb = kl_f(b, c);
        if (fa == 0.0) {
            w_out[found++] = a;
        } else if ((fa < 0.0) != (fb < 0.0)) {
            double lo = a, hi = b, flo = fa;
            for (int it = 0; it < 200; ++it) {
                double mid = 0.5 * (lo + hi);
                if (mid <= lo || mid >= hi) break;
                double fm = kl_f(mid, c);
                if ((fm < 0.0) == (flo < 0.0)) { lo = mid; flo = fm; } else { hi = mid; }
            }
            w_out[found++] = 0.5 * (lo + hi);
        }
        a = b; fa = fb;
        if (a > 1e7) return -1;
    }
    return 0;
}

OR_EXPORT double or_kl_theta(double corr_len, double w) {
    const double c = 1.0 / corr_len;
    return 2.0 * c / (w * w + c * c);
}

/* N_k from the closed form of int_0^1 (cos wx + (c/w) sin wx)^2 dx. */
OR_EXPORT double or_kl_norm(double corr_len, double w) {
    const double c = 1.0 / corr_len;
    double r = c / w;
    double I = 0.5 * (1.0 + r * r) + (1.0 - r * r) * sin(2.0 * w) / (4.0 * w)
             + c * (1.0 - cos(2.0 * w)) / (2.0 * w * w);
    return 1.0 / sqrt(I);
}

OR_EXPORT double or_kl_efun(double corr_len, double w, double x) {
    const double c = 1.0 / corr_len;
    return or_kl_norm(corr_len, w) * (cos(w * x) + (c / w) * sin(w * x));
}

/* The m largest 2D eigenvalues lambda_ij = sigma2 theta_i theta_j (1-based i,j),
 * sorted descending, ties broken by ascending i then ascending j (R11).
 * Uses K = m+1 1D modes: any pair with i > m or j > m is strictly smaller than
 * the m pairs (1,1..m).  Outputs ik, jk (1-based), lam (length m) and the 1D
 * roots w1d[0..m] (w1d[i-1] is the root of 1D mode i). */
OR_EXPORT int or_kl_modes(double sigma2, double corr_len, int m, int* ik, int* jk,
                          double* lam, double* w1d) {
    int K = m + 1;
    if (or_kl_roots_1d(corr_len, K, w1d) != 0) return -1;
    double* th = (double*)malloc(sizeof(double) * K);
    for (int i = 0; i < K; ++i) th[i] = or_kl_theta(corr_len, w1d[i]);
    int total = K * K;
    int* ci = (int*)malloc(sizeof(int) * total);
    int* cj = (int*)malloc(sizeof(int) * total);
    double* cl = (double*)malloc(sizeof(double) * total);
    int n = 0;
    for (int i = 1; i <= K; ++i)
        for (int j = 1; j <= K; ++j) {
            /* theta_i theta_j first: IEEE multiplication is commutative, so the
             * (i,j)/(j,i) ties of R11 stay exact ties */
            ci[n] = i; cj[n] = j; cl[n] = sigma2 * (th[i - 1] * th[j - 1]); ++n;
        }
    /* selection of the m largest, plain O(m * K^2) */
    char* used = (char*)calloc(total, 1);
    for (int k = 0; k < m; ++k) {
        int best = -1;
        for (int q = 0; q < total; ++q) {
            if (used[q]) continue;
            if (best < 0 || cl[q] > cl[best] ||
                (cl[q] == cl[best] && (ci[q] < ci[best] || (ci[q] == ci[best] && cj[q] < cj[best]))))
                best = q;
        }
        used[best] = 1;
        ik[k] = ci[best]; jk[k] = cj[best]; lam[k] = cl[best];
    }
    free(used); free(cl); free(cj); free(ci); free(th);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* 3. Mesh and random field at the triangle centroids (R10).                  */
/*    Uniform N x N cells of size h = 1/N on (0,1)^2, each cell (i,j) split   */
/*    along its SW-NE diagonal into                                           */
/*       T_L = {(i,j), (i+1,j), (i+1,j+1)}   (tri index 2*(j*N+i))            */
/*       T_U = {(i,j), (i+1,j+1), (i,j+1)}   (tri index 2*(j*N+i)+1)          */
/*    Coefficient: one-point centroid rule per triangle.                      */
/* ------------------------------------------------------------------------- */
static void tri_vertices(int N, int t, int vi[3], int vj[3]) {
    int cell = t / 2, i = cell % N, j = cell / N;
    if (t % 2 == 0) { vi[0] = i; vj[0] = j; vi[1] = i + 1; vj[1] = j; vi[2] = i + 1; vj[2] = j + 1; }
    else            { vi[0] = i; vj[0] = j; vi[1] = i + 1; vj[1] = j + 1; vi[2] = i; vj[2] = j + 1; }
}

OR_EXPORT void or_centroid(int N, int t, double* x1, double* x2) {
    int vi[3], vj[3];
    tri_vertices(N, t, vi, vj);
    double h = 1.0 / N;
    *x1 = (vi[0] + vi[1] + vi[2]) * h / 3.0;
    *x2 = (vj[0] + vj[1] + vj[2]) * h / 3.0;
}

typedef struct {
    int field;         /* 0 = separable exponential covariance KL (BASELINE), 1 = paper Eq. (20) */
    int m;             /* number of KL terms (field 0) or s (field 1) */
    double sigma2;     /* field variance sigma^2 (field 0) / omega_j variance (field 1) */
    double corr_len;   /* correlation length l (field 0) */
    double q_decay;    /* j^{-q} decay (field 1) */
    int h0_inv;        /* 1/h0 */
    /* filled by or_problem_init (field 0): the m retained modes and the 1D roots */
    int* ik; int* jk; double* lam; double* w1d; int K_used;
} or_problem;

OR_EXPORT int or_problem_init(or_problem* pr) {
    pr->ik = NULL; pr->jk = NULL; pr->lam = NULL; pr->w1d = NULL; pr->K_used = 0;
    if (pr->field != 0) return 0;
    int m = pr->m;
    pr->ik = (int*)malloc(sizeof(int) * m);
    pr->jk = (int*)malloc(sizeof(int) * m);
    pr->lam = (double*)malloc(sizeof(double) * m);
    pr->w1d = (double*)malloc(sizeof(double) * (m + 1));
    if (or_kl_modes(pr->sigma2, pr->corr_len, m, pr->ik, pr->jk, pr->lam, pr->w1d) != 0) return -1;
    for (int k = 0; k < m; ++k) {
        if (pr->ik[k] > pr->K_used) pr->K_used = pr->ik[k];
        if (pr->jk[k] > pr->K_used) pr->K_used = pr->jk[k];
    }
    return 0;
}

OR_EXPORT void or_problem_free(or_problem* pr) {
    free(pr->ik); free(pr->jk); free(pr->lam); free(pr->w1d);
    pr->ik = NULL; pr->jk = NULL; pr->lam = NULL; pr->w1d = NULL;
}

/* a_T = exp(g(centroid_T)) for all 2N^2 triangles, g evaluated term by term. */
OR_EXPORT int or_field_triangles(const or_problem* pr, int N, const double* xi, double* a_out) {
    int P = 2 * N * N;
    if (pr->field == 0) {
        /* g(x) = sum_k sqrt(lambda_k) xi_k e_{i_k}(x1) e_{j_k}(x2); the 1D values
         * e_i(x1), e_j(x2) of the modes in use are evaluated once per triangle. */
        int m = pr->m, K = pr->K_used;
        double* e1 = (double*)malloc(sizeof(double) * (K + 1));
        double* e2 = (double*)malloc(sizeof(double) * (K + 1));
        for (int t = 0; t < P; ++t) {
            double x1, x2;
            or_centroid(N, t, &x1, &x2);
            for (int i = 1; i <= K; ++i) {
                e1[i] = or_kl_efun(pr->corr_len, pr->w1d[i - 1], x1);
                e2[i] = or_kl_efun(pr->corr_len, pr->w1d[i - 1], x2);
            }
            double g = 0.0;
            for (int k = 0; k < m; ++k)
                g += sqrt(pr->lam[k]) * xi[k] * e1[pr->ik[k]] * e2[pr->jk[k]];
            a_out[t] = exp(g);
        }
        free(e1); free(e2);
    } else {
        /* Eq. (20): a = exp(sum_{j=1}^s omega_j j^{-q} sin(2 pi j x1) cos(2 pi j x2)),
         * omega_j ~ N(0, sigma^2) -> omega_j = sigma * xi_j. */
        const double pi = 3.14159265358979323846264338328;
        double sigma = sqrt(pr->sigma2);
        for (int t = 0; t < P; ++t) {
            double x1, x2;
            or_centroid(N, t, &x1, &x2);
            double g = 0.0;
            for (int j = 1; j <= pr->m; ++j)
                g += sigma * xi[j - 1] * pow((double)j, -pr->q_decay)
                     * sin(2.0 * pi * j * x1) * cos(2.0 * pi * j * x2);
            a_out[t] = exp(g);
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* 4. Generic P1 element-by-element assembly.                         */
/*    Interior unknown p = (j-1)(N-1) + (i-1) for node (i,j), 1<=i,j<=N-1.     */
/*    Dirichlet rows/cols eliminated (u = 0 on the boundary).          */
/*    Element stiffness a_T |T| G G^T with G the barycentric gradients.       */
/*    Load: b_i = int f phi_i; f == 1 exactly gives |T|/3 per element         */
/*    ("f == 1"); f_kind 1 is the test-only manufactured right-hand     */
/*    side f = 2 pi^2 sin(pi x) sin(pi y) with the 3-point edge-midpoint rule. */
/*    Output: lower band AB[p*(bw+1) + d] = A[p][p-d], d = 0..bw, bw = N-1,    */
/*    or (if dense != NULL) the full dense n x n matrix.                      */
/* ------------------------------------------------------------------------- */
static int node_index(int N, int i, int j) {
    if (i <= 0 || j <= 0 || i >= N || j >= N) return -1;
    return (j - 1) * (N - 1) + (i - 1);
}

OR_EXPORT int or_assemble(int N, const double* a_tri, int f_kind, double* AB, double* dense, double* b) {
    const double pi = 3.14159265358979323846264338328;
    int n = (N - 1) * (N - 1), bw = N - 1;
    double h = 1.0 / N;
    if (AB) memset(AB, 0, sizeof(double) * (size_t)n * (bw + 1));
    if (dense) memset(dense, 0, sizeof(double) * (size_t)n * n);
    memset(b, 0, sizeof(double) * n);
    for (int t = 0; t < 2 * N * N; ++t) {
        int vi[3], vj[3];
        tri_vertices(N, t, vi, vj);
        double X[3], Y[3];
        for (int q = 0; q < 3; ++q) { X[q] = vi[q] * h; Y[q] = vj[q] * h; }
        /* barycentric gradients: grad phi_q = (Y[q+1]-Y[q+2], X[q+2]-X[q+1]) / (2|T|) */
        double det = (X[1] - X[0]) * (Y[2] - Y[0]) - (X[2] - X[0]) * (Y[1] - Y[0]);
        double area = 0.5 * fabs(det);
        double gx[3], gy[3];
        for (int q = 0; q < 3; ++q) {
            int q1 = (q + 1) % 3, q2 = (q + 2) % 3;
            gx[q] = (Y[q1] - Y[q2]) / det;
            gy[q] = (X[q2] - X[q1]) / det;
        }
        double fl[3] = {0, 0, 0};
        if (f_kind == 0) {
            for (int q = 0; q < 3; ++q) fl[q] = area / 3.0;
        } else {
            /* edge-midpoint rule: weights |T|/3 at the 3 midpoints, phi_q = 1/2 at the
             * two midpoints of edges touching vertex q, 0 at the opposite one */
            for (int e = 0; e < 3; ++e) {
                int pa = e, pb = (e + 1) % 3;
                double mx = 0.5 * (X[pa] + X[pb]), my = 0.5 * (Y[pa] + Y[pb]);
                double f = 2.0 * pi * pi * sin(pi * mx) * sin(pi * my);
                fl[pa] += area / 3.0 * f * 0.5;
                fl[pb] += area / 3.0 * f * 0.5;
            }
        }
        for (int r = 0; r < 3; ++r) {
            int pr_ = node_index(N, vi[r], vj[r]);
            if (pr_ < 0) continue;
            b[pr_] += fl[r];
            for (int s = 0; s < 3; ++s) {
                int ps = node_index(N, vi[s], vj[s]);
                if (ps < 0) continue;
                double kval = a_tri[t] * area * (gx[r] * gx[s] + gy[r] * gy[s]);
                if (dense) dense[(size_t)pr_ * n + ps] += kval;
                if (AB && ps <= pr_) {
                    int d = pr_ - ps;
                    if (d > bw) {                   /* the SW-NE hypotenuse: its coupling must be 0 */
                        if (kval != 0.0) return -2;
                        continue;
                    }
                    AB[(size_t)pr_ * (bw + 1) + d] += kval;
                }
            }
        }
    }
    return 0;
}

/* y = A x with A given by its lower band (symmetric). */
OR_EXPORT void or_band_matvec(int n, int bw, const double* AB, const double* x, double* y) {
    for (int i = 0; i < n; ++i) y[i] = 0.0;
    for (int i = 0; i < n; ++i) {
        y[i] += AB[(size_t)i * (bw + 1)] * x[i];
        for (int d = 1; d <= bw && d <= i; ++d) {
            double a = AB[(size_t)i * (bw + 1) + d];
            y[i] += a * x[i - d];
            y[i - d] += a * x[i];
        }
    }
}

/* ------------------------------------------------------------------------- */
/* 5. Direct solves in binary64 (reference solver, "double precision    */
/*    Cholesky").  Band: L[i*(bw+1)+d] = L(i, i-d).  Returns -1 on a          */
/*    non-positive pivot.                                                     */
/* ------------------------------------------------------------------------- */
OR_EXPORT int or_chol_band(int n, int bw, const double* AB, double* L) {
    for (int j = 0; j < n; ++j) {
        for (int i = j; i < n && i <= j + bw; ++i) {
            double s = AB[(size_t)i * (bw + 1) + (i - j)];
            int k0 = i - bw > 0 ? i - bw : 0;
            for (int k = k0; k < j; ++k)
                s -= L[(size_t)i * (bw + 1) + (i - k)] * L[(size_t)j * (bw + 1) + (j - k)];
            if (i == j) {
                if (!(s > 0.0)) return -1;
                L[(size_t)j * (bw + 1)] = sqrt(s);
            } else {
                L[(size_t)i * (bw + 1) + (i - j)] = s / L[(size_t)j * (bw + 1)];
            }
        }
    }
    return 0;
}

OR_EXPORT void or_chol_band_solve(int n, int bw, const double* L, const double* b, double* x) {
    double* y = (double*)malloc(sizeof(double) * n);
    for (int i = 0; i < n; ++i) {
        double s = b[i];
        for (int d = 1; d <= bw && d <= i; ++d) s -= L[(size_t)i * (bw + 1) + d] * y[i - d];
        y[i] = s / L[(size_t)i * (bw + 1)];
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = y[i];
        for (int d = 1; d <= bw && i + d < n; ++d) s -= L[(size_t)(i + d) * (bw + 1) + d] * x[i + d];
        x[i] = s / L[(size_t)i * (bw + 1)];
    }
    free(y);
}

OR_EXPORT int or_chol_dense(int n, const double* A, double* L) {
    memset(L, 0, sizeof(double) * (size_t)n * n);
    for (int j = 0; j < n; ++j) {
        for (int i = j; i < n; ++i) {
            double s = A[(size_t)i * n + j];
            for (int k = 0; k < j; ++k) s -= L[(size_t)i * n + k] * L[(size_t)j * n + k];
            if (i == j) {
                if (!(s > 0.0)) return -1;
                L[(size_t)j * n + j] = sqrt(s);
            } else {
                L[(size_t)i * n + j] = s / L[(size_t)j * n + j];
            }
        }
    }
    return 0;
}

OR_EXPORT void or_chol_dense_solve(int n, const double* L, const double* b, double* x) {
    double* y = (double*)malloc(sizeof(double) * n);
    for (int i = 0; i < n; ++i) {
        double s = b[i];
        for (int k = 0; k < i; ++k) s -= L[(size_t)i * n + k] * y[k];
        y[i] = s / L[(size_t)i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = y[i];
        for (int k = i + 1; k < n; ++k) s -= L[(size_t)k * n + i] * x[k];
        x[i] = s / L[(size_t)i * n + i];
    }
    free(y);
}

/* ------------------------------------------------------------------------- */
/* 6. MINRES: x0 = 0, no preconditioner (R9), all arithmetic in    */
/*    binary64, stop at the first k with phibar_k / ||b|| <= tol,     */
/*    i.e. the relative-residual criterion of Eq. (2) with C = 1 (P:70-73,   */
/*    P:102).  Textbook Paige-Saunders recurrences (Lanczos + Givens).         */
/*    status: 0 converged, 1 max_iter reached.                                */
/* ------------------------------------------------------------------------- */
static double dot(int n, const double* a, const double* b) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

OR_EXPORT int or_minres_band(int n, int bw, const double* AB, const double* b, double tol,
                             int max_iter, double* x, int* iters_out, double* relres_out) {
    double *r1 = malloc(sizeof(double) * n), *r2 = malloc(sizeof(double) * n),
           *y = malloc(sizeof(double) * n), *v = malloc(sizeof(double) * n),
           *w = malloc(sizeof(double) * n), *w1 = malloc(sizeof(double) * n),
           *w2 = malloc(sizeof(double) * n);
    for (int i = 0; i < n; ++i) { r1[i] = r2[i] = y[i] = b[i]; w[i] = w2[i] = 0.0; x[i] = 0.0; }
    double beta1 = sqrt(dot(n, b, b));
    double oldb = 0.0, beta = beta1, dbar = 0.0, epsln = 0.0, phibar = beta1;
    double cs = -1.0, sn = 0.0;
    int k = 0, status = 1;
    if (beta1 == 0.0) { status = 0; goto done; }
    while (k < max_iter) {
        ++k;
        for (int i = 0; i < n; ++i) v[i] = y[i] / beta;
        or_band_matvec(n, bw, AB, v, y);
        if (k >= 2)
            for (int i = 0; i < n; ++i) y[i] -= (beta / oldb) * r1[i];
        double alpha = dot(n, v, y);
        for (int i = 0; i < n; ++i) y[i] -= (alpha / beta) * r2[i];
        for (int i = 0; i < n; ++i) { r1[i] = r2[i]; r2[i] = y[i]; }
        oldb = beta;
        beta = sqrt(dot(n, r2, r2));
        double oldeps = epsln;
        double delta = cs * dbar + sn * alpha;
        double gbar = sn * dbar - cs * alpha;
        epsln = sn * beta;
        dbar = -cs * beta;
        double gamma = hypot(gbar, beta);
        if (gamma < DBL_MIN) gamma = DBL_MIN;
        cs = gbar / gamma;
        sn = beta / gamma;
        double phi = cs * phibar;
        phibar = sn * phibar;
        for (int i = 0; i < n; ++i) {
            w1[i] = w2[i];
            w2[i] = w[i];
            w[i] = (v[i] - oldeps * w1[i] - delta * w2[i]) / gamma;
            x[i] += phi * w[i];
        }
        if (phibar / beta1 <= tol) { status = 0; break; }
    }
done:
    if (iters_out) *iters_out = k;
    if (relres_out) {
        or_band_matvec(n, bw, AB, x, y);
        double s = 0.0;
        for (int i = 0; i < n; ++i) { double r = b[i] - y[i]; s += r * r; }
        *relres_out = beta1 > 0 ? sqrt(s) / beta1 : 0.0;
    }
    free(r1); free(r2); free(y); free(v); free(w); free(w1); free(w2);
    return status;
}

/* 6b. MINRES from an initial guess x0 (NEXT-4, coarse-to-fine; reading R32): Paige-Saunders on  */
/*     A e = r0 = b - A x0, x = x0 + e, stopped at the first k with phibar_k <= tol ||b|| -- the relative-   */
/*     residual criterion of Eq. (2) is relative to ||b||, not to ||r0||.  x0 = 0 gives or_minres_band.      */
OR_EXPORT int or_minres_band_x0(int n, int bw, const double* AB, const double* b, const double* x0, double tol,
                                int max_iter, double* x, int* iters_out, double* relres_out) {
    double *r1 = malloc(sizeof(double) * n), *r2 = malloc(sizeof(double) * n),
           *y = malloc(sizeof(double) * n), *v = malloc(sizeof(double) * n),
           *w = malloc(sizeof(double) * n), *w1 = malloc(sizeof(double) * n),
           *w2 = malloc(sizeof(double) * n);
    or_band_matvec(n, bw, AB, x0, y);
    for (int i = 0; i < n; ++i) { r1[i] = r2[i] = y[i] = b[i] - y[i]; w[i] = w2[i] = 0.0; x[i] = x0[i]; }
    double bnorm = sqrt(dot(n, b, b));
    double beta1 = sqrt(dot(n, r1, r1));
    double oldb = 0.0, beta = beta1, dbar = 0.0, epsln = 0.0, phibar = beta1;
    double cs = -1.0, sn = 0.0;
    int k = 0, status = 1;
    if (beta1 <= tol * bnorm) { status = 0; goto done; }
    while (k < max_iter) {
        ++k;
        for (int i = 0; i < n; ++i) v[i] = y[i] / beta;
        or_band_matvec(n, bw, AB, v, y);
        if (k >= 2)
            for (int i = 0; i < n; ++i) y[i] -= (beta / oldb) * r1[i];
        double alpha = dot(n, v, y);
        for (int i = 0; i < n; ++i) y[i] -= (alpha / beta) * r2[i];
        for (int i = 0; i < n; ++i) { r1[i] = r2[i]; r2[i] = y[i]; }
        oldb = beta;
        beta = sqrt(dot(n, r2, r2));
        double oldeps = epsln;
        double delta = cs * dbar + sn * alpha;
        double gbar = sn * dbar - cs * alpha;
        epsln = sn * beta;
        dbar = -cs * beta;
        double gamma = hypot(gbar, beta);
        if (gamma < DBL_MIN) gamma = DBL_MIN;
        cs = gbar / gamma;
        sn = beta / gamma;
        double phi = cs * phibar;
        phibar = sn * phibar;
        for (int i = 0; i < n; ++i) {
            w1[i] = w2[i];
            w2[i] = w[i];
            w[i] = (v[i] - oldeps * w1[i] - delta * w2[i]) / gamma;
            x[i] += phi * w[i];
        }
        if (phibar <= tol * bnorm) { status = 0; break; }
    }
done:
    if (iters_out) *iters_out = k;
    if (relres_out) {
        or_band_matvec(n, bw, AB, x, y);
        double s = 0.0;
        for (int i = 0; i < n; ++i) { double r = b[i] - y[i]; s += r * r; }
        *relres_out = bnorm > 0 ? sqrt(s) / bnorm : 0.0;
    }
    free(r1); free(r2); free(y); free(v); free(w); free(w1); free(w2);
    return status;
}

/* ------------------------------------------------------------------------- */
/* 7. Precision emulation: round to a binary format with t          */
/*    significand bits (incl. the implicit one), minimum normal exponent      */
/*    emin and largest finite xmax; round-to-nearest-even; gradual underflow; */
/*    overflow -> +-inf.  fmt: 0 = q43 (E4M3-like, R17), 1 = half, 2 = single, */
/*    3 = double.                                                             */
/* ------------------------------------------------------------------------- */
OR_EXPORT double or_round(double x, int fmt) {
    int t, emin; double xmax;
    switch (fmt) {
        case 0: t = 4;  emin = -6;   xmax = 240.0; break;        /* q43: 4 exp bits, 3 stored sig bits, bias 7 */
        case 1: t = 11; emin = -14;  xmax = 65504.0; break;
        case 2: t = 24; emin = -126; xmax = (double)FLT_MAX; break;
        default: return x;
    }
    if (x == 0.0 || !isfinite(x)) return x;
    int E;
    frexp(x, &E);                   /* |x| = f 2^E, 0.5 <= f < 1: leading bit exponent E-1 */
    int e = E - 1;
    if (e < emin) e = emin;         /* subnormal range: fixed quantum */
    double q = ldexp(1.0, e - (t - 1));
    double r = nearbyint(x / q) * q;  /* default rounding mode: nearest-even */
    if (fabs(r) > xmax) return x > 0 ? INFINITY : -INFINITY;
    return r;
}

/* ------------------------------------------------------------------------- */
/* 8. Algorithm 1 (iterative refinement) around a banded Cholesky   */
/*    factor computed with every operation rounded to u_f; substitutions in    */
/*    u_s (R24: initial solve and corrections both in u_s); residual in u_r    */
/*    rounded to the working precision u (R13); x stored and updated in u.     */
/*    quad = {u_f, u_s, u, u_r} as or_round fmt codes.                          */
/*    status: 0 converged, 1 no convergence after i_max, 2 breakdown (pivot    */
/*    <= 0 or non-finite after rounding), 3 overflow.                          */
/* ------------------------------------------------------------------------- */
static void band_solve_rounded(int n, int bw, const double* L, const double* rhs, double* x, int fs) {
    double* y = (double*)malloc(sizeof(double) * n);
    for (int i = 0; i < n; ++i) {
        double s = or_round(rhs[i], fs);
        for (int d = 1; d <= bw && d <= i; ++d)
            s = or_round(s - or_round(L[(size_t)i * (bw + 1) + d] * y[i - d], fs), fs);
        y[i] = or_round(s / L[(size_t)i * (bw + 1)], fs);
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = y[i];
        for (int d = 1; d <= bw && i + d < n; ++d)
            s = or_round(s - or_round(L[(size_t)(i + d) * (bw + 1) + d] * x[i + d], fs), fs);
        x[i] = or_round(s / L[(size_t)i * (bw + 1)], fs);
    }
    free(y);
}

/* Exported for the Algorithm 1 emulation pins (tests/test_oracle_alg1_minres.py); the
 * arithmetic is band_solve_rounded's, unchanged. */
OR_EXPORT void or_band_solve_rounded(int n, int bw, const double* L, const double* rhs, double* x, int fs) {
    band_solve_rounded(n, bw, L, rhs, x, fs);
}

OR_EXPORT int or_chol_band_rounded(int n, int bw, const double* AB, double* L, int ff) {
    for (int j = 0; j < n; ++j) {
        for (int i = j; i < n && i <= j + bw; ++i) {
            double s = or_round(AB[(size_t)i * (bw + 1) + (i - j)], ff);
            int k0 = i - bw > 0 ? i - bw : 0;
            for (int k = k0; k < j; ++k)
                s = or_round(s - or_round(L[(size_t)i * (bw + 1) + (i - k)] * L[(size_t)j * (bw + 1) + (j - k)], ff), ff);
            if (!isfinite(s)) return 3;
            if (i == j) {
                if (!(s > 0.0)) return 2;
                L[(size_t)j * (bw + 1)] = or_round(sqrt(s), ff);
            } else {
                L[(size_t)i * (bw + 1) + (i - j)] = or_round(s / L[(size_t)j * (bw + 1)], ff);
            }
        }
    }
    return 0;
}

OR_EXPORT int or_ir_band(int n, int bw, const double* AB, const double* b, const int quad[4],
                         double tol, int i_max, double* x, int* steps_out, double* relres_out) {
    int ff = quad[0], fs = quad[1], fu = quad[2], fr = quad[3];
    double* L = (double*)calloc((size_t)n * (bw + 1), sizeof(double));
    double* r = (double*)malloc(sizeof(double) * n);
    double* d = (double*)malloc(sizeof(double) * n);
    double* Ax = (double*)malloc(sizeof(double) * n);
    int status = or_chol_band_rounded(n, bw, AB, L, ff);          /* step 1 */
    int i = 0;
    double bn = sqrt(dot(n, b, b)), rel = 1.0;
    if (status != 0) goto done;
    band_solve_rounded(n, bw, L, b, x, fs);                       /* step 2 */
    for (int q = 0; q < n; ++q) x[q] = or_round(x[q], fu);
    status = 1;
    for (i = 0; i <= i_max; ++i) {                                 /* step 3 */
        /* step 4: r_i = b - A x_i in u_r, rounded to the storage precision u */
        for (int q = 0; q < n; ++q) Ax[q] = 0.0;
        for (int q = 0; q < n; ++q) {
            Ax[q] = or_round(Ax[q] + or_round(AB[(size_t)q * (bw + 1)] * x[q], fr), fr);
            for (int dd = 1; dd <= bw && dd <= q; ++dd) {
                double a = AB[(size_t)q * (bw + 1) + dd];
                Ax[q] = or_round(Ax[q] + or_round(a * x[q - dd], fr), fr);
                Ax[q - dd] = or_round(Ax[q - dd] + or_round(a * x[q], fr), fr);
            }
        }
        for (int q = 0; q < n; ++q) r[q] = or_round(or_round(b[q] - Ax[q], fr), fu);
        rel = sqrt(dot(n, r, r)) / bn;
        if (!isfinite(rel)) { status = 3; break; }
        if (rel < tol) { status = 0; break; }                      /* steps 5-6 */
        if (i == i_max) break;
        band_solve_rounded(n, bw, L, r, d, fs);                   /* step 7 */
        for (int q = 0; q < n; ++q) x[q] = or_round(x[q] + or_round(d[q], fu), fu);   /* step 8 */
    }
done:
    if (steps_out) *steps_out = i;
    if (relres_out) *relres_out = rel;
    free(L); free(r); free(d); free(Ax);
    return status;
}

/* ------------------------------------------------------------------------- */
/* 9. One coupled sample: xi = RNG(seed, l, k); the     */
/*    same xi drives the level-l mesh (h_l = h0 2^-l) and the level    */
/*    l-1 mesh; Q = int_D u_h = sum_i x_i int phi_i = h^2 sum_i x_i.           */
/*    solver: 0 = direct fp64 banded Cholesky (O-exact), 1 = MINRES at tol     */
/*    (O-alg), 2 = Algorithm 1 with quad (O-alg).                              */
/*    out[0..7] = Qf, Qc, iters_f, iters_c, relres_f, relres_c, status_f,      */
/*    status_c (coarse entries 0 at level 0).                                  */
/* ------------------------------------------------------------------------- */
OR_EXPORT int or_solve_level_mesh(const or_problem* pr, int N, const double* xi, int solver,
                                  const int quad[4], double tol, int max_iter, double out[4]) {
    int n = (N - 1) * (N - 1), bw = N - 1;
    double h = 1.0 / N;
    double* a = (double*)malloc(sizeof(double) * 2 * N * N);
    double* AB = (double*)malloc(sizeof(double) * (size_t)n * (bw + 1));
    double* b = (double*)malloc(sizeof(double) * n);
    double* x = (double*)malloc(sizeof(double) * n);
    int st = or_field_triangles(pr, N, xi, a);
    if (st == 0) st = or_assemble(N, a, 0, AB, NULL, b);
    int iters = 0;
    double relres = 0.0;
    if (st == 0) {
        if (solver == 0) {
            double* L = (double*)malloc(sizeof(double) * (size_t)n * (bw + 1));
            st = or_chol_band(n, bw, AB, L);
            if (st == 0) or_chol_band_solve(n, bw, L, b, x);
            free(L);
            double* Ax = (double*)malloc(sizeof(double) * n);
            or_band_matvec(n, bw, AB, x, Ax);
            double s = 0, bb = 0;
            for (int i = 0; i < n; ++i) { s += (b[i] - Ax[i]) * (b[i] - Ax[i]); bb += b[i] * b[i]; }
            relres = sqrt(s / bb);
            free(Ax);
        } else if (solver == 1) {
            st = or_minres_band(n, bw, AB, b, tol, max_iter, x, &iters, &relres);
        } else {
            st = or_ir_band(n, bw, AB, b, quad, tol, max_iter, x, &iters, &relres);
        }
    }
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += x[i];
    out[0] = h * h * s;
    out[1] = iters;
    out[2] = relres;
    out[3] = st;
    free(a); free(AB); free(b); free(x);
    return st;
}

OR_EXPORT int or_coupled_sample(const or_problem* pr, int level, uint64_t seed, uint64_t index,
                                int solver, const int quad_f[4], const int quad_c[4],
                                double tol_f, double tol_c, int max_iter, double out[8]) {
    int m = pr->m;
    double* xi = (double*)malloc(sizeof(double) * (m + 1));
    or_normals(seed, level, index, m, xi);
    int Nf = pr->h0_inv << level;
    double of[4] = {0, 0, 0, 0}, oc[4] = {0, 0, 0, 0};
    int st = or_solve_level_mesh(pr, Nf, xi, solver, quad_f, tol_f, max_iter, of);
    if (level > 0) {
        int st2 = or_solve_level_mesh(pr, Nf / 2, xi, solver, quad_c, tol_c, max_iter, oc);
        if (st == 0) st = st2;
    }
    out[0] = of[0]; out[1] = oc[0]; out[2] = of[1]; out[3] = oc[1];
    out[4] = of[2]; out[5] = oc[2]; out[6] = of[3]; out[7] = oc[3];
    free(xi);
    return st;
}
