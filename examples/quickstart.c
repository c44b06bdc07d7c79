/* quickstart.c -- the C ABI of include/mlmc.h used directly from C (no Python, no PyTorch).
 *
 *   plan configs[1]'s problem -> lend a device workspace -> one coupled pass of every level with
 *   binary64 MINRES at the level's tolerance -> Algorithm 2 (adaptive MPML) on configs[3].
 *
 * Build (tests/test_gpu_parity.py::test_c_quickstart does this):
 *   gcc -std=c99 -O2 examples/quickstart.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2503_05533_b200 -lmlmc -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2503_05533_b200 -o quickstart
 */
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "mlmc.h"

#define CHECK(call)                                                                   \
    do {                                                                              \
        int rc_ = (call);                                                             \
        if (rc_ != MLMC_OK) {                                                         \
            fprintf(stderr, "%s failed: %s (%s)\n", #call, mlmc_strerror(rc_),       \
                    ctx ? mlmc_last_error(ctx) : "");                                 \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

int main(void) {
    mlmc_ctx* ctx = NULL;
    /* configs[1]: expcov KL, m = 64, sigma^2 = 1, l = 0.3, h = 1/8 .. 1/64 */
    mlmc_problem pr = {MLMC_FIELD_EXPCOV_KL, 64, 1.0, 0.3, 2.0, 8, 2, 3, 0};
    CHECK(mlmc_plan_levels(&pr, &ctx));

    size_t bytes = 0;
    CHECK(mlmc_workspace_bytes(ctx, 3, 20000, &bytes));
    void* ws = NULL;
    if (cudaMalloc(&ws, bytes) != cudaSuccess) { fprintf(stderr, "cudaMalloc failed\n"); return 1; }
    CHECK(mlmc_bind_workspace(ctx, ws, bytes, NULL));

    const uint64_t N[4] = {20000, 5000, 1200, 300};
    const double tol[4] = {1e-4, 1e-5, 1e-6, 1e-8};
    const mlmc_precision minres = {MLMC_SOLVER_MINRES, MLMC_FMT_F64, MLMC_FMT_F64, MLMC_FMT_F64, MLMC_FMT_F64, 0, 0};
    double estimate = 0.0;
    for (int l = 0; l < 4; ++l) {
        mlmc_level_sums s;
        CHECK(mlmc_sample_level(ctx, l, N[l], 1, 0, &minres, &minres, tol[l], l ? tol[l - 1] : tol[0], &s, NULL));
        const double mean = s.sum_y / s.n, var = s.sum_y2 / s.n - mean * mean;
        printf("level %d: n %.0f  mean Y %.6e  var Y %.3e  MINRES steps %.1f (fine) %.1f (coarse)  failed %.0f\n", l,
               s.n, mean, var, s.iters_f / s.n, l ? s.iters_c / s.n : 0.0, s.n_fail);
        estimate += mean;
    }
    printf("fixed-N MLMC estimate of E[Q]: %.6f\n", estimate);
    mlmc_destroy(ctx);
    ctx = NULL;

    /* Algorithm 2 on configs[3]: m = 128, l = 0.1, h0 = 1/8, L_max = 5, eps = 1e-3, k_p = 0.05 */
    mlmc_problem pr4 = {MLMC_FIELD_EXPCOV_KL, 128, 1.0, 0.1, 2.0, 8, 2, 5, 0};
    CHECK(mlmc_plan_levels(&pr4, &ctx));
    CHECK(mlmc_bind_workspace(ctx, ws, bytes, NULL));
    mlmc_adaptive_opts o = {0.05, 1e-10, 1.0, 100, 0, 0, 1, 100, 4, 0, 0};
    mlmc_result r;
    CHECK(mlmc_adaptive_run(ctx, 1e-3, &o, NULL, NULL, &r));
    printf("adaptive MPML: estimate %.6f  L %d  rounds %d  N_0 %llu\n", r.estimate, r.L, r.rounds,
           (unsigned long long)r.N[0]);
    mlmc_destroy(ctx);
    cudaFree(ws);
    const int ok = estimate > 0.030 && estimate < 0.038 && r.estimate > 0.030 && r.estimate < 0.038;
    printf("%s\n", ok ? "ok" : "UNEXPECTED");
    return ok ? 0 : 2;
}
