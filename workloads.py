"""Seeded synthetic workloads (BASELINE.json configs) -- parameters only, no arithmetic.

Shared by tests/, bench.py and the oracle leg; neither the oracle nor the CUDA
path derives anything from here except these literal parameters.  Inputs are
the standard-normal KL coefficients xi drawn per (seed, level, sample index)
by each side's own Philox4x32-10 implementation.
"""

CONFIGS = {
    # configs[0]: 2-level MLMC, fp64 only, corr 0.3, m = 16, N = (2000, 500), seed 0
    "C1": dict(field="expcov", field_code=0, m=16, sigma2=1.0, corr_len=0.3, h0_inv=8, L_max=1,
               N=[2000, 500], seed=0, tol=1e-12),
    # configs[1]: 4 levels h = 1/8..1/64, m = 64, fixed N, MINRES tols 1e-4/1e-5/1e-6/1e-8, seed 1
    # (variance 1 and corr 0.3 inherited from "same PDE" = configs[0])
    "C2": dict(field="expcov", field_code=0, m=64, sigma2=1.0, corr_len=0.3, h0_inv=8, L_max=3,
               N=[20000, 5000, 1200, 300], tols=[1e-4, 1e-5, 1e-6, 1e-8], seed=1),
    # configs[2]: Cholesky fp16/fp32 + fp64 IR to 1e-10, h = 1/8, 1/16, 1/32, 100000 samples per level
    "C3": dict(field="expcov", field_code=0, m=64, sigma2=1.0, corr_len=0.3, h0_inv=8, L_max=2,
               N=[100000, 100000, 100000], tol=1e-10, seed=2),
    # configs[3]: adaptive to eps = 1e-3, h = 1/8..1/256 (6 levels), m = 128, var 1, corr 0.1
    "C4": dict(field="expcov", field_code=0, m=128, sigma2=1.0, corr_len=0.1, h0_inv=8, L_max=5,
               eps=1e-3, k_p=0.05, seed=4),
    # configs[4]: adaptive to eps = 2.5e-4, h = 1/8..1/512 (7 levels), m = 256, var 2, corr 0.1
    "C5": dict(field="expcov", field_code=0, m=256, sigma2=2.0, corr_len=0.1, h0_inv=8, L_max=6,
               eps=2.5e-4, k_p=0.05, seed=5),
    # the paper's own field, Eq. (20): s = 4, q = 2, sigma = 2
    "EQ20": dict(field="eq20", field_code=1, m=4, sigma2=4.0, corr_len=0.0, q_decay=2.0, h0_inv=8, L_max=4,
                 seed=6),
}
