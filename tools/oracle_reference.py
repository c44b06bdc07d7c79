"""The reference QoI of the paper's Section 5.1 experiment: "computed by the standard MLMC algorithm
with tolerance TOL^2 = 2e-8 and a direct, double precision linear solver" -- here the ORACLE's Algorithm 2
(oracle/mlmc.py adaptive_mpml with k_p = None: standard MLMC) driven by the oracle's binary64 banded
Cholesky on every sample (oracle/oracle.c or_chol_band, O-exact), cost model C_l = 2^(gamma l) with gamma = 2
(the paper's choice for its direct-solver section).  Eq. (20) field, s = 4, q = 2, sigma = 2, h0 = 1/8
(P:611).  Calls only oracle/ (TEST INFRASTRUCTURE); writes tests/golden/eq20_reference_tol2_2e-8.json.

    python tools/oracle_reference.py [threads]
"""
import json
import math
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import core as oc  # noqa: E402
from oracle import mlmc as om  # noqa: E402

SEED, N_INIT, L_MAX, TOL2 = 10 ** 8, 10, 6, 2e-8


def main(threads):
    P = oc.OracleProblem(1, 4, 4.0, 0.0, 2.0, 8)      # Eq. (20): s = 4, sigma^2 = 4 (sigma = 2), q = 2
    ex = ThreadPoolExecutor(threads)

    def sampler(level, first, count, tf, tc):
        outs = list(ex.map(lambda k: P.coupled_sample(level, SEED, k, solver=oc.SOLVER_DIRECT),
                           range(first, first + count)))
        assert all(o[6] == 0 and o[7] == 0 for o in outs)
        return [o[0] - o[1] for o in outs], [4.0 ** level] * count
    t0 = time.perf_counter()
    r = om.adaptive_mpml(sampler, math.sqrt(TOL2), 1 / 8, None, L_max=L_MAX, N_init=N_INIT)
    out = {"estimate": r.estimate, "L": r.L, "N": r.N, "means": r.means, "variances": r.variances,
           "rounds": r.rounds, "code": r.code, "TOL2": TOL2, "seed": SEED, "N_init": N_INIT,
           "how": "oracle Algorithm 2 without step 2 (standard MLMC, P:429) at TOL^2 = 2e-8, every sample by the "
                  "oracle's binary64 banded Cholesky (P:681), C_l = 4^l (gamma = 2, P:699); Eq. (20) field s=4, q=2, "
                  "sigma=2, h0=1/8 (P:611); written by tools/oracle_reference.py",
           "seconds": time.perf_counter() - t0, "threads": threads}
    path = os.path.join(ROOT, "tests", "golden", "eq20_reference_tol2_2e-8.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else (os.cpu_count() or 8))
