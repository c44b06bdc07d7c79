"""Condense tools/gpu_tune.sh output (check_variants / tune_minres JSON lines) to one line per variant."""
import json
import sys
for l in sys.stdin:
    l = l.strip()
    if not l.startswith("{"):
        print(l[:300]); continue
    d = json.loads(l)
    if "iters_gpu" in d:
        print("CHK", d["N"], d["variant"], "iterdiff %.3f qerr/bound %.2e relres/tol %.3f" % (
            d["worst_rel_iter_diff"], d["worst_q_err_over_bound"], d["max_true_relres_over_tol"]))
    elif "ms_per_launch" in d:
        print("TUNE", d["N"], d["variant"], "%.3f ms  %.2f TF" % (d["ms_per_launch"], d["fp64_tflops_alg"]))
    else:
        print(l[:300])
