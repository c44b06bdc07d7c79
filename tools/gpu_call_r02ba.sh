# longest-first order also at h = 1/16 (kOrderMinN 16, kOrderMax 8192): C2 step A/B (tuning build), parity subset
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
MLMC_TUNING=1 python -c "from paper_2503_05533_b200 import build as b; b.build(force=True)" > gpurun_out/build_t.log 2>&1 || { tail -30 gpurun_out/build_t.log; exit 1; }
export MLMC_TUNING=1
for n in 16 32 16 32 16 32; do
  echo "order from N=$n: $(MLMC_ORDER_MIN_N=$n STEP_PROBE_QUICK=1 timeout 120 python tools/step_probe.py 2>&1 | tail -1)"
done
