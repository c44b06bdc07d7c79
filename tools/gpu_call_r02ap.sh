# K3 h = 1/8 with four systems per warp (v2, tuning build): per-launch time, step time, bit-identity of the step's sums
mkdir -p gpurun_out
MLMC_TUNING=1 python -c "from paper_2503_05533_b200 import build as b; b.build(force=True)" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
export MLMC_TUNING=1
timeout 300 python tools/tune_minres.py
for v in 0 2 0 2; do
  echo "N8 v$v: $(MLMC_MINRES_TILE_N8=$v STEP_PROBE_QUICK=1 timeout 120 python tools/step_probe.py 2>&1 | tail -1)"
done
