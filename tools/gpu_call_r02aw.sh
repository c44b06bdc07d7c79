# K3 h = 1/16 and 1/32 capped at 128 registers (4 CTAs per SM) vs the defaults (tuning build)
mkdir -p gpurun_out
MLMC_TUNING=1 python -c "from paper_2503_05533_b200 import build as b; b.build(force=True)" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
export MLMC_TUNING=1
timeout 300 python tools/tune_minres.py
for v in "0 0" "4 0" "0 7" "4 7" "0 0"; do
  set -- $v
  echo "N16 v$1 N32 v$2: $(MLMC_MINRES_TILE_N16=$1 MLMC_MINRES_TILE_N32=$2 STEP_PROBE_QUICK=1 timeout 120 python tools/step_probe.py 2>&1 | tail -1)"
done
