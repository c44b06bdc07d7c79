# K3 tile-shape A/B at h = 1/16 (R = 8, 16 systems per 128-thread CTA) and h = 1/32 (R = 8, 2 systems per CTA)
mkdir -p gpurun_out
MLMC_TUNING=1 python -c "from paper_2503_05533_b200 import build as b; b.build(force=True)" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
MLMC_TUNING=1 timeout 600 python tools/tune_minres.py
for v in "0 0" "3 0" "0 6" "3 6"; do
  set -- $v
  echo "N16 v$1 N32 v$2: $(MLMC_TUNING=1 MLMC_MINRES_TILE_N16=$1 MLMC_MINRES_TILE_N32=$2 STEP_PROBE_QUICK=1 timeout 300 python tools/step_probe.py 2>&1 | tail -1)"
done
