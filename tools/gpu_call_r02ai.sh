# C2 step with the level-3 (h = 1/64) MINRES kernel capped at c persistent CTAs (the other levels take the rest)
mkdir -p gpurun_out
MLMC_TUNING=1 python -c "from paper_2503_05533_b200 import build as b; b.build(force=True)" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
export MLMC_TUNING=1
for g in 1 0; do
for c in 148 128 112 100 90 80; do
  echo "gate $g cap $c: $(MLMC_SCHED_GATE=$g MLMC_TILE_CTAS_N64=$c STEP_PROBE_QUICK=1 timeout 300 python tools/step_probe.py 2>&1 | tail -1)"
done
done
