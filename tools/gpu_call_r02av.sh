# small levels on top (MLMC_SCHED_PRIO=6) with / without the gate (tuning build), alternating with the default
mkdir -p gpurun_out
MLMC_TUNING=1 python -c "from paper_2503_05533_b200 import build as b; b.build(force=True)" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
export MLMC_TUNING=1
for v in "1 1" "6 1" "6 0" "1 1" "6 1" "6 0"; do
  set -- $v
  echo "prio $1 gate $2: $(MLMC_SCHED_PRIO=$1 MLMC_SCHED_GATE=$2 STEP_PROBE_QUICK=1 timeout 120 python tools/step_probe.py 2>&1 | tail -1)"
done
