# scheduling knobs of the concurrent configs[1] step (tuning build): gate, coarse fork, stream priorities
mkdir -p gpurun_out
MLMC_TUNING=1 python -c "from paper_2503_05533_b200 import build as b; b.build(force=True)" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for v in "1 1 1" "0 1 1" "1 0 1" "1 1 0" "1 1 2" "1 1 1"; do
  set -- $v
  echo "gate $1 fork $2 prio $3: $(MLMC_TUNING=1 MLMC_SCHED_GATE=$1 MLMC_SCHED_FORK=$2 MLMC_SCHED_PRIO=$3 STEP_PROBE_QUICK=1 timeout 300 python tools/step_probe.py 2>&1 | tail -1)"
done
