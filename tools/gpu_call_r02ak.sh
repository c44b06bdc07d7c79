# stream-priority variants of the concurrent configs[1] step (tuning build), with the job-trace timeline
mkdir -p gpurun_out
MLMC_TUNING=1 python -c "from paper_2503_05533_b200 import build as b; b.build(force=True)" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
export MLMC_TUNING=1
for p in 1 3 4 5 1; do
  echo "prio $p: $(MLMC_SCHED_PRIO=$p STEP_PROBE_QUICK=1 timeout 300 python tools/step_probe.py 2>&1 | tail -1)"
done
python -c "import torch; print(torch.cuda.Stream.priority_range())"
