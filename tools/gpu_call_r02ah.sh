# coarse-half fork next to a K3b fine half: level pass times with and without (tuning build)
mkdir -p gpurun_out
MLMC_TUNING=1 python -c "from paper_2503_05533_b200 import build as b; b.build(force=True)" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for f in 1 0 1; do MLMC_TUNING=1 MLMC_SCHED_FORK=$f timeout 600 python tools/fork_probe.py; done
