# job-trace timeline of the configs[1] step (tuning build)
mkdir -p gpurun_out
MLMC_TUNING=1 python -c "from paper_2503_05533_b200 import build as b; b.build(force=True)" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
MLMC_TUNING=1 timeout 300 python tools/step_trace.py gpurun_out/step_trace.json
