# job-trace timeline of the configs[1] step with fine / coarse halves told apart (tuning build)
mkdir -p gpurun_out
MLMC_TUNING=1 python -c "from paper_2503_05533_b200 import build as b; b.build(force=True)" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
MLMC_TUNING=1 timeout 300 python tools/step_trace.py gpurun_out/step_trace2.json | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(d['step_ms_events'], d['span_us'], d['mean_busy_sms']); [print(k, v) for k, v in d['meshes'].items()]; print(d['busy_sms_per_25us'])"
