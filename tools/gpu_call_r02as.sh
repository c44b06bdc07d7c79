# orders formed before the gate: the C2 step (production build, alternating with the previous commit's library) + trace
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
for i in 1 2 3; do echo "new: $(STEP_PROBE_QUICK=1 timeout 120 python tools/step_probe.py 2>&1 | tail -1)"; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['ms_per_step'], d['value'])"
MLMC_TUNING=1 python -c "from paper_2503_05533_b200 import build as b; b.build(force=True)" > gpurun_out/build_t.log 2>&1 || { tail -30 gpurun_out/build_t.log; exit 1; }
MLMC_TUNING=1 timeout 300 python tools/step_trace.py gpurun_out/step_trace3.json | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(d['step_ms_events'], d['span_us'], d['mean_busy_sms']); [print(k, v) for k, v in d['meshes'].items()]; print(d['busy_sms_per_25us'])"
