# fused order with its own counters: parity tests, step time
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do echo "step: $(STEP_PROBE_QUICK=1 timeout 120 python tools/step_probe.py 2>&1 | tail -1)"; done
