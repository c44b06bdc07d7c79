# chunk sums with 512-thread CTAs: parity subset, step, launch list
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for i in 1 2 3; do echo "step: $(STEP_PROBE_QUICK=1 timeout 120 python tools/step_probe.py 2>&1 | tail -1)"; done
CMD="python bench.py --steps 2 --warmup 3 --no-extras"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
