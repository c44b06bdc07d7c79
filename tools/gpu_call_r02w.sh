mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -x -q -k "C3 or ir_ or half or single or quarter or binary64 or paper_direct or escalation or smoke" > gpurun_out/pytest_k4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_k4.log
for uf in s h; do for lv in 0 1 2; do C3_WS_GB=48 python tools/c3_one.py $lv $uf 100000; done; done
