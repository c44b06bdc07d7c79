mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_dd.py -x -q > gpurun_out/pytest_dd.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_dd.log
