mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity_full.py -x -q -s --durations=0 > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
tail -30 gpurun_out/pytest_full.log
