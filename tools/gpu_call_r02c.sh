mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_dd.py -x -q > gpurun_out/pytest_dd.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dd.log
tail -30 gpurun_out/pytest_dd.log
timeout 600 python tools/dd_time.py > gpurun_out/dd_time.json 2> gpurun_out/dd_time.err; echo "dd_time rc=$?"
cat gpurun_out/dd_time.json; tail -5 gpurun_out/dd_time.err
