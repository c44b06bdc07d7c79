mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_dd.py -x -q > gpurun_out/pytest_dd.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dd.log
tail -3 gpurun_out/pytest_dd.log
timeout 600 python tools/dd_time.py > gpurun_out/dd_time.json 2> gpurun_out/dd_time.err; echo "dd_time rc=$?"
cat gpurun_out/dd_time.json
timeout 300 python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1; rc=$?; echo "plain rc=$rc"; tail -3 gpurun_out/sanitize_plain.log
if [ $rc -eq 0 ]; then
  timeout 1500 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck rc=$?"
  tail -8 gpurun_out/sanitize_memcheck.log
fi
