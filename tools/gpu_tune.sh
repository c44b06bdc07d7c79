#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python tools/check_variants.py > gpurun_out/check_variants.log 2>&1; echo "check rc=$?"
cat gpurun_out/check_variants.log | cut -c1-400
timeout 600 python tools/tune_minres.py > gpurun_out/tune.log 2>&1; echo "tune rc=$?"
cat gpurun_out/tune.log
if [ -n "$WITH_TESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log; fi
