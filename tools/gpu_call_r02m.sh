mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -k "ir_step_counts" > gpurun_out/pytest_ir.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_ir.log | cut -c1-3000
