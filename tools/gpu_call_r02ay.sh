# screened MINRES pilots of policy 3: policy tests + first-run time of configs[4] at eps = 1e-5
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -q -k "auto" > gpurun_out/pytest_auto.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_auto.log
timeout 600 python tools/auto_probe.py
