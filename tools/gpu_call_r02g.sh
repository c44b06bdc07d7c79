mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -s -k "coarse_to_fine" > gpurun_out/pytest_c2f.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c2f.log
tail -12 gpurun_out/pytest_c2f.log
timeout 300 python tools/c2f_study.py > gpurun_out/c2f_study.jsonl 2> gpurun_out/c2f.err; echo "c2f rc=$?"; cat gpurun_out/c2f_study.jsonl; tail -3 gpurun_out/c2f.err
