# K3b (cluster-resident MINRES, h = 1/128 and 1/256): parity tests, timing against K3c
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -k "cluster_resident or h256" > gpurun_out/pytest_k3b.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_k3b.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "streamed_minres or mgcg_edge" >> gpurun_out/pytest_k3b.log 2>&1; echo "pytest2 rc=$?"; tail -3 gpurun_out/pytest_k3b.log
timeout 900 python tools/k3b_time.py > gpurun_out/k3b_time.jsonl 2>&1; echo "time rc=$?"; cat gpurun_out/k3b_time.jsonl
