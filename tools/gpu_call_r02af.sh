# K3b: parity tests (h = 1/128, 1/256 vs oracle and K3c; h = 1/64 cluster path bit-identical to the tile) + fine-mesh bench leg
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -k "cluster" > gpurun_out/pytest_k3b.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_k3b.log
timeout 600 python -c "
import json, sys; sys.argv=['bench.py']
import bench
print(json.dumps(bench.fine_leg(0, __import__('torch')), indent=1))" > gpurun_out/fine_leg.json 2>&1; echo "leg rc=$?"; cat gpurun_out/fine_leg.json | head -60
