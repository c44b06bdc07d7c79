#!/bin/bash
# K3c cluster-split A/B (CTAs per system 1/2/4/8) on configs[4] levels 5 and 6, then the streamed parity tests.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "streamed" 2>&1 | tail -2
for cs in 1 2 4 8; do
  MLMC_STREAM_CLUSTER=$cs timeout 300 python tools/k3c_cluster.py 5 100 3.4e-6 gpurun_out/l5_cs$cs.npy
done
for cs in 1 8; do
  MLMC_STREAM_CLUSTER=$cs timeout 300 python tools/k3c_cluster.py 6 100 1.9e-7 gpurun_out/l6_cs$cs.npy
done
python -c "
import numpy as np
for l, cs in ((5, (2, 4, 8)), (6, (8,))):
    a = np.load(f'gpurun_out/l{l}_cs1.npy')
    for c in cs:
        b = np.load(f'gpurun_out/l{l}_cs{c}.npy')
        print(l, c, 'max rel dQ', np.max(np.abs(a[:, :2] - b[:, :2]) / np.abs(a[:, :2])), 'iters diff max', np.max(np.abs(a[:, 2:4] - b[:, 2:4])))
"
