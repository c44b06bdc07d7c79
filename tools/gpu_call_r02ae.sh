# K3b cluster-size A/B (tuning build): h = 1/128 on 8-CTA clusters of 128 threads; h = 1/64 on 2-CTA clusters (v7)
mkdir -p gpurun_out
MLMC_TUNING=1 python -c "from paper_2503_05533_b200 import build as b; b.build(force=True)" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
export MLMC_TUNING=1
MLMC_MINRES_CLUSTER_N128=8 timeout 600 python tools/k3b_time.py --one 2>&1 | head -2 | sed 's/^/CL8 /'
timeout 300 python tools/k3b_ab.py /tmp/v0.json && MLMC_MINRES_K3B_N64=1 timeout 300 python tools/k3b_ab.py /tmp/v7.json && python -c "
import json, numpy as np
a=np.array(json.load(open('/tmp/v0.json'))); b=np.array(json.load(open('/tmp/v7.json')))
print('v7 vs v0: max |dQ|/Q', np.max(np.abs(a[:,:2]-b[:,:2])/np.abs(a[:,:2])), 'max dsteps', np.max(np.abs(a[:,2:4]-b[:,2:4])), 'status', np.max(b[:,6:8]), 'relres max', b[:,4].max())"
for v in 0 1; do
  MLMC_MINRES_K3B_N64=$v timeout 300 python tools/tune_minres.py --one 64 | sed "s/^/N64 v$v /"
  echo "N64 k3b=$v step: $(MLMC_MINRES_K3B_N64=$v STEP_PROBE_QUICK=1 timeout 300 python tools/step_probe.py 2>&1 | tail -1)"
done
