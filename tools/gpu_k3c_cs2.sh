#!/bin/bash
python __graft_entry__.py > /dev/null 2>&1
MLMC_STREAM_CLUSTER=2 timeout 300 python tools/k3c_cluster.py 6 100 1.9e-7 gpurun_out/x.npy
for cs in 1 2; do
  MLMC_STREAM_CLUSTER=$cs python bench.py --steps 3 --warmup 3 2>/dev/null > gpurun_out/bench_cs$cs.json
  python - "$cs" <<'PY'
import json, sys
cs = sys.argv[1]
d = json.loads(open(f"gpurun_out/bench_cs{cs}.json").read().strip().splitlines()[-1])
k = d["k3c_fine_meshes"]
print("cs", cs, "k3c hbm frac h=1/256", round(k["h=1/256"]["hbm_frac"], 3), "h=1/512", round(k["h=1/512"]["hbm_frac"], 3))
PY
done
