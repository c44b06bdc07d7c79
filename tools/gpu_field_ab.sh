#!/bin/bash
# Separable KL synthesis (K1s, default) vs the P x m one (MLMC_FIELD_KERNEL=dense): parity tests, per-kernel times.
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for v in sep dense; do
  for a in "C5 0 1000000" "C5 1 200000" "C2 0 20000" "C2 3 300" "C5 4 200"; do
    if [ $v = dense ]; then MLMC_FIELD_KERNEL=dense python tools/level_profile.py $a | grep field; else python tools/level_profile.py $a | grep field; fi
  done
done
python tools/first_call_time.py
python bench.py --steps 10 --warmup 3 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2 step', d['ms_per_step'], d['value'], [ (k['kernel'],k['N'],round(k['ms_total'],3)) for k in d['kernels'] if k['kernel']=='field'])"
