#!/bin/bash
# parity tests of the MINRES path + three C2 bench runs (no extras): quick A/B of a K3 change
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "C1 or C2 or minres_iteration or full_size or concurrent or adaptive_C4" 2>&1 | tail -2
for i in 1 2 3; do python bench.py --steps 20 --warmup 5 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), [round(v['ms_alone'],3) for v in d['per_level'].values()])"; done
