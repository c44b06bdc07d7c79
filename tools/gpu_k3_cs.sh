#!/bin/bash
# A/B of the K3 conductances-in-shared-memory variants (bit-for-bit records + time), then the C2 step.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
python tools/k3_variant.py 3 gpurun_out/l3_v0.npy
MLMC_MINRES_TILE_N64=4 python tools/k3_variant.py 3 gpurun_out/l3_v4.npy
python tools/k3_variant.py 2 gpurun_out/l2_v0.npy
MLMC_MINRES_TILE_N32=4 python tools/k3_variant.py 2 gpurun_out/l2_v4.npy
MLMC_MINRES_TILE_N32=5 python tools/k3_variant.py 2 gpurun_out/l2_v5.npy
python -c "
import numpy as np
for a, b in (('l3_v0', 'l3_v4'), ('l2_v0', 'l2_v4'), ('l2_v0', 'l2_v5')):
    x, y = np.load(f'gpurun_out/{a}.npy'), np.load(f'gpurun_out/{b}.npy')
    print(a, b, 'bit-identical' if np.array_equal(x, y) else f'DIFFER max {np.max(np.abs(x - y)):.3e}')
"
for v in "" "MLMC_MINRES_TILE_N64=4" "MLMC_MINRES_TILE_N64=4 MLMC_MINRES_TILE_N32=4" "MLMC_MINRES_TILE_N64=4 MLMC_MINRES_TILE_N32=5"; do
  echo "== $v"; env $v python bench.py --steps 10 --warmup 3 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['roofline']['frac'])"
done
