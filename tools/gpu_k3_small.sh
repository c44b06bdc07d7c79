#!/bin/bash
# A/B of the h = 1/8 and 1/16 K3 variants (conductances in shared memory, more systems per SM)
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
for v in 0 1 2 3; do MLMC_MINRES_TILE_N8=$v python tools/k3_variant.py 0 gpurun_out/l0_v$v.npy; done
for v in 0 3 4; do MLMC_MINRES_TILE_N16=$v python tools/k3_variant.py 1 gpurun_out/l1_v$v.npy; done
python -c "
import numpy as np
for l, vs in ((0, (1, 2, 3)), (1, (3, 4))):
    a = np.load(f'gpurun_out/l{l}_v0.npy')
    for v in vs:
        b = np.load(f'gpurun_out/l{l}_v{v}.npy')
        print(l, v, 'bit-identical' if np.array_equal(a, b) else 'DIFFER')
"
