#!/bin/bash
# A/B of the streamed-mesh MG-PCG kernels (tiled default vs MLMC_MG_GM=plain), parity, ncu of the tiled one.
python -m pytest tests/test_gpu_parity.py -x -q -k "mgcg" 2>&1 | tail -2
timeout 300 python tools/mg_fine.py 148 1e-6 mg 2>&1 | tail -3
MLMC_MG_GM=plain timeout 300 python tools/mg_fine.py 148 1e-6 mg 2>&1 | tail -3
[ "$1" = "ncu" ] && bash tools/gpu_ncu_mgg.sh
true
