#!/bin/bash
# ncu full capture of the global-memory MG-PCG kernel (K3m-g, h = 1/512, 148 systems) from tools/mg_one.py,
# then the small-eps adaptive run with policy 2.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
CMD="python tools/mg_one.py 6 148 1e-6"
$CMD > gpurun_out/mgg_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:mgcg_(gm|tile)_kernel<.int.512" -c 1 \
   -o gpurun_out/prof_mgg -f $CMD > gpurun_out/ncu_mgg.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_mgg.log
