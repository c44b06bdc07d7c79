#!/bin/bash
# ncu full capture of the MG-PCG kernel (K3m, h = 1/64) from tools/minres_step_time.py 20 mgcg.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
CMD="python tools/minres_step_time.py 20 mgcg"
$CMD > gpurun_out/mg_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:mgcg_kernel<.int.64" -s 1 -c 1 \
   -o gpurun_out/prof_mg -f $CMD > gpurun_out/ncu_mg.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_mg.log
