#!/bin/bash
# ncu full capture of one K3c launch (h = 1/256, 148 systems x 60 steps) after a plain run.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
CMD="python tools/big_levels.py 148 60"
$CMD > gpurun_out/k3c_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:minres_stream" -s 4 -c 1 \
   -o gpurun_out/prof_k3c -f $CMD > gpurun_out/ncu_k3c.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_k3c.log
