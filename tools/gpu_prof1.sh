#!/bin/bash
# ncu full capture of one MINRES mesh (tools/tune_minres.py --one N), after a plain run.
N=${N:-64}
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
CMD="python tools/tune_minres.py --one $N"
$CMD > gpurun_out/plain_$N.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:minres -s 2 -c 1 \
   -o gpurun_out/prof_N$N -f $CMD > gpurun_out/ncu_N$N.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_N$N.log
