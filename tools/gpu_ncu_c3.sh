#!/bin/bash
# ncu full capture of the K4 kernel at one C3 level (LEVEL, UF env), after a plain run.
LEVEL=${LEVEL:-2}; UF=${UF:-h}; NS=${NS:-20000}
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
CMD="python tools/c3_one.py $LEVEL $UF $NS"
$CMD > gpurun_out/c3_one_${LEVEL}${UF}.log 2>&1 && cat gpurun_out/c3_one_${LEVEL}${UF}.log && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chol_ir_kernel -s 2 -c 1 \
   -o gpurun_out/prof_chol_${LEVEL}${UF} -f $CMD > gpurun_out/ncu_chol_${LEVEL}${UF}.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_chol_${LEVEL}${UF}.log
