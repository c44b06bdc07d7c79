#!/bin/bash
# K4 ncu pass at one C3 level (LEVEL, UF, NS env): launch list + full capture of the h=1/32 kernels.
LEVEL=${LEVEL:-2}; UF=${UF:-h}; NS=${NS:-20000}
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
CMD="python tools/c3_one.py $LEVEL $UF $NS"
$CMD > gpurun_out/c3_one_${LEVEL}${UF}.log 2>&1 && cat gpurun_out/c3_one_${LEVEL}${UF}.log && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches_${LEVEL}${UF}.csv $CMD > /dev/null 2>&1; \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:chol_(factor|refine)_kernel<.int.32," -s 2 -c 2 \
   -o gpurun_out/prof_chol_${LEVEL}${UF} -f $CMD > gpurun_out/ncu_chol_${LEVEL}${UF}.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_chol_${LEVEL}${UF}.log
