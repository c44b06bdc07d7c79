#!/bin/bash
# ncu pass: launch list of the bench step, then a full capture of the top MINRES kernels.
set -x
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
CMD="python bench.py --steps 2 --warmup 3 --no-extras"
$CMD > gpurun_out/plain.log 2>&1 && [ -n "$NOLIST" ] ||
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:minres_tile_kernel<.int.(64|32)," -s 6 -c 3 -o gpurun_out/prof_minres -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -3 gpurun_out/ncu_full.log
