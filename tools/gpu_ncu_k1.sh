#!/bin/bash
# ncu full capture of the KL-synthesis kernel (K1, DMMA) on the configs[1] level-3 fields (h = 1/64, m = 64).
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
CMD="python bench.py --steps 1 --warmup 3 --no-extras"
$CMD > gpurun_out/k1_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:field_dmma" -s 12 -c 2 \
   -o gpurun_out/prof_k1 -f $CMD > gpurun_out/ncu_k1.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_k1.log
