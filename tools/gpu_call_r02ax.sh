# ncu source-level capture of the h = 1/64 MINRES launch (configs[1] level 3 alone)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 300 python tools/tune_minres.py --one 64 > gpurun_out/t64.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:minres_tile_kernel<.int.64" -s 3 -c 1 -o /tmp/prof_k64 -f python tools/tune_minres.py --one 64 > gpurun_out/ncu_k64.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_k64.ncu-rep --page source --csv > gpurun_out/prof_k64.src.csv 2> gpurun_out/prof_k64.src.err; echo "src rc=$?"
ncu -i /tmp/prof_k64.ncu-rep --page raw --csv > gpurun_out/prof_k64.raw.csv
