# ncu full capture of the separable field kernel (K1s) launches of configs[1] level 3 (h = 1/64 fine with the fused
# order, h = 1/32 coarse)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 300 python tools/level_profile.py C2 3 300 > gpurun_out/lp.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:field_sep_kernel" -s 2 -c 2 \
   -o /tmp/prof_k1s -f python tools/level_profile.py C2 3 300 > gpurun_out/ncu_k1s.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_k1s.ncu-rep --page raw --csv > gpurun_out/prof_k1s.raw.csv
