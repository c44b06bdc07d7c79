# ncu full capture of one K3b launch (h = 1/128, 148 systems x 300 steps)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
python tools/k3b_one.py > gpurun_out/k3b_one.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:minres_tile_kernel<.int.128" -s 1 -c 1 -o /tmp/prof_k3b -f python tools/k3b_one.py > gpurun_out/ncu_k3b.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_k3b.ncu-rep --page raw --csv > gpurun_out/prof_k3b.raw.csv
ncu -i /tmp/prof_k3b.ncu-rep --page source --csv > gpurun_out/prof_k3b.src.csv 2> gpurun_out/prof_k3b.src.err; echo "src rc=$?"; head -c 600 gpurun_out/prof_k3b.src.csv
