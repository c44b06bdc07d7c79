# source-level stall profile of K4b (fp16 factor, configs[2] level 2)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
C3="python tools/c3_one.py 2 h 20000"
$C3 > gpurun_out/c3_one_2h.log 2>&1 && cat gpurun_out/c3_one_2h.log && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:chol_refine_kernel<.int.32," -s 1 -c 1 \
   -o /tmp/prof_ref -f $C3 > gpurun_out/ncu_ref.log 2>&1
echo "rc=$?"
ncu -i /tmp/prof_ref.ncu-rep --page source --csv > gpurun_out/prof_ref.source.csv 2>/dev/null
ncu -i /tmp/prof_ref.ncu-rep --page source --csv --print-source cuda > gpurun_out/prof_ref.cuda.csv 2>/dev/null
ls -la gpurun_out/prof_ref*
