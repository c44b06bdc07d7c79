# ncu full capture of the small-mesh K3 launches (h = 1/16, 1/8) of the bench step
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
CMD="python bench.py --steps 2 --warmup 3 --no-extras"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:minres_tile_kernel<.int.(16|8)," -s 8 -c 4 -o /tmp/prof_small -f $CMD > gpurun_out/ncu_small.log 2>&1
echo "full rc=$?"
ncu -i /tmp/prof_small.ncu-rep --page raw --csv > gpurun_out/prof_small.raw.csv
ncu -i /tmp/prof_small.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_small.src.csv 2>/dev/null; echo "src rc=$?"
ls -la gpurun_out/prof_small*
