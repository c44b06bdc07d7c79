# ncu evidence of round 2 (one ncu pass per call; reports exported to CSV on the box, .ncu-rep removed):
# launch list of the bench step, full capture of the top MINRES kernels, K4 at configs[2] level 2 (fp16, fp32)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
CMD="python bench.py --steps 2 --warmup 3 --no-extras"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:minres_tile_kernel<.int.(64|32)," -s 6 -c 3 -o /tmp/prof_minres -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
ncu -i /tmp/prof_minres.ncu-rep --page raw --csv > gpurun_out/prof_minres.raw.csv
ncu -i /tmp/prof_minres.ncu-rep --page source --csv --kernel-name regex:minres_tile_kernel --launch-skip 0 --launch-count 1 > gpurun_out/prof_minres.source.csv 2>/dev/null
for UF in h s; do
  C3="python tools/c3_one.py 2 $UF 20000"
  $C3 > gpurun_out/c3_one_2$UF.log 2>&1 && cat gpurun_out/c3_one_2$UF.log && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches_2$UF.csv $C3 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:chol_(factor|refine)_kernel<.int.32," -s 2 -c 2 \
     -o /tmp/prof_chol_2$UF -f $C3 > gpurun_out/ncu_chol_2$UF.log 2>&1
  echo "chol $UF rc=$?"
  ncu -i /tmp/prof_chol_2$UF.ncu-rep --page raw --csv > gpurun_out/prof_chol_2$UF.raw.csv
done
ls -la gpurun_out | tail -12
