# round-2 evidence: bench (no profiler) + ncu launch list of the bench step + full captures of the top
# MINRES kernels and of the K4 kernels at configs[2] level 2 (fp16 / fp32); one ncu pass per call by the guide
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -50 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -2 gpurun_out/bench.err
CMD="python bench.py --steps 2 --warmup 3 --no-extras"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k "regex:minres_tile_kernel<.int.(64|32)," -s 6 -c 3 -o gpurun_out/prof_minres -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
for UF in h s; do
  C3="python tools/c3_one.py 2 $UF 20000"
  $C3 > gpurun_out/c3_one_2$UF.log 2>&1 && cat gpurun_out/c3_one_2$UF.log && \
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:chol_(factor|refine)_kernel<.int.32," -s 2 -c 2 \
     -o gpurun_out/prof_chol_2$UF -f $C3 > gpurun_out/ncu_chol_2$UF.log 2>&1
  echo "chol $UF rc=$?"
done
