#!/bin/bash
# Measure the ALU peaks (tools/peak_alu.cu) with the SM clocks sampled during the run.
# Output: gpurun_out/peaks.json (one JSON line + clocks summary), gpurun_out/peaks_clocks.csv
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peak_alu tools/peak_alu.cu || exit 1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap \
    --format=csv -lms 100 > gpurun_out/peaks_clocks.csv &
SMI=$!
sleep 0.5
/tmp/peak_alu > gpurun_out/peaks_raw.json; rc=$?
kill $SMI
python tools/clocks_summary.py gpurun_out/peaks_clocks.csv > gpurun_out/peaks_clocks.json
cat gpurun_out/peaks_raw.json gpurun_out/peaks_clocks.json
exit $rc
