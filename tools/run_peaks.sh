#!/bin/bash
# Measure FP64 peaks on the box; clocks sampled during the run.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
./tools/peaks_fp64 > gpurun_out/peaks_fp64.jsonl 2>&1
RC=$?
kill $SMI
nproc > gpurun_out/host_cores.txt; lscpu | head -20 >> gpurun_out/host_cores.txt
exit $RC
