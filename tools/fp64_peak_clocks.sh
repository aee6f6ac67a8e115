#!/bin/bash
# fp64 peak microbenchmark with nvidia-smi clocks / throttle reasons sampled
# beside it (the denominator of the fp64 roofline fractions)
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 100 > gpurun_out/fp64_clocks.csv &
SMI=$!
sleep 0.5
./tools/microbench/fp64_peak > gpurun_out/fp64_peak.jsonl
kill $SMI
