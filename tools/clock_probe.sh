#!/bin/bash
# SM clock / power while the C2 session runs for a few seconds (diagnostics).
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown --format=csv -lms 100 > gpurun_out/clocks_probe.csv &
SMI=$!
python bench.py --steps 4000 --warmup 10 --no-cpu-baseline ${@} > gpurun_out/clock_bench.json 2>&1
kill $SMI
sort gpurun_out/clocks_probe.csv | uniq -c | sort -rn | head -12
