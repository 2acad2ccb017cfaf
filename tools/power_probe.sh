#!/bin/bash
# sample power / clocks / throttle reasons while the C3 step loop runs
nvidia-smi --query-gpu=power.draw,power.limit,clocks.sm,clocks.mem,clocks_throttle_reasons.active,temperature.gpu --format=csv,noheader -lms 100 > gpurun_out/power.csv &
P=$!
python tools/steptime.py
python tools/steptime.py
kill $P
sort gpurun_out/power.csv | uniq -c | sort -rn | head -15
