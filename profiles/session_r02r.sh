#!/bin/bash
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for ms in none 20 100; do
echo "== nvidia-smi -lms $ms" >> gpurun_out/r02r_m2c.txt
if [ "$ms" != none ]; then
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -i 0 -lms $ms > /dev/null 2>&1 &
SMI=$!
sleep 1
fi
timeout 300 python profiles/m2_protocol.py 5 >> gpurun_out/r02r_m2c.txt 2>&1
if [ "$ms" != none ]; then kill $SMI; fi
done
cat gpurun_out/r02r_m2c.txt
