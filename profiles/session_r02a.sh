#!/bin/bash
# round 2, session a: cross-process IPC flag probe on one GPU (R = 2, 4, 8) + baseline bench of HEAD
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02a_smi.txt 2>&1
nvidia-smi -q | grep -i -A3 "compute mode\|MIG" >> gpurun_out/r02a_smi.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o /tmp/ipcp.so profiles/microbench/ipc_flag_probe.cu
for R in 2 4 8; do
  timeout 120 python profiles/microbench/ipc_flag_probe.py $R 200 >> gpurun_out/r02a_ipc.txt 2>&1; echo "R=$R rc=$?" >> gpurun_out/r02a_ipc.txt
done
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
echo bench_rc=$?
cat gpurun_out/r02a_ipc.txt
