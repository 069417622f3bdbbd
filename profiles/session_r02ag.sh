#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/launch_floor profiles/microbench/launch_floor.cu
/tmp/launch_floor > gpurun_out/r02ag_launch_floor.txt 2>&1
cat gpurun_out/r02ag_launch_floor.txt
