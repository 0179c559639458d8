#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe scripts/tma_probe.cu > gpurun_out/tma_probe_build.log 2>&1
for v in 0 1 2 3 4 5; do timeout 60 /tmp/tma_probe $v >> gpurun_out/tma_probe.txt 2>&1; echo "v$v rc=$?" >> gpurun_out/tma_probe.txt; done
cat gpurun_out/tma_probe.txt
