#!/bin/bash
# One gpurun call: GPU suite, the default bench line, ncu evidence for K2 (C3), K3g (C5), K4 (C4).
#   /usr/local/graft/bin/gpurun --timeout 5400 -- bash scripts/gpu_evidence.sh
set -x
mkdir -p gpurun_out
bash scripts/gpu_suite.sh
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.log; echo "rc=$?" >> gpurun_out/bench_c3.log
CFG=C3 SPS=2 TAG=k2 KREGEX='gett_kernel<float' timeout 1500 bash scripts/gpu_prof.sh
CFG=C5 SPS=1 TAG=k3g KREGEX='gett_tcg' timeout 1200 bash scripts/gpu_prof.sh
CFG=C4 SPS=1 TAG=k4 KREGEX='gett_dmma' timeout 1200 bash scripts/gpu_prof.sh
ls -la gpurun_out
