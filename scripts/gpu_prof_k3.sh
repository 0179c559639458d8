#!/bin/bash
# K3 stage split + one full ncu capture of the top C3 contraction launch
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TAG=${TAG:-k3}
timeout 900 python scripts/k3_split.py C3 6 ${MODES:-0,32,3,35,31,63} > gpurun_out/k3_split_$TAG.log 2>&1
CFG=C3 SPS=2 TAG=$TAG timeout 1500 bash scripts/gpu_prof_top.sh
