#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python scripts/bench_permute.py > gpurun_out/permute.log 2>&1
TAG=k3v2 SKIPS="1336 1343" bash scripts/gpu_ncu_ids.sh
