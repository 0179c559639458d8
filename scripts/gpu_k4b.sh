#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TAG=${TAG:-x}
timeout 600 python scripts/node_bench.py C4 6 > gpurun_out/node_C4_$TAG.txt 2>&1
timeout 600 python scripts/node_bench.py G88d8 4 > gpurun_out/node_G88d8_$TAG.txt 2>&1
