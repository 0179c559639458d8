#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "k3g" > gpurun_out/pytest_ys.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ys.log
for YS in 2 3 4; do JETB200_TCG_YS=$YS timeout 600 python scripts/node_bench.py C5 3 > gpurun_out/node_C5_ys$YS.txt 2>&1; done
