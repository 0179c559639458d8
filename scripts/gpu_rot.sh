#!/bin/bash
# K3g rotating accumulator regions: C5 parity (goldens, P7 bound, rot vs single, K3g vs K2) and node timings
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 240 python scripts/node_bench.py C5 1 2 > gpurun_out/rot_smoke.txt 2>&1 || { echo "smoke failed rc=$?" >> gpurun_out/rot_smoke.txt; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -rA -k "C5 or c5 or k3g" --timeout 600 --timeout-method thread > gpurun_out/pytest_rot.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rot.log
for v in X=1 JETB200_TCG_ROT=0 JETB200_TCG_SEG=30; do echo "== $v" >> gpurun_out/nodes_C5_rot.txt; env $v timeout 600 python scripts/node_bench.py C5 3 2 >> gpurun_out/nodes_C5_rot.txt 2>&1; done
