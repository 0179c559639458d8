#!/bin/bash
# per-warp K3g segment drains (JETB200_TCG_EPI=warp): parity and C5 node timings A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
JETB200_TCG_EPI=warp timeout 240 python scripts/node_bench.py C5 1 2 > gpurun_out/epiwarp_smoke.txt 2>&1 || { echo "smoke failed" >> gpurun_out/epiwarp_smoke.txt; exit 1; }
JETB200_TCG_EPI=warp timeout 1200 python -m pytest tests -m gpu -q -rA -k "C5 or c5 or k3g" --timeout 600 --timeout-method thread > gpurun_out/pytest_epiwarp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_epiwarp.log
for v in X=1 JETB200_TCG_EPI=warp X=2 JETB200_TCG_EPI=warp; do echo "== $v" >> gpurun_out/nodes_C5_epi.txt; env $v timeout 600 python scripts/node_bench.py C5 3 2 >> gpurun_out/nodes_C5_epi.txt 2>&1; done
