#!/bin/bash
# K3 per-item cost diagnostics on C3: MMA-pass sweep, ncu of a tm=3 and a tm=4 node; K2 tiny-node ranking
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -rA -k "k3g_streamed" > gpurun_out/pytest_k3g.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k3g.log
bash scripts/gpu_nodevar.sh C3 14 base pass1:JETB200_DEBUG_K3_PASSES=1
timeout 600 python scripts/node_bench.py C3 12 0 > gpurun_out/nodes_C3_k2tiny.txt 2>&1
export JETB200_PDL=0
for n in 928 552; do
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -c 1 \
    -o gpurun_out/prof_C3_node$n -f python scripts/node_once.py C3 $n > gpurun_out/prof_C3_node$n.txt 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_C3_node$n.ncu-rep >> gpurun_out/prof_C3_node$n.txt 2>&1
  ncu -i gpurun_out/prof_C3_node$n.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_C3_node${n}_source.csv 2>&1
done
