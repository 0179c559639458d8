#!/bin/bash
# K3g accumulation-segment length on the benched C5 plan: oracle-golden errors, K3g vs K2, node time
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for seg in 4 5 6 7; do
  rm -f gpurun_out/parity_errors.json
  JETB200_TCG_SEG=$seg timeout 900 python -m pytest tests -m gpu -q -k "(benched_plan_golden_slices and C5) or c5_benched_slice_k3g_vs_k2" --timeout 600 --timeout-method thread > gpurun_out/seg_$seg.log 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/parity_errors.json'))
print(json.dumps({'seg': $seg, 'golden_max': d['C5_benched']['max_rel'], 'golden': d['C5_benched']['per_slice'], 'k3g_vs_k2': d['C5_k3g_vs_k2']['rel']}))" >> gpurun_out/segstudy.txt 2>&1
  echo "== seg $seg" >> gpurun_out/segstudy_nodes.txt
  JETB200_TCG_SEG=$seg timeout 600 python scripts/node_bench.py C5 3 2 >> gpurun_out/segstudy_nodes.txt 2>&1
done
