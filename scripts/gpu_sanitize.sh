#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on the K3 (TMA and cp.async), K3g, K2, K4, K1 kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export JETB200_GRAPHS=0
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py \
    > gpurun_out/sanitize_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.txt
done
tail -3 gpurun_out/sanitize_*.txt
