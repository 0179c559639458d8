#!/bin/bash
# compute-sanitizer on the K3 (TMA and cp.async), K3g (incl. segmented bulk adds), K2s, K2, K4
# and K1 kernels (scripts/sanitize_case.py).  Usage: bash scripts/gpu_sanitize.sh [tools...]
# (default memcheck).  Each tool under its own timeout.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export JETB200_GRAPHS=0
for tool in ${@:-memcheck}; do
  timeout -s INT 600 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py \
    > gpurun_out/sanitize_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.txt
done
tail -4 gpurun_out/sanitize_*.txt
