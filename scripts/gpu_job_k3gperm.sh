#!/bin/bash
# K1-fed K3g: parity (C2 forced, C5 P7 / vs K2), C5 K3g node timings with and without the copies
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q -rA -k "k3g or c5 or C5" > gpurun_out/pytest_k3gperm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k3gperm.log
for v in base noperm:JETB200_TCG_PERM=0; do
  tag=${v%%:*}; envs="X=1"; [[ "$v" == *:* ]] && envs=${v#*:}
  echo "== $tag" >> gpurun_out/nodes_C5_perm.txt
  env $envs timeout 900 python scripts/node_bench.py C5 6 2 >> gpurun_out/nodes_C5_perm.txt 2>&1
done
