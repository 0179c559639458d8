#!/bin/bash
# Heaviest nodes of a benched plan under env variants (kernel A/B on real shapes):
#   bash scripts/gpu_nodevar.sh CFG N_NODES tag[:ENV=VAL,ENV=VAL] ...
#   (KIND=2 bash scripts/gpu_nodevar.sh C5 3 ...: rank the nodes of one kernel kind by time x runs)
# one JSON line per node and variant in gpurun_out/nodevar_<CFG>.txt
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CFG=$1; NN=$2; shift 2
OUT=gpurun_out/nodevar_${CFG}.txt
for v in "$@"; do
  tag=${v%%:*}
  envs="X=1"
  if [[ "$v" == *:* ]]; then envs=$(echo "${v#*:}" | tr ',' ' '); fi
  echo "== $tag $envs" >> $OUT
  env $envs timeout 900 python scripts/node_bench.py $CFG $NN $KIND >> $OUT 2> gpurun_out/nodevar_${CFG}_${tag}.log
  echo "rc=$?" >> $OUT
done
