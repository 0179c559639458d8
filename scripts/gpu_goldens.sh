#!/bin/bash
# Oracle goldens for plans whose slices do not fit this container's RAM (C4/C5 at width 30), on the
# GPU box's host cores (the oracle is CPU-only: scripts/make_goldens.py imports only oracle/ and
# circuits/), with the GPU test suite running meanwhile.  Usage: bash scripts/gpu_goldens.sh C5:2 C4:4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
(
  for spec in "$@"; do
    cfg=${spec%%:*}; blocks=${spec#*:}
    timeout 5400 python scripts/make_goldens.py $cfg --blocks $blocks > gpurun_out/golden_$cfg.log 2>&1
    echo "rc=$?" >> gpurun_out/golden_$cfg.log
    cp tests/golden/parity_$cfg.json gpurun_out/ 2>/dev/null
  done
) &
GPID=$!
timeout 2400 python -m pytest tests -m gpu -q -rA -k "not C4 and not C5 and not c5" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
wait $GPID
