#!/bin/bash
# GPU test suite + the default bench line (run under gpurun; logs land in gpurun_out/)
#   bash scripts/gpu_suite.sh [pytest -k expression]
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
K=${1:+-k "$1"}
eval timeout 2400 python -m pytest tests -m gpu -q -rA $K > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
