#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "k3g" > gpurun_out/pytest_tmt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tmt.log
for T in 6 7; do JETB200_TCG_TMT=$T timeout 600 python scripts/node_bench.py C5 4 > gpurun_out/node_C5_tmt$T.txt 2>&1; done
