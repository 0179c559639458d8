#!/bin/bash
# K3g staged bulk-store epilogue + K3 accumulator/CTA variants: parity tests, C5 and C3 node timings
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q -rA -k "k3g or c5 or variants or p7 or error_study" > gpurun_out/pytest_epi.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_epi.log
bash scripts/gpu_nodevar.sh C5 4 base seg30:JETB200_TCG_SEG=30 seg5:JETB200_TCG_SEG=5
bash scripts/gpu_nodevar.sh C3 14 base acc4:JETB200_K3_ACC=4 ctas1:JETB200_K3_CTAS=1
