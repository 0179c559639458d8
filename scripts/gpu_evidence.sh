#!/bin/bash
# One gpurun call for the round's evidence: GPU suite + default C3 bench line (gpu_round.sh), the
# C4 / C5 bench lines (gpu_lines.sh), ncu launch lists + top-kernel captures + sanitizers (gpu_ncu.sh)
#   /usr/local/graft/bin/gpurun --timeout 7200 -- bash scripts/gpu_evidence.sh
bash scripts/gpu_round.sh
bash scripts/gpu_lines.sh
bash scripts/gpu_ncu.sh
