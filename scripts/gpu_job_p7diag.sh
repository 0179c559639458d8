#!/bin/bash
# P7 error of the benched C5 plan under kernel-path variants (is it the 3xTF32 tensor path, the
# accumulation segments, the K1 copies, or the conditioning of the P7 network in FP32?), while the
# oracle goldens of C5 / C4 run on the host cores
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
(
  for spec in C5:2 C4:4; do
    cfg=${spec%%:*}; blocks=${spec#*:}
    timeout 4800 python scripts/make_goldens.py $cfg --blocks $blocks > gpurun_out/golden_$cfg.log 2>&1
    echo "rc=$?" >> gpurun_out/golden_$cfg.log
    cp tests/golden/parity_$cfg.json gpurun_out/ 2>/dev/null
  done
) &
GPID=$!
for v in "X=1" "JETB200_TC=0" "JETB200_TCG_SEG=0" "JETB200_TCG_SEG=2" "JETB200_TCG_PERM=0" "JETB200_K2S=0"; do
  env $v timeout 900 python scripts/p7_errors.py C5 >> gpurun_out/p7diag_C5.txt 2>> gpurun_out/p7diag_C5.log
done
wait $GPID
