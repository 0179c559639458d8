#!/bin/bash
# ncu evidence for one bench config (under gpurun, 1 GPU):
#   1. launch list of one bench step (gpu__time_duration + dram bytes per launch)
#   2. one `--set full` capture of the longest launch of the kernel class KREGEX
# env: CFG (C3), SPS (slices per step, 2), TAG, KREGEX (gett), EXTRA (extra bench args)
mkdir -p gpurun_out
CFG=${CFG:-C3}; SPS=${SPS:-2}; TAG=${TAG:-top}; KREGEX=${KREGEX:-gett}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export JETB200_PDL=0
BENCH="python bench.py --config $CFG --steps 1 --warmup 1 --slices-per-step $SPS --no-e2e --no-cpu-baseline $EXTRA"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${CFG}_${TAG}.csv $BENCH > /dev/null 2>&1
SKIP=$(python - <<PY
import sys; sys.path.insert(0, 'scripts')
from launches import load
per, meta = load('gpurun_out/launches_${CFG}_${TAG}.csv')
import re
g = [i for i in sorted(per) if re.search(r'${KREGEX}', meta[i][0])]
t = max(g, key=lambda i: per[i]['gpu__time_duration.sum'])
print(g.index(t))
PY
)
echo "top ${KREGEX} index $SKIP" > gpurun_out/prof_${CFG}_${TAG}.txt
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"${KREGEX}" -s $SKIP -c 1 \
  -o gpurun_out/prof_${CFG}_${TAG} -f $BENCH >> gpurun_out/prof_${CFG}_${TAG}.txt 2>&1
python scripts/ncu_summary.py gpurun_out/prof_${CFG}_${TAG}.ncu-rep >> gpurun_out/prof_${CFG}_${TAG}.txt 2>&1
python scripts/launches.py gpurun_out/launches_${CFG}_${TAG}.csv > gpurun_out/launches_${CFG}_${TAG}_summary.txt 2>&1
