#!/bin/bash
# full ncu capture of the longest K2 (gett_kernel) launch of the bench config, from a launch list
mkdir -p gpurun_out
CFG=${CFG:-C3}; SPS=${SPS:-64}; TAG=${TAG:-k2}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export JETB200_PDL=0
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:gett_kernel --log-file gpurun_out/launches_${CFG}_${TAG}.csv python bench.py --config $CFG --steps 1 --warmup 1 \
  --slices-per-step $SPS --no-e2e --no-cpu-baseline > /dev/null 2>&1
SKIP=$(python - <<PY
import sys; sys.path.insert(0, 'scripts')
from launches import load
per, meta = load('gpurun_out/launches_${CFG}_${TAG}.csv')
g = sorted(per)
t = max(g, key=lambda i: per[i]['gpu__time_duration.sum'])
print(g.index(t))
PY
)
echo "top gett_kernel index $SKIP" > gpurun_out/prof_top_${CFG}_${TAG}.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gett_kernel -s $SKIP -c 1 \
  -o gpurun_out/prof_${CFG}_${TAG} -f python bench.py --config $CFG --steps 1 --warmup 1 --slices-per-step $SPS \
  --no-e2e --no-cpu-baseline >> gpurun_out/prof_top_${CFG}_${TAG}.txt 2>&1
