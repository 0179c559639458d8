#!/bin/bash
# full ncu capture of specific K2 launches (index among gett launches) of the bench workload
mkdir -p gpurun_out
CFG=${CFG:-C3}; SPS=${SPS:-2}; TAG=${TAG:-v0}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for S in $SKIPS; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gett -s $S -c 1 \
  -o gpurun_out/prof_${CFG}_${TAG}_$S -f python bench.py --config $CFG --steps 1 --warmup 1 --slices-per-step $SPS \
  --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_${CFG}_${TAG}_$S.log 2>&1
done
