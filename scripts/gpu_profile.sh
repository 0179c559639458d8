#!/bin/bash
# ncu evidence for the bench workload: launch list (all kernels, device time) + full
# capture of a few K2 launches.  Never a bench value: numbers under ncu are profiles only.
mkdir -p gpurun_out
CFG=${CFG:-C3}
SPS=${SPS:-2}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${CFG}.csv python bench.py --config $CFG --steps 1 --warmup 1 \
  --slices-per-step $SPS --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_${CFG}.log 2>&1
echo "launch rc=$?" >> gpurun_out/ncu_launch_${CFG}.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gett -s ${SKIP:-300} -c ${COUNT:-4} \
  -o gpurun_out/prof_${CFG} -f python bench.py --config $CFG --steps 1 --warmup 1 --slices-per-step $SPS \
  --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_${CFG}.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full_${CFG}.log
