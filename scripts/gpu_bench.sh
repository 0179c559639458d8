#!/bin/bash
# bench lines (+ optional launch list) only
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TAG=${TAG:-x}
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_$TAG.json 2> gpurun_out/bench_c2_$TAG.log
timeout 900 python bench.py --config C3 --steps ${STEPS:-3} --warmup 3 --slices-per-step ${SPS:-8} ${C3ARGS} > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.log
if [ -n "$LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_C3_$TAG.csv python bench.py --config C3 --steps 1 --warmup 1 \
  --slices-per-step 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_C3_$TAG.log 2>&1
fi
