#!/bin/bash
# One GPU session: build, tests, smoke, short benches, launch list.  Logs go to gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log; echo "rc=$?" >> gpurun_out/bench_c2.log
timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --slices-per-step ${SPS:-8} > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.log; echo "rc=$?" >> gpurun_out/bench_c3.log
if [ -n "$LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_C3.csv python bench.py --config C3 --steps 1 --warmup 1 \
  --slices-per-step 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_C3.log 2>&1
fi
