#!/bin/bash
# state check: build, GPU suite, default bench (C3 + cpu_baseline), reference arm, C4/C5 lines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.log; echo "rc=$?" >> gpurun_out/bench_default.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log; echo "rc=$?" >> gpurun_out/bench_c4.log
nproc > gpurun_out/nproc.txt; grep -m1 'model name' /proc/cpuinfo >> gpurun_out/nproc.txt
