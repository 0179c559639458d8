#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_vec.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_vec.log
timeout 900 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_vec.json 2> gpurun_out/bench_c3_vec.log
JETB200_K3_VEC=0 timeout 900 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_novec.json 2> gpurun_out/bench_c3_novec.log
