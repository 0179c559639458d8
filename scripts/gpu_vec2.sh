#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c2_full or k3 or consumer" > gpurun_out/pytest_vec2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_vec2.log
JETB200_CONSUMER_LAYOUT=1 JETB200_K3_VEC=1 timeout 900 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_vec2.json 2> gpurun_out/bench_c3_vec2.log
timeout 900 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_base2.json 2> gpurun_out/bench_c3_base2.log
