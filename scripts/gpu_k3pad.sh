#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1 or c2 or c3 or k3 or reuse or graph" > gpurun_out/pytest_k3pad.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k3pad.log
timeout 900 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_k3pad.json 2> gpurun_out/bench_c3_k3pad.log
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_k3pad.json 2> gpurun_out/bench_c2_k3pad.log
