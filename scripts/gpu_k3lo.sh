#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TAG=${TAG:-x}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c2 or c3 or k3" > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python scripts/node_bench.py C5 4 > gpurun_out/node_C5_$TAG.txt 2>&1
timeout 900 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.log
