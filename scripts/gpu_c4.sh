#!/bin/bash
# C4 (GBS, complex128, K4): parity tests, K4 node ranking, the C4 bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -q -rA -k "C4 or k4 or gbs" > gpurun_out/pytest_c4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c4.log
timeout 900 python scripts/node_bench.py C4 8 3 > gpurun_out/nodes_C4_k4.txt 2>&1
timeout 1800 python bench.py --config C4 --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log; echo "rc=$?" >> gpurun_out/bench_c4.log
