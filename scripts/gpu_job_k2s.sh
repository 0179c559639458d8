#!/bin/bash
# K2s (register-resident streaming GETT) on the GPU: parity tests, the C3 bench line, C3 node timings
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q -rA -k "k2s or benched_plan_golden or p7 or error_study or k4" > gpurun_out/pytest_k2s.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k2s.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_k2s.json 2> gpurun_out/bench_c3_k2s.log
timeout 600 python scripts/node_bench.py C3 14 > gpurun_out/nodes_C3_k2s.txt 2>&1
