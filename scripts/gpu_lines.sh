#!/bin/bash
# C4 and C5 bench lines as BASELINE.json configures them (per-GPU blocks of the fixed subsets),
# plus the tests touched since the last full suite run
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -q -rA -k "k3g or c5 or C5 or k2s or k4" > gpurun_out/pytest_lines.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lines.log
timeout 1500 python bench.py --config C4 --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log; echo "rc=$?" >> gpurun_out/bench_c4.log
timeout 2700 python bench.py --config C5 --steps 1 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.log; echo "rc=$?" >> gpurun_out/bench_c5.log
