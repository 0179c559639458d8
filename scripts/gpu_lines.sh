#!/bin/bash
# The non-default bench lines as BASELINE.json configures them: C2 (whole m=10 amplitude per
# step), C4 and C5 (per-GPU blocks of the fixed slice subsets)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python bench.py --config C2 --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log; echo "rc=$?" >> gpurun_out/bench_c2.log
timeout 1800 python bench.py --config C4 --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log; echo "rc=$?" >> gpurun_out/bench_c4.log
timeout 2700 python bench.py --config C5 --steps 1 --warmup 3 --cpu-max-slice-s 120 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.log; echo "rc=$?" >> gpurun_out/bench_c5.log
