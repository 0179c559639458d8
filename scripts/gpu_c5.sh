#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.log; echo "rc=$?" >> gpurun_out/bench_C5.log
timeout 600 python scripts/node_bench.py C5 8 > gpurun_out/node_C5.txt 2>&1
