#!/bin/bash
# ncu full capture of the top C3 contraction launch + C4 / C5 bench lines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CFG=C3 SPS=2 TAG=v11 timeout 1500 bash scripts/gpu_prof_top.sh
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log; echo "rc=$?" >> gpurun_out/bench_c4.log
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.log; echo "rc=$?" >> gpurun_out/bench_c5.log
