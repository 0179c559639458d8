#!/bin/bash
# GPU suite + the default bench line as the driver runs it (N=1)
mkdir -p gpurun_out
bash scripts/gpu_suite.sh
timeout 1500 python bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/bench_c3_round.json 2> gpurun_out/bench_c3_round.log
echo "bench rc=$?" >> gpurun_out/bench_c3_round.log
tail -2 gpurun_out/bench_c3_round.log
