#!/bin/bash
# K4 (c128 DMMA): GPU parity for the c128 paths, then C4 / G88 bench lines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "k4 or gbs or c1_parity or errors" > gpurun_out/pytest_k4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k4.log
for C in C4 G88d4 G88d8; do
timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${C}_k4.json 2> gpurun_out/bench_${C}_k4.log; echo "rc=$?" >> gpurun_out/bench_${C}_k4.log
done
