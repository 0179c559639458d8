#!/bin/bash
# K3 TMA bring-up: the TMA probe, parity of the K3 paths, per-node timing TMA vs cp.async, bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe scripts/tma_probe.cu > gpurun_out/tma_probe_build.log 2>&1
timeout 300 /tmp/tma_probe > gpurun_out/tma_probe.txt 2>&1; echo "rc=$?" >> gpurun_out/tma_probe.txt
timeout 1200 python -m pytest tests/test_gpu_benched.py tests/test_gpu_parity.py -q -x -k "c2 or c3 or k3 or C2 or C3" > gpurun_out/pytest_k3tma.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k3tma.log
timeout 600 python scripts/node_bench.py C3 12 > gpurun_out/nodes_C3_tma.txt 2>&1
JETB200_K3_RS=8 timeout 600 python scripts/node_bench.py C3 12 > gpurun_out/nodes_C3_tma_rs8.txt 2>&1
JETB200_K3_TMA=0 timeout 600 python scripts/node_bench.py C3 12 > gpurun_out/nodes_C3_gather.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c3_tma.json 2> gpurun_out/bench_c3_tma.log
JETB200_K3_MINTM=2 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c3_tma_mintm2.json 2> gpurun_out/bench_c3_tma_mintm2.log
JETB200_K3_RS=8 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c3_tma_rs8.json 2> gpurun_out/bench_c3_tma_rs8.log
