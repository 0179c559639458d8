#!/bin/bash
# TMA bring-up (K3, K3g, K2s): TMA probe, parity of the TMA paths, per-node timing TMA vs
# cp.async gathers, bench variants
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_benched.py tests/test_gpu_parity.py -q -rA -k "benched or k2s or k3g or c2_full or c3 or reuse or graph or golden or partition" > gpurun_out/pytest_tma.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tma.log
timeout 600 python scripts/node_bench.py C3 14 > gpurun_out/nodes_C3_tma.txt 2>&1
JETB200_K3_TMA=0 timeout 600 python scripts/node_bench.py C3 14 > gpurun_out/nodes_C3_gather.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_tma.json 2> gpurun_out/bench_c3_tma.log
JETB200_K3_RS=8 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_tma_rs8.json 2> gpurun_out/bench_c3_tma_rs8.log
JETB200_K2S=0 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_tma_nok2s.json 2> gpurun_out/bench_c3_tma_nok2s.log
timeout 600 python scripts/node_bench.py C5 6 > gpurun_out/nodes_C5_tma.txt 2>&1
JETB200_K3_TMA=0 timeout 600 python scripts/node_bench.py C5 6 > gpurun_out/nodes_C5_gather.txt 2>&1
timeout 900 python bench.py --config C5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_tma.json 2> gpurun_out/bench_c5_tma.log
