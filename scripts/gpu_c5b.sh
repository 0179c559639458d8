#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "k3g or c2 or c3" > gpurun_out/pytest_c5b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c5b.log
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5_tmt7.json 2> gpurun_out/bench_C5_tmt7.log
timeout 900 python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_tmt7.json 2> gpurun_out/bench_c3_tmt7.log
