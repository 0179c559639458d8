#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 3 python scripts/k3_debug.py > gpurun_out/k3_debug.log 2>&1; echo rc=$? >> gpurun_out/k3_debug.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
TAG=${TAG:-k3v2} LAUNCHES=1 bash scripts/gpu_bench.sh
