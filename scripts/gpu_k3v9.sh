mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_v9.log 2>&1
timeout 600 python scripts/node_bench.py C3 8 > gpurun_out/node_C3_v9.log 2>&1
timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --slices-per-step 8 > gpurun_out/bench_c3_v9.json 2> gpurun_out/bench_c3_v9.log
