mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1800 python -m pytest tests -m gpu -q -rA -k "C4 or C5 or c5 or k4" > gpurun_out/pytest_c45.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c45.log
timeout 1800 python bench.py --config C4 --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log; echo "rc=$?" >> gpurun_out/bench_c4.log
