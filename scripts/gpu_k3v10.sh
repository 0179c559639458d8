mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
T=${TAG:-v10}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$T.log 2>&1
timeout 600 python scripts/node_bench.py C3 8 > gpurun_out/node_C3_$T.log 2>&1
timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --slices-per-step 8 > gpurun_out/bench_c3_$T.json 2> gpurun_out/bench_c3_$T.log
for bm in 0 3 4 5; do
JETB200_TCG_BM=$bm timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_${T}_bm$bm.json 2> gpurun_out/bench_c5_${T}_bm$bm.log
done
