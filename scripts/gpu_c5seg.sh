#!/bin/bash
# C5 long-K precision: K3g accumulation segment length vs error (against K2 and P7) and time
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for seg in 20 8 6 4; do
  rm -f gpurun_out/parity_errors.json
  JETB200_TCG_SEG=$seg timeout 900 python -m pytest tests/test_gpu_benched.py -q -x -k "c5_benched or p7_closed_form_slices" > gpurun_out/c5seg_$seg.log 2>&1
  cp gpurun_out/parity_errors.json gpurun_out/c5seg_errors_$seg.json 2>/dev/null
  JETB200_TCG_SEG=$seg timeout 900 python bench.py --config C5 --steps 1 --warmup 1 --slices-per-step 8 --no-cpu-baseline --no-e2e > gpurun_out/c5seg_bench_$seg.json 2>/dev/null
done
timeout 900 python -m pytest tests/test_gpu_benched.py tests/test_gpu_parity.py -q -k "p7_full_amplitude or consumer_layout or variants" > gpurun_out/pytest_fix.log 2>&1
tail -2 gpurun_out/pytest_fix.log
