#!/bin/bash
# ncu evidence for the current state: launch lists (one bench step) + one --set full capture of the
# top launch per kernel class: K3 (C3), K2s (C3), K3g (C5), K4 (C4); sanitizer runs; smoke(); the
# reference arm line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo "rc=$?" >> gpurun_out/bench_ref.log
timeout 600 python scripts/bench_permute.py > gpurun_out/permute.json 2> gpurun_out/permute.log
CFG=C3 SPS=2 TAG=k3 KREGEX='gett_tc_kernel' timeout 1500 bash scripts/gpu_prof.sh
CFG=C3 SPS=2 TAG=k2s KREGEX='stream_gett' timeout 900 bash scripts/gpu_prof.sh
CFG=C5 SPS=1 TAG=k3g KREGEX='gett_tcg' timeout 1500 bash scripts/gpu_prof.sh
CFG=C4 SPS=1 TAG=k4 KREGEX='gett_dmma' timeout 1200 bash scripts/gpu_prof.sh
for t in C3_k3 C5_k3g; do
  ncu -i gpurun_out/prof_$t.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${t}_source.csv 2>&1
done
bash scripts/gpu_sanitize.sh
ls -la gpurun_out
