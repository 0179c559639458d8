mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA -k "k4 or C4 or gbs" > gpurun_out/pytest_k4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k4.log
bash scripts/gpu_nodevar.sh C4 4 g3 m4:JETB200_K4_3M=0 g3tn4:JETB200_DMMA_TN=4
CFG=C5 SPS=1 TAG=k3g KREGEX=gett_tcg bash scripts/gpu_prof.sh
ncu -i gpurun_out/prof_C5_k3g.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_C5_k3g_source.csv 2>&1
ls -la gpurun_out
