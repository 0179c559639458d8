mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -k "fsim or k3 or tensor_cores or c2" -rA > gpurun_out/pytest_gpu_v11.log 2>&1
CFG=C5 SPS=1 TAG=v11 timeout 1500 bash scripts/gpu_prof_top.sh
