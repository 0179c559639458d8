#!/bin/bash
# C3 bench under env variants (kernel path / launch-mode A/B), one short bench line each
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() {  # tag, env...
  local tag=$1; shift
  env "$@" timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e ${BENCH_ARGS} \
    > gpurun_out/var_${tag}.json 2> gpurun_out/var_${tag}.log
  python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/var_{t}.json"))
except Exception as e:
    print(t, "ERR", e); sys.exit()
r = d["roofline"]
ks = {k: (v["launches"], round(v["ms"], 1), v["GBps"] and round(v["GBps"])) for k, v in r["kernels"].items() if v["launches"]}
print(t, "ms/step %.1f" % d["ms_per_step"], "frac %.3f" % r["frac"], "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"], ks)
PY
}
for v in "$@"; do
  case $v in
    default) run default X=1 ;;
    nopdl) run nopdl JETB200_PDL=0 ;;
    nographs) run nographs JETB200_GRAPHS=0 ;;
    gather) run gather JETB200_K3_TMA=0 ;;
    rs8) run rs8 JETB200_K3_RS=8 ;;
    rs4) run rs4 JETB200_K3_RS=4 ;;
    mincopy2k) run mincopy2k JETB200_TMA_MINCOPY=2048 ;;
    mincopy8k) run mincopy8k JETB200_TMA_MINCOPY=8192 ;;
    k2s) run k2s JETB200_K2S=1 ;;
  esac
done
