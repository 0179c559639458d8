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
# each argument: tag or tag:ENV=VAL,ENV=VAL (e.g. nopdl_gather:JETB200_PDL=0,JETB200_K3_TMA=0)
for v in "$@"; do
  tag=${v%%:*}
  envs="X=1"
  if [[ "$v" == *:* ]]; then envs=$(echo "${v#*:}" | tr ',' ' '); fi
  run "$tag" $envs
done
