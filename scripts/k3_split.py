"""Time the heaviest K3 nodes of a bench plan with the kernel's debug modes (JETB200_K3_DBG, a
bit mask: 1 no output stores, 2 no input loads, 4 no split/STTM, 8 no MMAs, 16 no LDTM) --
which stage bounds K3.  usage: k3_split.py C3 <n nodes> <modes, e.g. 0,3,7,11,19,31>"""
import json, os, re, sys
sys.path.insert(0, '.')
import torch
from circuits import workload
from paper_2107_09793_b200 import jet
from paper_2107_09793_b200.runtime import plan_best

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
k = {"C3": 10, "C2": 6}[cfg]
circ, bits = workload(cfg)
net = jet.Network.from_circuit(circ, bits)
plan, info = plan_best(net, k, seeds=tuple(range(1, 9)), trials=4096)
order = plan.describe_exec("c64")["nodes"]
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
cands = [i for i in sorted(range(len(order)), key=lambda i: -order[i]["bytes"] * 2 ** (order[i]["maxpos"] + 1))
         if order[i]["kind"] == 1][:int(sys.argv[2]) if len(sys.argv) > 2 else 6]
res = {}
MODES = sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "1", "2", "3"]
for dbg in MODES:
    # a mode is "<dbg bits>" or "<dbg bits>L<lag>" (JETB200_K3_LAG: gather distance = stages - lag)
    # "<dbg bits>[L<lag>][Y<0|1>]" (JETB200_K3_LAG / JETB200_K3_YCAT)
    import re
    m = re.fullmatch(r"(\d+)(?:L(\d+))?(?:Y(\d+))?", dbg)
    bits, lag, ycat = m.group(1), m.group(2), m.group(3)
    os.environ["JETB200_K3_DBG"] = bits
    for key, val in (("JETB200_K3_LAG", lag), ("JETB200_K3_YCAT", ycat)):
        if val:
            os.environ[key] = val
        else:
            os.environ.pop(key, None)
    stream = torch.cuda.Stream()
    ex = jet.Exec(plan, "c64", stream=stream)
    acc = torch.zeros(2, dtype=torch.float64, device="cuda")
    ex.contract(0, 1, acc)
    torch.cuda.synchronize()
    for i in cands:
        r = ex.time_node(i, reps=10)
        res.setdefault(i, {})[dbg] = r["ms"]
        res[i]["bytes"] = r["bytes"]
    del ex
    torch.cuda.synchronize()
for i in cands:
    n = order[i]
    print(json.dumps({"idx": i, "tm": n["tc_tm"], "tk": n["tc_tk"], "outer": n["tc_outer"], "bytes": n["bytes"],
                      "ms": {d: round(res[i][d], 4) for d in MODES},
                      "frac_hbm": {d: round(res[i]["bytes"] / (res[i][d] / 1e3) / 1e9 / peak, 3) for d in MODES
                                   if re.match(r"0(?!\d)", d)}}), flush=True)
