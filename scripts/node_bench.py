"""Time the heaviest nodes of a bench plan one by one (kernel tuning on real shapes)."""
import json, os, sys
sys.path.insert(0, '.')
import torch
from circuits import workload
from paper_2107_09793_b200 import jet
from paper_2107_09793_b200.runtime import plan_best

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
k = {"C3": 10, "C2": 6, "C5": -1}[cfg]
circ, bits = workload(cfg)
net = jet.Network.from_circuit(circ, bits)
plan, info = plan_best(net, k, seeds=(1,), trials=1024, width_cap=30 if k < 0 else 0)
d = plan.describe_exec("c64")
order = d["nodes"]
stream = torch.cuda.Stream()
ex = jet.Exec(plan, "c64", stream=stream)
acc = torch.zeros(2, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
ex.contract(0, 1, acc)
torch.cuda.synchronize()
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
cands = sorted(range(len(order)), key=lambda i: -order[i]["bytes"] * (2 ** (order[i]["maxpos"] + 1)))[:int(sys.argv[2]) if len(sys.argv) > 2 else 8]
for i in cands:
    n = order[i]
    r = ex.time_node(i, reps=5)
    gbs = r["bytes"] / (r["ms"] / 1e3) / 1e9
    tfs = r["flop"] / (r["ms"] / 1e3) / 1e12
    print(json.dumps({"idx": i, "kind": r["kind"], "ms": round(r["ms"], 4), "GBps": round(gbs), "frac_hbm": round(gbs / peak, 3),
                      "TFs": round(tfs, 1), "tm": n.get("tc_tm"), "tk": n.get("tc_tk"), "outer": n.get("tc_outer"),
                      "k2": [n["tm"], n["tn"], n["tk"], n["n_outer"], n["n_ok"]]}), flush=True)
