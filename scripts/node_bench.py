"""Time the heaviest nodes of a bench plan one by one (kernel tuning on real shapes)."""
import json, os, sys
sys.path.insert(0, '.')
import torch
from circuits import workload
from paper_2107_09793_b200 import jet
from paper_2107_09793_b200.runtime import plan_best

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
k, dt, cap = {"C3": (10, "c64", 0), "C2": (6, "c64", 0), "C5": (-1, "c64", 30), "C4": (-1, "c128", 28),
              "G88d8": (-1, "c128", 30)}[cfg]
circ, bits = workload(cfg)
net = jet.Network.from_circuit(circ, bits)
plan, info = plan_best(net, k, dtype=dt, seeds=(1,) if dt == "c64" else (1, 2), trials=1024 if dt == "c64" else 4096,
                       width_cap=cap)
d = plan.describe_exec(dt)
order = d["nodes"]
stream = torch.cuda.Stream()
ex = jet.Exec(plan, dt, stream=stream)
acc = torch.zeros(2, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
ex.contract(0, 1, acc)
torch.cuda.synchronize()
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
wkey = "bytes" if dt == "c64" else "flop"
cands = sorted(range(len(order)), key=lambda i: -order[i][wkey] * (circ.d ** (order[i]["maxpos"] + 1)))[:int(sys.argv[2]) if len(sys.argv) > 2 else 8]
for i in cands:
    n = order[i]
    r = ex.time_node(i, reps=5)
    gbs = r["bytes"] / (r["ms"] / 1e3) / 1e9
    tfs = r["flop"] / (r["ms"] / 1e3) / 1e12
    print(json.dumps({"idx": i, "kind": r["kind"], "ms": round(r["ms"], 4), "GBps": round(gbs), "frac_hbm": round(gbs / peak, 3),
                      "TFs": round(tfs, 1), "tm": n.get("tc_tm"), "tk": n.get("tc_tk"), "outer": n.get("tc_outer"),
                      "k2": [n["tm"], n["tn"], n["tk"], n["n_outer"], n["n_ok"], n["splits"], n["RM"], n["RN"]]}), flush=True)
