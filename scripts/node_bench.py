"""Time the heaviest nodes of a benched plan (plans/<cfg>.json) one by one, back to back
(kernel tuning on real shapes), with the clocks seen during the run.

  python scripts/node_bench.py C3 [n_nodes] [kind]
With `kind` (0 = K2, 1 = K3, ...), the n_nodes nodes of that kind with the most total time over
the amplitude (per-run time x runs), timed one by one."""
import json, os, sys
sys.path.insert(0, '.')
import torch
from circuits import workload
from paper_2107_09793_b200 import jet
import bench

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
rec = bench.load_plan_file(cfg)   # the committed benched plan
dt = rec["dtype"]
circ, bits = workload(rec["circuit"], rec["circuit_seed"])
net = jet.Network.from_circuit(circ, bits)
plan = jet.Plan.create(net, [tuple(x) for x in rec["ssa_path"]], rec["sliced_labels"])
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
nn = int(sys.argv[2]) if len(sys.argv) > 2 else 8
if len(sys.argv) > 3:   # every node of one kind, ranked by measured per-run time x runs
    kind = int(sys.argv[3])
    ks = [i for i in range(len(order)) if order[i]["kind"] == kind]
    tr = {i: ex.time_node(i, reps=3)["ms"] * circ.d ** (order[i]["maxpos"] + 1) for i in ks}
    print(json.dumps({"kind": kind, "nodes": len(ks), "total_ms_per_amplitude": round(sum(tr.values()), 2)}), flush=True)
    cands = sorted(ks, key=lambda i: -tr[i])[:nn]
else:
    cands = sorted(range(len(order)), key=lambda i: -order[i][wkey] * (circ.d ** (order[i]["maxpos"] + 1)))[:nn]
clk = bench.ClockSampler(0)
clk.start()
for i in cands:
    n = order[i]
    r = ex.time_node(i, reps=5)
    gbs = r["bytes"] / (r["ms"] / 1e3) / 1e9
    tfs = r["flop"] / (r["ms"] / 1e3) / 1e12
    print(json.dumps({"idx": i, "kind": r["kind"], "ms": round(r["ms"], 4), "runs": circ.d ** (n["maxpos"] + 1), "GBps": round(gbs), "frac_hbm": round(gbs / peak, 3),
                      "TFs": round(tfs, 1), "tm": n.get("tc_tm"), "tk": n.get("tc_tk"), "outer": n.get("tc_outer"),
                      "k2": [n["tm"], n["tn"], n["tk"], n["n_outer"], n["n_ok"], n["splits"], n["RM"], n["RN"]]}), flush=True)
print(json.dumps({"clocks": clk.stop()}), flush=True)
