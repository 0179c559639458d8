"""Per-item clock64 trace of CTA 0 of the heaviest K3 nodes (JETB200_K3_TRACE): where the
cycles of one item go in each warp role (producer warps 4 / 11, MMA warp, epilogue warp 0)."""
import json, os, sys
sys.path.insert(0, '.')
import numpy as np
import torch
from circuits import workload
from paper_2107_09793_b200 import jet
from paper_2107_09793_b200.runtime import plan_best

circ, bits = workload("C3")
net = jet.Network.from_circuit(circ, bits)
plan, info = plan_best(net, 10, seeds=tuple(range(1, 9)), trials=4096)
order = plan.describe_exec("c64")["nodes"]
cands = [i for i in sorted(range(len(order)), key=lambda i: -order[i]["bytes"] * 2 ** (order[i]["maxpos"] + 1))
         if order[i]["kind"] == 1][:int(sys.argv[1]) if len(sys.argv) > 1 else 3]
os.environ["JETB200_K3_DBG"] = sys.argv[2] if len(sys.argv) > 2 else "0"
stream = torch.cuda.Stream()
ex = jet.Exec(plan, "c64", stream=stream)
acc = torch.zeros(2, dtype=torch.float64, device="cuda")
ex.contract(0, 1, acc)
torch.cuda.synchronize()
names = {0: ["start", "landed", "split", "sttm", "arrive", "xempty", "copied"], 1: ["start", "landed", "split", "sttm", "arrive", "xempty", "copied"],
         2: ["start", "tempty", "xfull", "issued"], 3: ["start", "tfull", "stored", "arrived"]}
for i in cands:
    path = f"/tmp/k3trace_{i}.bin"
    os.environ["JETB200_K3_TRACE"] = path
    r = ex.time_node(i, reps=1)
    os.environ.pop("JETB200_K3_TRACE")
    t = np.fromfile(path, dtype=np.uint64).reshape(4, 64, 8).astype(np.int64)
    n = order[i]
    out = {"idx": i, "tm": n["tc_tm"], "tk": n["tc_tk"], "ms": round(r["ms"], 4),
           "nonzero_per_role": [int(x) for x in (t > 0).sum(axis=(1, 2))]}
    for role in range(4):
        ks = names[role]
        st = t[role, :, :len(ks)]
        if role < 2:  # slot 6 (xempty) sits between slots 4 and 5
            st = t[role][:, [0, 1, 2, 3, 4, 6, 5]]
        ok = st[:, 0] > 0
        st = st[ok]
        if len(st) < 3:
            continue
        per_item = np.median(np.diff(st[:, 0]))
        seg = {f"{ks[k-1]}->{ks[k]}": int(np.median(st[:, k] - st[:, k - 1])) for k in range(1, len(ks))}
        out[f"role{role}"] = {"cycles_per_iter": int(per_item), **seg}
    print(json.dumps(out), flush=True)
