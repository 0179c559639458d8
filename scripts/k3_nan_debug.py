import os, sys, numpy as np, torch
sys.path.insert(0, '.')
from circuits import workload
from paper_2107_09793_b200 import jet
c, x = workload("C2")
net = jet.Network.from_circuit(c, x)
plan = jet.Plan.greedy(net, seed=1, trials=256, n_sliced=6, bytes_weight=5.0)
res = {}
for tc in ("0", "1"):
    os.environ["JETB200_TC"] = tc
    d = plan.describe_exec("c64")
    stream = torch.cuda.Stream()
    ex = jet.Exec(plan, "c64", stream=stream)
    acc = torch.zeros(2, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    v = ex.contract(0, 1, acc, slice_values=True)
    torch.cuda.synchronize()
    ws = ex.ws
    vals = {}
    for n in d["nodes"]:
        if n["maxpos"] < 0 or True:
            off = n["out_off"]; cnt = n["n_out"]
            t = ws[off: off + cnt * 8].view(torch.complex64).cpu().numpy()
            vals[n["v"]] = (n, t)
    res[tc] = (v, vals)
    print("tc", tc, "slice0", v)
v0, vals0 = res["0"]; v1, vals1 = res["1"]
for n in plan.describe_exec("c64")["nodes"]:
    a = vals0[n["v"]][1]; b = vals1[n["v"]][1]; nn = vals1[n["v"]][0]
    bad = np.isnan(b).any() or np.abs(b - a).max() > 1e-3 * (np.abs(a).max() + 1e-30)
    if bad:
        print("FIRST BAD node", nn, "nan", np.isnan(b).sum(), "of", b.size, "maxdiff", np.nanmax(np.abs(b - a)), "max", np.abs(a).max())
        break
