import sys, numpy as np, torch
sys.path.insert(0, '.')
from circuits import workload
from paper_2107_09793_b200 import jet
c, x = workload("C2")
net = jet.Network.from_circuit(c, x)
plan = jet.Plan.greedy(net, seed=1, trials=256, n_sliced=6, bytes_weight=5.0)
d = plan.describe_exec("c64")
for n in d['nodes']:
    if n['kind'] == 1:
        print({k: n[k] for k in ('v', 'tc_tm', 'tc_tk', 'tc_outer', 'smem', 'n_out')})
        break
ex = jet.Exec(plan, "c64")
acc = torch.zeros(2, dtype=torch.float64, device="cuda")
v = ex.contract(0, 2, acc, slice_values=True)
print(v)
