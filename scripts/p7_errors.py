"""P7 closed-form errors of 8 slices (one per rank block of G=8, seeded as in the test) of a
benched plan under the current environment (kernel-path variants), plus the slice magnitude
structure: python scripts/p7_errors.py C5"""
import json, os, sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import torch
from p7_closed import slice_closed_form
from circuits import workload
from circuits.rng import SplitMix64
from circuits.sycamore import random_circuit, sycamore_qubits
from paper_2107_09793_b200 import jet
from paper_2107_09793_b200.runtime import shard_range

cfg = sys.argv[1]
rec = json.load(open(f"plans/{cfg}.json"))
m = {"C2": 10, "C3": 14, "C5": 20}[rec["circuit"]]
circ = random_circuit(sycamore_qubits(53), m, seed=rec["circuit_seed"], theta=0.0, phi=0.0)
_, bits = workload(rec["circuit"], rec["circuit_seed"])
net = jet.Network.from_circuit(circ, bits)
plan = jet.Plan.create(net, [tuple(x) for x in rec["ssa_path"]], rec["sliced_labels"])
ex = jet.Exec(plan, "c64", stream=torch.cuda.Stream())
acc = torch.zeros(2, dtype=torch.float64, device="cuda")
n_sl = plan.cost()["n_sl"]
rng = SplitMix64(77)
out = {}
for g in range(8):
    b, e = shard_range(n_sl, g, 8)
    i = b + int(rng.next_u64() % (e - b))
    want = slice_closed_form(circ, bits, rec["sliced_labels"], i)
    ex.invalidate()
    v = ex.contract(i, i + 1, acc, slice_values=True)[0]
    torch.cuda.synchronize()
    out[i] = abs(v - want) / abs(want) if want != 0 else (0.0 if v == 0 else float("inf"))
env = {k: v for k, v in os.environ.items() if k.startswith("JETB200_")}
print(json.dumps({"cfg": cfg, "env": env, "max_rel": max(out.values()), "per_slice": out}), flush=True)
