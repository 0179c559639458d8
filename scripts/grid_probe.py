import sys; sys.path.insert(0,'.')
import torch
from circuits import workload
from paper_2107_09793_b200 import jet
import bench
rec = bench.load_plan_file("C3")
circ, bits = workload(rec["circuit"], rec["circuit_seed"])
net = jet.Network.from_circuit(circ, bits)
plan = jet.Plan.create(net, [tuple(x) for x in rec["ssa_path"]], rec["sliced_labels"])
ex = jet.Exec(plan, "c64")
print("ok")
