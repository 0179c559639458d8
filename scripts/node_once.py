"""One node of a benched plan (plans/<cfg>.json) launched once inside a cudaProfilerStart/Stop
range, after a warm contraction of slice 0 (inputs in place): for
  ncu --profile-from-start off -c 1 ... python scripts/node_once.py C3 928"""
import sys
sys.path.insert(0, '.')
import torch
from circuits import workload
from paper_2107_09793_b200 import jet
import bench

cfg, idx = sys.argv[1], int(sys.argv[2])
rec = bench.load_plan_file(cfg)
circ, bits = workload(rec["circuit"], rec["circuit_seed"])
net = jet.Network.from_circuit(circ, bits)
plan = jet.Plan.create(net, [tuple(x) for x in rec["ssa_path"]], rec["sliced_labels"])
ex = jet.Exec(plan, rec["dtype"], stream=torch.cuda.Stream())
acc = torch.zeros(2, dtype=torch.float64, device="cuda")
ex.contract(0, 1, acc)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
ex.time_node(idx, reps=1)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("node", idx, "done")
