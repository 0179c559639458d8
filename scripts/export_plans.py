"""Run the host planner exactly as bench.py's make_plan did in round 1 and write the chosen
plans to plans/<cfg>.json (jt_plan_export format + the planner record).  The committed plan
files are the problem inputs (the code "takes in a special file ... which stores the
contraction path"): bench.py, the parity goldens and the reference arm all read them.

  python scripts/export_plans.py C3 [C2 C4 C5 ...]
  python scripts/export_plans.py C5 --seeds 1-40 --trials 1024 --weights 0,5,15   (wider search)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS  # noqa: E402
from circuits import workload  # noqa: E402
from paper_2107_09793_b200 import jet  # noqa: E402
from paper_2107_09793_b200.runtime import plan_best  # noqa: E402


def export(name, seed=1, trials=4096, width_cap=31, seeds=None, weights=None):
    cfg = CONFIGS[name]
    circ, bits = workload(cfg["circ"], seed)
    net = jet.Network.from_circuit(circ, bits)
    k = cfg["k"]
    t0 = time.time()
    seeds = tuple(seeds) if seeds else tuple(range(seed, seed + cfg.get("seeds", 8)))
    kw = {"weights": tuple(weights)} if weights else {}
    plan, info = plan_best(net, k if k is not None else -1, dtype=cfg["dtype"], seeds=seeds, trials=trials,
                           width_cap=cfg.get("cap", width_cap) if k is None else 0, **kw)
    dt = time.time() - t0
    c = plan.cost()
    rec = {"config": name, "workload": cfg["workload"], "circuit": cfg["circ"], "circuit_seed": seed,
           "bitstring_seed": seed, "n_wires": circ.n_wires, "d": circ.d, "dtype": cfg["dtype"],
           "ssa_path": [list(s) for s in plan.ssa_path], "sliced_labels": plan.sliced_labels,
           "planner": dict(info, trials=trials, seeds=list(seeds), weights=list(weights) if weights else None,
                           width_cap=cfg.get("cap", width_cap) if k is None else 0, plan_seconds=round(dt, 1)),
           "cost": {kk: (float(v) if isinstance(v, float) else int(v)) for kk, v in c.items()}}
    out = os.path.join(ROOT, "plans", f"{name}.json")
    with open(out, "w") as f:
        json.dump(rec, f)
    print(name, json.dumps(rec["planner"]), json.dumps(rec["cost"]), flush=True)


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--seeds", default=None, help="a-b (inclusive)")
    ap.add_argument("--trials", type=int, default=4096)
    ap.add_argument("--weights", default=None, help="comma-separated roofline bytes weights")
    a = ap.parse_args()
    sd = None
    if a.seeds:
        lo, hi = (int(x) for x in a.seeds.split("-"))
        sd = range(lo, hi + 1)
    wt = [float(x) for x in a.weights.split(",")] if a.weights else None
    for n in a.configs:
        export(n, trials=a.trials, seeds=sd, weights=wt)
