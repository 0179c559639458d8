"""Small GPU workload for compute-sanitizer (memcheck / racecheck / synccheck): one C2 slice on
the default path (K3 TMA + K2), the same slice with K3g forced and with the cp.async K3, a 5x5
grid slice on K2s + K3 (and K3 with four accumulators), one c128 GBS slice on K4 (DMMA), and a
K1 permute; each checked against the oracle.

  compute-sanitizer --tool racecheck python scripts/sanitize_case.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from circuits import generate_gbs, random_bitstring, workload  # noqa: E402
from oracle import contract  # noqa: E402
from oracle.network import build_network  # noqa: E402
from paper_2107_09793_b200 import jet  # noqa: E402


def one(plan, dtype, i, ref, tol, tag):
    ex = jet.Exec(plan, dtype)
    acc = torch.zeros(2, dtype=torch.float64, device="cuda")
    v = ex.contract(i, i + 1, acc, slice_values=True)[0]
    torch.cuda.synchronize()
    err = abs(v - ref) / abs(ref)
    print(f"{tag}: rel err {err:.3e}", flush=True)
    assert err < tol, (tag, err)


def main():
    torch.cuda.set_device(0)
    circ, bits = workload("C2")
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=1, trials=64, n_sliced=6, bytes_weight=5.0)
    ref = contract.slice_values(build_network(circ, bits), plan.ssa_path, plan.sliced_labels, indices=[3])[0]
    kinds = [(n["kind"], n.get("tma", 0)) for n in plan.describe_exec("c64")["nodes"]]
    assert (1, 1) in kinds
    one(plan, "c64", 3, ref, 1e-4, "C2 K3-TMA + K2")
    for envs, tag in (({"JETB200_TCG_FORCE": "1"}, "C2 K3g"),
                      ({"JETB200_TCG_FORCE": "1", "JETB200_TCG_SEG": "0"}, "C2 K3g, one segment per chunk (bulk adds)"),
                      ({"JETB200_K3_TMA": "0"}, "C2 K3 cp.async")):
        os.environ.update(envs)
        p = jet.Plan.create(net, plan.ssa_path, plan.sliced_labels)
        one(p, "c64", 3, ref, 1e-4, tag)
        for k in envs:
            del os.environ[k]
    # K2s (register-resident streaming GETT, with and without 16-B k-pair loads) on a 5x5 grid
    from circuits import grid_rqc
    gc = grid_rqc(5, 5, 10, 1)
    gcb = random_bitstring(25, 2, 1)
    gcn = jet.Network.from_circuit(gc, gcb)
    gcp = jet.Plan.greedy(gcn, seed=1, trials=16, n_sliced=4)
    assert any(n["kind"] == 4 and n["st_vec"] for n in gcp.describe_exec("c64")["nodes"])
    gcref = contract.slice_values(build_network(gc, gcb), gcp.ssa_path, gcp.sliced_labels, indices=[5])[0]
    one(gcp, "c64", 5, gcref, 1e-4, "grid K2s + K3")
    os.environ["JETB200_K3_ACC"] = "4"
    one(jet.Plan.create(gcn, gcp.ssa_path, gcp.sliced_labels), "c64", 5, gcref, 1e-4, "grid K3 4 accumulators")
    del os.environ["JETB200_K3_ACC"]
    g = generate_gbs(2, 4, 1, 0.5, 4, seed=5)
    gb = random_bitstring(g.n_wires, 4, 12)
    gnet = jet.Network.from_circuit(g, gb)
    gp = jet.Plan.greedy(gnet, seed=1, trials=16, n_sliced=2)
    assert any(n["kind"] == 3 for n in gp.describe_exec("c128")["nodes"])
    gref = contract.slice_values(build_network(g, gb), gp.ssa_path, gp.sliced_labels, indices=[1])[0]
    if abs(gref) > 0:
        one(gp, "c128", 1, gref, 1e-10, "GBS K4")
    src = torch.randn(1 << 16, dtype=torch.complex64, device="cuda")
    perm = list(np.random.default_rng(0).permutation(16))
    jet.permute(src, perm)
    torch.cuda.synchronize()
    print("sanitize case done", flush=True)


if __name__ == "__main__":
    main()
