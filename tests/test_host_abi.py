"""Host-side tests of libjetb200 (no GPU): the library loads, exports every symbol the
header declares, builds networks with the documented id conventions, validates plans,
and its cost counters equal the oracle's (P12)."""

import json
import os
import re

import numpy as np
import pytest

from circuits import Circuit, generate_gbs, grid_rqc, random_bitstring, workload
from circuits.gates import CZ, HADAMARD
from oracle import contract, cost, path
from oracle.network import build_network

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def jet():
    import __graft_entry__

    __graft_entry__.build()
    from paper_2107_09793_b200 import jet as j

    return j


def test_header_symbols_exported(jet):
    hdr = open(os.path.join(ROOT, "include", "jetb200.h")).read()
    declared = set(re.findall(r"\b(jt_[a-z_0-9]+)\s*\(", hdr))
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(jet._lib, name), name
    assert set(jet.EXPORTED) == declared


def test_network_ids_match_oracle(jet, tmp_path):
    c, x = workload("C1")
    net = jet.Network.from_circuit(c, x)
    onet = build_network(c, x)
    nt, nl = net.info()
    assert nt == onet.n_tensors and nl == len(onet.dims)
    f = tmp_path / "net.json"
    net.export(str(f))
    exp = json.load(open(f))
    assert [tuple(t) for t in exp["tensors"]] == [tuple(l) for l in onet.labels]


def test_plan_validation_errors(jet):
    c = Circuit(2, 2)
    c.add((0,), HADAMARD)
    c.add((1,), HADAMARD)
    c.add((0, 1), CZ)
    net = jet.Network.from_circuit(c, [0, 0])
    good = [(5, 4), (3, 1), (2, 0), (6, 7), (10, 8), (9, 11)]
    jet.Plan.create(net, good, [3])
    with pytest.raises(jet.JetError) as e:
        jet.Plan.create(net, good[:-1], [])
    assert e.value.code == 3
    with pytest.raises(jet.JetError) as e:
        jet.Plan.create(net, [(5, 5)] + good[1:], [])
    assert e.value.code == 3
    with pytest.raises(jet.JetError) as e:
        jet.Plan.create(net, good, [99])
    assert e.value.code == 3
    with pytest.raises(jet.JetError) as e:
        jet.Plan.create(net, good, [3, 3])
    assert e.value.code == 3
    n2 = jet.Network(2, 2)
    with pytest.raises(jet.JetError) as e:
        n2.add_gate((0, 0), np.eye(4))
    assert e.value.code == 2
    with pytest.raises(jet.JetError) as e:
        jet.Plan.greedy(n2)
    assert e.value.code == 3


@pytest.mark.parametrize("name,k", [("C1", 0), ("C1", 3), ("gbs", 2)])
def test_cost_counters_equal_oracle(jet, name, k):
    if name == "gbs":
        c = generate_gbs(2, 2, 1, 0.5, 4, seed=3)
        x = random_bitstring(4, 4, 3)
    else:
        c, x = workload(name)
    net = jet.Network.from_circuit(c, x)
    plan = jet.Plan.greedy(net, seed=2, trials=16, n_sliced=k)
    onet = build_network(c, x)
    p, sl = plan.ssa_path, plan.sliced_labels
    assert len(sl) == k
    contract.validate_path(onet.n_tensors, p)
    ref = cost.cost_report(onet, p, sl)
    got = plan.cost()
    for key in ("n_sl", "flop_sl", "flop_shared", "e_flsl", "e_fltask", "exact_reuse", "prefix"):
        assert got[key] == ref[key], key
    # every sub-range (the library counts them in closed form, the oracle slice by slice)
    n = ref["n_sl"]
    for b in range(n):
        for e in range(b, n + 1):
            assert plan.prefix_flop(b, e) == cost.prefix_flop(onet, p, sl, b, e), (b, e)


def test_greedy_plan_is_deterministic_and_valid(jet, tmp_path):
    c, x = workload("C1")
    net = jet.Network.from_circuit(c, x)
    a = jet.Plan.greedy(net, seed=5, trials=32, n_sliced=2, threads=4)
    b = jet.Plan.greedy(net, seed=5, trials=32, n_sliced=2, threads=1)
    assert a.ssa_path == b.ssa_path and a.sliced_labels == b.sliced_labels
    f = tmp_path / "plan.json"
    a.export(str(f))
    d = json.load(open(f))
    assert [tuple(s) for s in d["ssa_path"]] == a.ssa_path and d["sliced_labels"] == a.sliced_labels
    # the oracle evaluates the exported plan to the state-vector amplitude (P2 via P5)
    onet = build_network(c, x)
    amp = contract.amplitude(onet, d["ssa_path"], d["sliced_labels"])
    amp2 = contract.amplitude(onet, path.greedy_path(onet))
    assert abs(amp - amp2) < 1e-12


def test_planner_width_cap(jet):
    c, x = workload("C2")
    net = jet.Network.from_circuit(c, x)
    plan = jet.Plan.greedy(net, seed=1, trials=16, n_sliced=-1, width_cap=18)
    co = plan.cost()
    assert co["max_width"] <= 18 and co["n_sliced"] > 0


@pytest.mark.parametrize("name", ["C1", "C3", "C4"])
def test_network_export_matches_oracle_network(name, tmp_path):
    """Row a1 pinned at full size: the product's closed network (jt_network_export, labels and
    data) equals the oracle's own build from the same circuit (oracle/network.py),
    tensor by tensor, label order and every complex entry exactly (both copy the generator's gate
    matrices; the product's absorption happens later, in the plan)."""
    import json

    import numpy as np

    from circuits import workload
    from oracle.network import build_network
    from paper_2107_09793_b200 import jet

    circ, bits = workload(name)
    net = jet.Network.from_circuit(circ, bits)
    p = tmp_path / "net.json"
    net.export(str(p))
    d = json.load(open(p))
    onet = build_network(circ, bits)
    assert d["n_wires"] == circ.n_wires and d["d"] == circ.d and d["closed"]
    assert len(d["tensors"]) == onet.n_tensors == len(d["data"])
    for t in range(onet.n_tensors):
        assert tuple(d["tensors"][t]) == tuple(onet.labels[t]), t
        flat = np.asarray(d["data"][t], dtype=np.float64).view(np.complex128)
        assert np.array_equal(flat, np.asarray(onet.tensors[t], dtype=np.complex128).reshape(-1)), t
