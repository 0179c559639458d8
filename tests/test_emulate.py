"""CPU check of the plan compiler and the prefix-cache scheduler: the compiled K2 launch
descriptors (bit tiles, strides, split-K, workspace offsets) executed on the host with the
kernels' index arithmetic (jt_debug_emulate_host, test-only) must reproduce the oracle's
s_sigma.  The GPU parity tests then only have to cover the device code itself."""

import numpy as np
import pytest

from circuits import generate_gbs, random_bitstring, workload
from oracle import contract
from oracle.network import build_network


@pytest.fixture(scope="module")
def jet():
    import __graft_entry__

    __graft_entry__.build()
    from paper_2107_09793_b200 import jet as j

    return j


@pytest.mark.parametrize("k", [0, 1, 3, 5])
def test_emulated_descriptors_match_oracle_c1(jet, k):
    circ, _ = workload("C1")
    for seed in range(3):
        bits = random_bitstring(9, 2, 40 + seed)
        net = jet.Network.from_circuit(circ, bits)
        plan = jet.Plan.greedy(net, seed=seed, trials=8, n_sliced=k, bytes_weight=10.0 * (seed % 2))
        ref = np.array(contract.slice_values(build_network(circ, bits), plan.ssa_path, plan.sliced_labels))
        n = len(ref)
        v128 = jet.debug_emulate_host(plan, 0, n, "c128")
        assert np.max(np.abs(v128 - ref)) <= 1e-12 * np.max(np.abs(ref))
        v64 = jet.debug_emulate_host(plan, 0, n, "c64")
        assert np.max(np.abs(v64 - ref)) <= 1e-5 * np.max(np.abs(ref))
        # reuse on/off and split ranges give bitwise-identical values (P10 on the host)
        off = jet.debug_emulate_host(plan, 0, n, "c64", reuse=False)
        assert np.array_equal(v64, off)


@pytest.mark.parametrize("open_wires,k", [([4], 2), ([7, 2], 0), ([8, 0, 3], 3), (list(range(9)), 1)])
def test_emulated_batch_matches_oracle_c1(jet, open_wires, k):
    """f1 batch of amplitudes: every run r = sigma * n_batch + y of a batch plan reproduces the
    oracle's s_sigma of the y-th batch bitstring; reuse on/off bitwise identical."""
    circ, _ = workload("C1")
    bits = random_bitstring(9, 2, 77)
    net = jet.Network.from_circuit(circ, bits, open_wires=open_wires)
    plan = jet.Plan.greedy(net, seed=3, trials=8, n_sliced=k)
    c = plan.cost()
    nb = 2 ** len(open_wires)
    assert c["n_batch"] == nb and c["n_sl"] == 2 ** k and len(plan.sliced_labels) == k
    n = c["n_sl"] * nb
    ref = np.array(contract.batch_run_values(circ, bits, open_wires, plan.ssa_path, plan.sliced_labels, range(n)))
    v = jet.debug_emulate_host(plan, 0, n, "c128")
    assert np.max(np.abs(v - ref)) <= 1e-12 * np.max(np.abs(ref))
    v64 = jet.debug_emulate_host(plan, 0, n, "c64")
    assert np.max(np.abs(v64 - ref)) <= 1e-5 * np.max(np.abs(ref))
    assert np.array_equal(v64, jet.debug_emulate_host(plan, 0, n, "c64", reuse=False))
    # the prefix cache recomputes only what depends on the changed digits: executed FLOP over
    # the batch is below N_sl * n_batch independent contractions
    assert plan.prefix_flop(0, n) < c["e_flsl"]


def test_batch_validation(jet):
    circ, bits = workload("C1")
    for bad in ([9], [-1], [3, 3]):
        net = jet.Network(9, 2)
        for g in circ.gates:
            net.add_gate(g.wires, g.u)
        with pytest.raises(jet.JetError) as e:
            net.close_batch(bits, bad)
        assert e.value.code == 2


def test_emulated_descriptors_match_oracle_gbs(jet):
    circ = generate_gbs(2, 2, 1, 0.5, 4, seed=2)
    for seed in range(3):
        bits = random_bitstring(4, 4, seed)
        net = jet.Network.from_circuit(circ, bits)
        plan = jet.Plan.greedy(net, seed=seed, trials=8, n_sliced=seed)
        ref = np.array(contract.slice_values(build_network(circ, bits), plan.ssa_path, plan.sliced_labels))
        v = jet.debug_emulate_host(plan, 0, len(ref), "c128")
        assert np.max(np.abs(v - ref)) <= 1e-12 * max(np.max(np.abs(ref)), 1e-300)


def test_describe_exec_layout(jet):
    circ, bits = workload("C2")
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=1, trials=32, n_sliced=6)
    d = plan.describe_exec("c64")
    assert d["total_bytes"] == plan.workspace_bytes("c64")
    for n in d["nodes"]:
        assert n["block"] % 32 == 0 and n["block"] <= {1: 448, 2: 448, 4: 288}.get(n["kind"], 256)
        if n["kind"] in (1, 2):   # K3 / K3g: 128-row MMA tiles
            assert n["n_out"] == 2 ** (7 + n["tc_tm"] + n["tc_outer"])
            assert 3 <= n["tc_tm"] <= 7 and 2 <= n["tc_tk"] and n["smem"] <= 220 * 1024
        else:
            assert n["tm"] + n["tk"] <= 12 and n["tk"] + n["tn"] <= 12 and n["tm"] + n["tn"] <= 12
            assert n["n_out"] == 2 ** (n["tm"] + n["tn"] + n["n_outer"])


def test_emulated_k3_matches_oracle_c2_slices(jet, monkeypatch):
    monkeypatch.setenv("JETB200_TMA_MINCOPY", "16")   # every K3 item on the TMA engine: emulate its landing
    circ, bits = workload("C2")
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=1, trials=64, n_sliced=6, bytes_weight=5.0)
    nodes = plan.describe_exec("c64")["nodes"]
    assert sum(n["kind"] for n in nodes) > 0
    assert any(n["kind"] == 1 and n["tma"] for n in nodes)
    ref = np.array(contract.slice_values(build_network(circ, bits), plan.ssa_path, plan.sliced_labels, indices=[5]))
    v = jet.debug_emulate_host(plan, 5, 6, "c64")
    assert np.max(np.abs(v - ref) / np.abs(ref)) < 1e-4


def test_emulated_k3g_matches_oracle_c2_slice(jet, monkeypatch):
    """K3g (both operands streamed) descriptors: force the K3-eligible C2 nodes onto K3g."""
    monkeypatch.setenv("JETB200_TCG_FORCE", "1")
    monkeypatch.setenv("JETB200_TMA_MINCOPY", "16")
    circ, bits = workload("C2")
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=1, trials=64, n_sliced=6, bytes_weight=5.0)
    kinds = [n["kind"] for n in plan.describe_exec("c64")["nodes"]]
    assert kinds.count(2) > 0
    ref = np.array(contract.slice_values(build_network(circ, bits), plan.ssa_path, plan.sliced_labels, indices=[9]))
    v = jet.debug_emulate_host(plan, 9, 10, "c64")
    assert np.max(np.abs(v - ref) / np.abs(ref)) < 1e-4


def test_emulated_k1_fed_k3g_matches_oracle_c2_slice(jet, monkeypatch):
    """K3g fed by K1 bit-gathers (JETB200_TCG_PERM=force: every K3g operand whose chunk is not
    one TMA box is first copied into the K3g layout): the emulated gathers, the single-box TMA
    landings and the contraction against the oracle on a C2 slice."""
    monkeypatch.setenv("JETB200_TCG_FORCE", "1")
    monkeypatch.setenv("JETB200_TCG_PERM", "force")
    circ, bits = workload("C2")
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=1, trials=64, n_sliced=6, bytes_weight=5.0)
    nodes = [n for n in plan.describe_exec("c64")["nodes"] if n["kind"] == 2]
    assert any(n["permA"] for n in nodes) and any(n["permB"] for n in nodes)
    assert all(n["tma"] for n in nodes if n["permA"] and n["permB"])
    ref = np.array(contract.slice_values(build_network(circ, bits), plan.ssa_path, plan.sliced_labels, indices=[9]))
    v = jet.debug_emulate_host(plan, 9, 10, "c64")
    assert np.max(np.abs(v - ref) / np.abs(ref)) < 1e-4


@pytest.mark.parametrize("dim,width,d", [(2, 3, 4), (2, 2, 8), (3, 2, 4)])
def test_emulated_k4_descriptors_match_oracle_gbs(jet, dim, width, d):
    """K4 (c128 DMMA) shares K2's descriptor format; the emulated descriptors of plans that
    route nodes to K4 must reproduce the oracle's s_sigma (d = 8: 3-bit qudit labels, f4)."""
    circ = generate_gbs(dim, width, 1, 0.5, d, seed=3)
    M = circ.n_wires
    n_k4 = 0
    for seed in range(2):
        bits = random_bitstring(M, d, seed + 7)
        net = jet.Network.from_circuit(circ, bits)
        plan = jet.Plan.greedy(net, seed=seed, trials=8, n_sliced=seed)
        nodes = plan.describe_exec("c128")["nodes"]
        for n in nodes:
            if n["kind"] == 3:
                n_k4 += 1
                assert 3 <= n["tm"] <= 7 and 3 <= n["tn"] <= 7 and n["tm"] + n["tn"] <= 13
                assert 2 <= n["tk"] <= 5 and n["KG"] == 1 and n["smem"] <= 200 * 1024
                assert n["block"] == 32 * (2 ** (n["tm"] - 3) // n["RM"]) * (2 ** (n["tn"] - 3) // n["RN"])
                assert n["n_out"] == 2 ** (n["tm"] + n["tn"] + n["n_outer"])
        ref = np.array(contract.slice_values(build_network(circ, bits), plan.ssa_path, plan.sliced_labels))
        v = jet.debug_emulate_host(plan, 0, len(ref), "c128")
        assert np.max(np.abs(v - ref)) <= 1e-12 * max(np.max(np.abs(ref)), 1e-300)
    assert n_k4 > 0, "no node was routed to K4"


def test_emulated_k2s_and_k3_tma_match_oracle_grid(monkeypatch):
    """K2s (register-resident streaming GETT) and K3-TMA descriptors on a 4x5 m=10 grid circuit
    with 4 sliced labels: the emulated column offsets (every column), TMA landings (every tile) and
    the emulated contraction match the oracle's s_sigma on every slice (c64 arithmetic, 1e-4)."""
    import paper_2107_09793_b200.jet as jet
    from circuits import grid_rqc, random_bitstring

    monkeypatch.setenv("JETB200_TMA_MINCOPY", "16")
    circ = grid_rqc(4, 5, 10, 1)
    bits = random_bitstring(20, 2, 1)
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=1, trials=32, n_sliced=4)
    nodes = plan.describe_exec("c64")["nodes"]
    assert sum(n["kind"] == 4 for n in nodes) >= 1 and any(n["kind"] == 1 and n["tma"] for n in nodes)
    ref = np.array(contract.slice_values(build_network(circ, bits), plan.ssa_path, plan.sliced_labels))
    v = jet.debug_emulate_host(plan, 0, 16, "c64")
    assert np.max(np.abs(v - ref) / np.abs(ref)) < 1e-4


def test_emulated_k3_mlow_layout_matches_oracle(jet, monkeypatch):
    """K3 with the [M][rows][outer] output layout (JETB200_K3_MLOW=1) on C2: emulated descriptors
    (the layout propagates into every consumer's strides) match the oracle."""
    monkeypatch.setenv("JETB200_K3_MLOW", "1")
    circ, bits = workload("C2")
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=1, trials=64, n_sliced=6, bytes_weight=5.0)
    ref = np.array(contract.slice_values(build_network(circ, bits), plan.ssa_path, plan.sliced_labels, indices=[7]))
    v = jet.debug_emulate_host(plan, 7, 8, "c64")
    assert np.max(np.abs(v - ref) / np.abs(ref)) < 1e-4




def test_emulated_k2s_pair_loads_match_oracle():
    """K2s with 16-B k-pair loads (B's stride-1 bit contracted, as on the benched C3 plan's heavy
    skinny nodes) on a 5x5 m=10 grid circuit: the emulated descriptors (column tables, pair
    alignment, [n_lo][M][rest] output layout) against the oracle on every slice (1e-4)."""
    import paper_2107_09793_b200.jet as jet
    from circuits import grid_rqc

    circ = grid_rqc(5, 5, 10, 1)
    bits = random_bitstring(25, 2, 1)
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=1, trials=16, n_sliced=4)
    ks = [n for n in plan.describe_exec("c64")["nodes"] if n["kind"] == 4]
    assert any(n["st_vec"] for n in ks) and any(not n["st_vec"] for n in ks)
    for n in ks:
        if n["st_vec"]:
            assert n["stK"][0] == 1 and all(s % 2 == 0 for s in n["stN"] + n["stK"][1:])
    ref = np.array(contract.slice_values(build_network(circ, bits), plan.ssa_path, plan.sliced_labels))
    v = jet.debug_emulate_host(plan, 0, 16, "c64")
    assert np.max(np.abs(v - ref) / np.abs(ref)) < 1e-4
