"""Pins for the CPU oracle.  CPU only."""

import itertools
import json
import math
import os

import numpy as np
import pytest

from circuits import Circuit, generate_gbs, grid_rqc, random_bitstring, SplitMix64
from circuits.gates import CZ, HADAMARD, beamsplitter, fsim, squeezer, SYC_1Q
from circuits.sycamore import coupler_patterns, sycamore53, sycamore_qubits
from oracle import contract, cost, naive, path, statevector
from oracle.network import build_network


def worked_example(bits, d=2, s=HADAMARD, b=CZ):
    c = Circuit(2, d)
    c.add((0,), s)
    c.add((1,), s)
    c.add((0, 1), b)
    return c, build_network(c, bits)


# ---------------------------------------------------------------- P1 worked example
def test_worked_example_amplitudes(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "worked_example.json")))
    p = [tuple(x) for x in g["paper_path_ssa"]]
    for key, (re, im) in g["amplitudes"].items():
        bits = [int(ch) for ch in key]
        _, net = worked_example(bits)
        # Eq. sequence path (l.97-102), Eq. naive_summation (l.87) and a greedy path agree
        a_seq = contract.amplitude(net, p)
        a_naive = naive.full_sum(net)
        a_greedy = contract.amplitude(net, path.greedy_path(net))
        for a in (a_seq, a_naive, a_greedy):
            assert abs(a - complex(re, im)) < 1e-14


def test_worked_example_structure(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "worked_example.json")))
    p = [tuple(x) for x in g["paper_path_ssa"]]
    _, net = worked_example([0, 0])
    # tensors: |0>_a, |0>_d, S_ba, S_ed, B_cfbe, <a1|_c, <a2|_f  (l.81-83)
    a, d_, b, e, c, f = 0, 1, 2, 3, 4, 5
    assert net.labels == [(a,), (d_,), (b, a), (e, d_), (c, f, b, e), (c,), (f,)]
    # per-step costs D^4, D^2, D^2, D^3, D^2, D (l.97-102), 8 real FLOP per complex MAC
    steps = cost.tree_info(net, p, [])
    assert [fl for fl, _ in steps] == [8 * 2 ** k for k in g["paper_path_cost_exponents"]]
    # intermediate label sets T1_fbe, T2_e, T3_b, T4_be, T5_b, scalar
    vals, labs = {}, {}
    for t in range(net.n_tensors):
        vals[t], labs[t] = net.tensors[t], net.labels[t]
    nid = net.n_tensors
    want = [(f, b, e), (e,), (b,), (b, e), (b,), ()]
    for (i, j), w in zip(p, want):
        vals[nid], labs[nid] = contract.contract_pair(vals[i], labs[i], vals[j], labs[j])
        assert labs[nid] == w
        nid += 1


def test_worked_example_slicing_e(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "worked_example.json")))["slice_e_values_for_00"]
    p = [(5, 4), (3, 1), (2, 0), (6, 7), (10, 8), (9, 11)]
    _, net = worked_example([0, 0])
    e = 3
    s = contract.slice_values(net, p, [e])
    assert abs(s[0] - complex(*g["s0"])) < 1e-15 and abs(s[1] - complex(*g["s1"])) < 1e-15
    assert abs(sum(s) - 0.5) < 1e-15                                  # Eq. sliced_sum 3)
    rep = cost.cost_report(net, p, [e])
    assert rep["n_sl"] == 2
    # fig. 3: grey = "sliced or the result of a contraction involving a sliced tensor";
    # B_cfbe and S_ed carry e, so only T3 = sum_a S_ba |0>_a is shared
    steps = cost.tree_info(net, p, [e])
    assert [bool(sv) for _, sv in steps] == [True, True, False, True, True, True]
    assert rep["e_fltask"] < rep["e_flsl"]


def test_worked_example_cost_counters_by_hand():
    """Eq. sliced_flops and Eq. task_based_amplitude_flops on the worked
    example sliced on e (D = 2, path of Eq. sequence), every counter computed by hand:
      step (<c|, B_cfbe|e)   union {c,f,b}  8*2^3 = 64   S = {e}
      step (S_ed|e, |0>_d)   union {d}      8*2   = 16   S = {e}
      step (S_ba, |0>_a)     union {b,a}    8*2^2 = 32   S = {}    (T3, the shared task)
      step (<f|, T1_fb)      union {f,b}    8*2^2 = 32   S = {e}
      step (T4_b, T2)        union {b}      8*2   = 16   S = {e}
      step (T3_b, T5_b)      union {b}      8*2   = 16   S = {e}
    FLOP_sl = 176, shared = 32, f_sl = 32/176 (a fraction of FLOP, not of tasks),
    E-flsl = 2 * 176 = 352, E-fltask = f_sl FLOP_sl + N_sl (1 - f_sl) FLOP_sl = 32 + 2 * 144 = 320;
    exact dedup and the one-copy prefix cache (order [e]) both run T3 once: 320."""
    p = [(5, 4), (3, 1), (2, 0), (6, 7), (10, 8), (9, 11)]
    _, net = worked_example([0, 0])
    rep = cost.cost_report(net, p, [3])
    assert [f for f, _ in cost.tree_info(net, p, [3])] == [64, 16, 32, 32, 16, 16]
    assert rep["flop_sl"] == 176 and rep["flop_shared"] == 32
    assert rep["e_flsl"] == 352
    assert rep["e_fltask"] == 320          # a per-task f_sl (1 of 6 nodes) would give 322.67
    assert rep["exact_reuse"] == 320 and rep["prefix"] == 320
    assert cost.prefix_flop(net, p, [3], 0, 1) == 176 and cost.prefix_flop(net, p, [3], 1, 2) == 176


def test_slice_assignment_is_the_lexicographic_enumeration():
    """contract.slice_assignment(i) (direct mixed radix, used for N_sl up to 2^36) is the i-th
    element of the itertools enumeration with sliced_labels[0] most significant (reading A12),
    on mixed dimensions 2, 3, 4."""
    c = Circuit(3, 2)
    c.add((0, 1), np.eye(4))
    net = build_network(c, [0, 0, 0])
    net.dims = {0: 2, 1: 3, 2: 4, 3: 2, 4: 3}
    sl = [2, 0, 1]
    allsig = list(contract.slice_assignments(net, sl))
    assert len(allsig) == 24
    for i, sig in enumerate(allsig):
        assert contract.slice_assignment(net, sl, i) == sig
    assert allsig[1] == {2: 0, 0: 0, 1: 1} and allsig[3] == {2: 0, 0: 1, 1: 0}
    with pytest.raises(ValueError):
        contract.slice_assignment(net, sl, 24)


def test_worked_example_qutrit_vs_statevector():
    d = 3
    w = np.exp(2j * np.pi / 3)
    dft = np.array([[w ** (i * j) for j in range(3)] for i in range(3)]) / math.sqrt(3)
    rng = np.random.default_rng(5)
    m = rng.normal(size=(9, 9)) + 1j * rng.normal(size=(9, 9))
    q, _ = np.linalg.qr(m)
    for bits in itertools.product(range(3), repeat=2):
        c, net = worked_example(list(bits), d=3, s=dft, b=q)
        a = contract.amplitude(net, path.greedy_path(net))
        assert abs(a - statevector.amplitude(c, bits)) < 1e-14
        assert abs(a - naive.full_sum(net)) < 1e-14


# ---------------------------------------------------------------- pairwise step vs loops
def test_contract_pair_matches_nested_loops():
    rng = np.random.default_rng(0)
    for trial in range(30):
        dims = {l: int(rng.integers(1, 4)) for l in range(7)}
        la = tuple(int(x) for x in rng.permutation(7)[: rng.integers(0, 5)])
        lb = tuple(int(x) for x in rng.permutation(7)[: rng.integers(0, 5)])
        a = rng.normal(size=[dims[l] for l in la]) + 1j * rng.normal(size=[dims[l] for l in la])
        b = rng.normal(size=[dims[l] for l in lb]) + 1j * rng.normal(size=[dims[l] for l in lb])
        c1, l1 = contract.contract_pair(a, la, b, lb)
        c2, l2 = contract.contract_pair_loops(a, la, b, lb)
        assert l1 == l2
        np.testing.assert_allclose(c1, c2, rtol=0, atol=1e-12)


def test_contract_pair_mismatch_raises():
    with pytest.raises(ValueError):
        contract.contract_pair(np.ones((2, 3)), (0, 1), np.ones((2, 2)), (1, 2))


# ---------------------------------------------------------------- P2/P3 C1 vs state vector
@pytest.fixture(scope="module")
def c1():
    circ = grid_rqc(3, 3, 8, seed=1)
    return circ, statevector.final_state(circ)


def test_c1_all_amplitudes_vs_statevector(c1):
    circ, psi = c1
    net0 = build_network(circ, [0] * 9)
    p = path.greedy_path(net0)
    tot = 0.0
    for bits in itertools.product(range(2), repeat=9):
        net = build_network(circ, list(bits))
        a = contract.amplitude(net, p)
        assert abs(a - psi[bits]) < 1e-12
        tot += abs(a) ** 2
    assert abs(tot - 1.0) < 1e-12                                        # P3


def test_batch_amplitudes_vs_statevector(c1):
    """f1 batch of amplitudes: the y-th amplitude of the batch equals the
    state-vector entry of the y-th batch bitstring (open_wires[0] most significant), and the
    per-run values s_(sigma, y) sum over sigma to it (Eq. sliced_sum per bitstring)."""
    circ, psi = c1
    base = [1, 0, 1, 1, 0, 0, 1, 0, 1]
    p = path.greedy_path(build_network(circ, base))
    for open_wires in ([4], [7, 2], [8, 0, 3], list(range(9))):
        amps = contract.batch_amplitudes(circ, base, open_wires, p)
        assert len(amps) == 2 ** len(open_wires)
        for y, a in enumerate(amps):
            x = list(base)
            for i, w in enumerate(open_wires):
                x[w] = (y >> (len(open_wires) - 1 - i)) & 1
            assert abs(a - psi[tuple(x)]) < 1e-12
    net = build_network(circ, base)
    sliced = sorted(l for l, ts in net.carriers().items() if 9 <= l < 40)[:3]
    open_wires = [5, 1]
    runs = contract.batch_run_values(circ, base, open_wires, p, sliced, range(8 * 4))
    amps = contract.batch_amplitudes(circ, base, open_wires, p)
    for y in range(4):
        assert abs(sum(runs[s * 4 + y] for s in range(8)) - amps[y]) < 1e-12


def test_statevector_norm_sycamore_grid():
    for seed in (2, 3):
        psi = statevector.final_state(grid_rqc(3, 4, 6, seed))
        assert abs(np.vdot(psi, psi).real - 1.0) < 1e-12


def test_random_small_circuits_vs_statevector():
    """SPEC.md acceptance 1: >=200 random circuits, qudit d in {2,3,4}, <=6 wires, depth<=6."""
    rng = np.random.default_rng(11)
    count = 0
    while count < 200:
        d = int(rng.integers(2, 5))
        n = int(rng.integers(1, 6 if d < 4 else 5))
        c = Circuit(n, d)
        for _ in range(int(rng.integers(0, 7))):
            k = 1 if n == 1 else int(rng.integers(1, 3))
            wires = rng.permutation(n)[:k]
            m = rng.normal(size=(d ** k, d ** k)) + 1j * rng.normal(size=(d ** k, d ** k))
            q, _ = np.linalg.qr(m)
            c.add(wires, q)
        bits = [int(rng.integers(0, d)) for _ in range(n)]
        net = build_network(c, bits)
        a = contract.amplitude(net, path.greedy_path(net))
        assert abs(a - statevector.amplitude(c, bits)) < 1e-10
        count += 1


# ---------------------------------------------------------------- P4/P5 slicing and paths
def test_slice_sum_identity_and_path_independence(c1):
    circ, psi = c1
    bits = random_bitstring(9, 2, 7)
    net = build_network(circ, bits)
    p1 = path.greedy_path(net)
    p2 = path.greedy_path(net, order_key="reverse")
    assert p1 != p2
    a1 = contract.amplitude(net, p1)
    a2 = contract.amplitude(net, p2)
    assert abs(a1 - a2) < 1e-12                                            # P5
    assert abs(a1 - psi[tuple(bits)]) < 1e-12
    bonds = sorted(net.dims)
    rng = np.random.default_rng(3)
    for _ in range(20):
        k = int(rng.integers(1, 4))
        sl = [int(x) for x in rng.choice(bonds, size=k, replace=False)]
        s = contract.slice_values(net, p1, sl)
        assert len(s) == 2 ** k
        assert abs(sum(s) - a1) < 1e-12                                    # P4


def test_slice_validation():
    _, net = worked_example([0, 0])
    p = [(5, 4), (3, 1), (2, 0), (6, 7), (10, 8), (9, 11)]
    with pytest.raises(ValueError):
        contract.slice_values(net, p, [99])
    with pytest.raises(ValueError):
        contract.validate_path(net.n_tensors, [(0, 0)])
    with pytest.raises(ValueError):
        contract.validate_path(net.n_tensors, p[:-1])


# ---------------------------------------------------------------- P9 gates
def test_squeezer_closed_forms(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "gate_closed_forms.json")))
    np.testing.assert_allclose(squeezer(0.0, 6), np.eye(6), atol=1e-15)
    s = squeezer(g["r"], 6)
    assert abs(s[0, 0] - g["S_00"]) < 1e-12
    assert abs(s[2, 0] - g["S_20"]) < 1e-12
    assert abs(s[4, 0] - g["S_40"]) < 1e-12
    assert abs(s[1, 0]) < 1e-15 and abs(s[3, 0]) < 1e-15                 # parity


def test_beamsplitter_properties():
    rng = SplitMix64(3)
    for d in (2, 3, 4):
        np.testing.assert_allclose(beamsplitter(0.0, 1.3, d), np.eye(d * d), atol=1e-15)
        for _ in range(5):
            th, ph = 2 * math.pi * rng.uniform(), 2 * math.pi * rng.uniform()
            u = beamsplitter(th, ph, d)
            for p_, q_, n_, m_ in itertools.product(range(d), repeat=4):
                if p_ + q_ != n_ + m_:
                    assert u[d * p_ + q_, d * n_ + m_] == 0                # number conserving
            for N in range(d):                                              # complete blocks unitary
                idx = [d * k + (N - k) for k in range(N + 1)]
                blk = u[np.ix_(idx, idx)]
                np.testing.assert_allclose(blk.conj().T @ blk, np.eye(N + 1), atol=1e-13)
    for ph in (0.0, 0.7):                                                   # Hong-Ou-Mandel
        u = beamsplitter(math.pi / 4, ph, 4)
        assert abs(u[4 * 1 + 1, 4 * 1 + 1]) < 1e-15
    u = beamsplitter(math.pi / 2, 0.0, 2)                                   # full reflection
    assert abs(abs(u[2 * 0 + 1, 2 * 1 + 0]) - 1) < 1e-15


def test_sycamore_gate_set():
    for g in SYC_1Q + (fsim(math.pi / 2, math.pi / 6),):
        np.testing.assert_allclose(g.conj().T @ g, np.eye(g.shape[0]), atol=1e-15)


# ---------------------------------------------------------------- P8 GBS closed forms
from gbs_closed import p8_cases, single_photon_matrix  # noqa: E402


@pytest.mark.parametrize("dim,width,d", [(2, 2, 4), (3, 2, 4), (1, 4, 4), (2, 2, 8)])
def test_gbs_closed_forms(dim, width, d):
    r = 0.5
    circ = generate_gbs(dim, width, 1, r, d, seed=9)
    M = circ.n_wires
    pref = math.cosh(r) ** (-M / 2)
    W = single_photon_matrix(circ)
    B = math.tanh(r) * W @ W.T
    net0 = build_network(circ, [0] * M)
    p = path.greedy_path(net0)
    cases = [([0] * M, pref)]
    for i in range(M):
        for j in range(i + 1, M):
            x = [0] * M
            x[i] = x[j] = 1
            cases.append((x, pref * B[i, j]))
        x = [0] * M
        x[i] = 2
        cases.append((x, pref * B[i, i] / math.sqrt(2)))
    x = [0] * M
    x[0] = 1
    cases.append((x, 0.0))                                                 # odd photon number
    x = [0] * M
    x[-1] = 3
    cases.append((x, 0.0))
    for bits, want in cases[:40]:
        a = contract.amplitude(build_network(circ, bits), p)
        assert abs(a - want) < 1e-12, (bits, a, want)
    if M <= 4:   # same truncated matrices through the state vector
        for bits, _ in cases:
            assert abs(contract.amplitude(build_network(circ, bits), p)
                       - statevector.amplitude(circ, bits)) < 1e-12


# ---------------------------------------------------------------- P11 Alg. 1 counts
def test_alg1_counts():
    c = generate_gbs(3, 4, 1, 0.5, 4, seed=1)
    assert sum(1 for g in c.gates if len(g.wires) == 1) == 64
    assert sum(1 for g in c.gates if len(g.wires) == 2) == 63 + 60 + 48
    c = generate_gbs(1, 4, 1, 0.5, 4, seed=1)
    assert [g.wires for g in c.gates] == [(0,), (1,), (2,), (3,), (0, 1), (1, 2), (2, 3)]
    c1 = generate_gbs(2, 3, 2, 0.5, 3, seed=4)
    c2 = generate_gbs(2, 3, 2, 0.5, 3, seed=4)
    c3 = generate_gbs(2, 3, 2, 0.5, 3, seed=5)
    assert all(np.array_equal(a.u, b.u) for a, b in zip(c1.gates, c2.gates))
    assert not all(np.array_equal(a.u, b.u) for a, b in zip(c1.gates, c3.gates))
    assert len(c1.gates) == 9 + 2 * ((9 - 1) + (9 - 3))


def test_sycamore_generator_structure():
    qs = sycamore_qubits(53)
    assert len(qs) == 53
    pats = coupler_patterns(qs)
    assert sum(len(p) for p in pats.values()) == 86                        # Sycamore-53 couplers
    c = sycamore53(14, seed=1)
    assert sum(1 for g in c.gates if len(g.wires) == 1) == 53 * 15
    last = {}
    for g in c.gates:
        if len(g.wires) == 1:
            w = g.wires[0]
            assert last.get(w) != g.name
            last[w] = g.name


# ---------------------------------------------------------------- P12 FLOP identities
def test_cost_identities_bruteforce(c1):
    circ, _ = c1
    net = build_network(circ, [1, 0, 1, 0, 0, 1, 1, 0, 1])
    p = path.greedy_path(net)
    rng = np.random.default_rng(8)
    bonds = sorted(net.dims)
    for _ in range(10):
        sl = [int(x) for x in rng.choice(bonds, size=3, replace=False)]
        rep = cost.cost_report(net, p, sl)
        steps = cost.tree_info(net, p, sl)
        # exact dedup = distinct task names "(step, sigma|S(v))" (reading A9), enumerated
        names = set()
        for sig in contract.slice_assignments(net, sl):
            for s, (f, sv) in enumerate(steps):
                names.add((s, tuple(sorted((l, sig[l]) for l in sv))))
        assert rep["exact_reuse"] == sum(steps[s][0] for s, _ in names)
        assert rep["e_flsl"] == rep["n_sl"] * rep["flop_sl"]
        assert rep["e_fltask"] <= rep["e_flsl"]
        assert rep["exact_reuse"] <= rep["prefix"] <= rep["e_flsl"]
        # prefix closed form: v recomputed prod_{pos <= maxpos(S(v))} d times
        pos = {l: i for i, l in enumerate(sl)}
        closed = 0
        for f, sv in steps:
            mp = max((pos[l] for l in sv), default=-1)
            closed += f * (2 ** (mp + 1))
        assert rep["prefix"] == closed
        # split ranges: sum over blocks >= whole (each block restarts its cache)
        half = rep["n_sl"] // 2
        a = cost.prefix_flop(net, p, sl, 0, half)
        b = cost.prefix_flop(net, p, sl, half, rep["n_sl"])
        assert a + b >= rep["prefix"]


def test_p7_slice_closed_form_matches_oracle():
    """The P7 per-slice closed form (tests/p7_closed.py) used to pin the GPU path at C3/C5 size
    equals the oracle's s_sigma on a 3x3 grid with fSim(0, 0) = I, for random sliced labels and
    every slice (and so do their sums, Eq. sliced_sum)."""
    from circuits.sycamore import grid_qubits, random_circuit
    from p7_closed import slice_closed_form

    circ = random_circuit(grid_qubits(3, 3), 8, seed=3, theta=0.0, phi=0.0)
    rng = np.random.default_rng(4)
    for t in range(4):
        bits = [int(b) for b in rng.integers(0, 2, size=9)]
        net = build_network(circ, bits)
        p = path.greedy_path(net)
        sl = [int(x) for x in rng.choice(sorted(net.dims), size=4, replace=False)]
        ref = contract.slice_values(net, p, sl)
        for i, r in enumerate(ref):
            assert abs(slice_closed_form(circ, bits, sl, i) - r) < 1e-13
