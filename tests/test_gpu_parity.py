"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Tolerances (BASELINE.json north_star, reading A13): relative amplitude error 1e-4 for
complex64 and 1e-10 for complex128, rel = |a_gpu - a_ora| / |a_ora|; every s_sigma is
compared with the same rule.  K1 permutes are compared bit-exactly."""

import math

import numpy as np
import pytest

from circuits import Circuit, generate_gbs, grid_rqc, random_bitstring, workload
from circuits.sycamore import random_circuit, sycamore_qubits
from oracle import contract, statevector
from oracle.network import build_network

pytestmark = pytest.mark.gpu

TOL = {"c64": 1e-4, "c128": 1e-10}


@pytest.fixture(scope="module")
def jet():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build()
    from paper_2107_09793_b200 import jet as j

    torch.cuda.set_device(0)
    return j


def run(jet, plan, dtype, reuse=True, ranges=None):
    import torch

    ex = jet.Exec(plan, dtype)
    n_sl = plan.cost()["n_sl"]
    acc = torch.zeros(2, dtype=torch.float64, device="cuda")
    vals = []
    for b, e in (ranges or [(0, n_sl)]):
        vals.append(ex.contract(b, e, acc, slice_values=True, reuse=reuse))
    torch.cuda.synchronize()
    return complex(acc[0].item(), acc[1].item()), np.concatenate(vals), ex


def rel(a, b):
    return abs(a - b) / abs(b)


# ----------------------------------------------------------------------------- K1 permute
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("n", [0, 1, 3, 7, 12, 16, 21])
def test_permute_bit_exact(jet, dtype, n):
    import torch

    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    rng = np.random.default_rng(n)
    src = torch.randn(1 << n, dtype=tdt, device="cuda")
    perms = [list(range(n)), list(reversed(range(n))), list(rng.permutation(n))]
    if n >= 4:
        perms.append(list(range(1, n)) + [0])
    idx = np.arange(1 << n)
    s = src.cpu().numpy()
    for perm in perms:
        dst = jet.permute(src, perm)
        didx = np.zeros_like(idx)
        for b, p in enumerate(perm):
            didx |= ((idx >> b) & 1) << int(p)
        want = np.empty_like(s)
        want[didx] = s
        assert np.array_equal(dst.cpu().numpy(), want)


# ----------------------------------------------------------------------------- C1 (3x3, m=8)
@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("k", [0, 2, 4])
def test_c1_parity_vs_oracle_and_statevector(jet, dtype, k):
    circ, _ = workload("C1")
    psi = statevector.final_state(circ)
    for seed in range(6):
        bits = random_bitstring(9, 2, 100 + seed)
        net = jet.Network.from_circuit(circ, bits)
        plan = jet.Plan.greedy(net, seed=seed, trials=16, n_sliced=k)
        onet = build_network(circ, bits)
        ref_vals = contract.slice_values(onet, plan.ssa_path, plan.sliced_labels)
        ref = sum(ref_vals)
        assert abs(ref - psi[tuple(bits)]) < 1e-12
        amp, vals, _ = run(jet, plan, dtype)
        assert rel(amp, ref) < TOL[dtype]
        for v, r in zip(vals, ref_vals):   # A13: the same rule for every s_sigma, no floor
            assert abs(v - r) <= TOL[dtype] * abs(r), (v, r)


def test_reuse_on_off_bitwise_and_ranges(jet):
    """P10: prefix-cache reuse on vs off gives bitwise-identical s_sigma; splitting the slice
    range across calls (the cache persists) also gives identical values."""
    circ, bits = workload("C1")
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=3, trials=16, n_sliced=5)
    n = plan.cost()["n_sl"]
    for dtype in ("c64", "c128"):
        _, v_on, ex_on = run(jet, plan, dtype, reuse=True)
        _, v_off, ex_off = run(jet, plan, dtype, reuse=False)
        _, v_rng, _ = run(jet, plan, dtype, ranges=[(0, 7), (7, 19), (19, n)])
        assert np.array_equal(v_on, v_off)
        assert np.array_equal(v_on, v_rng)
        # executed FLOP equals the cost model (P12): prefix cache vs E-flsl
        c = plan.cost()
        assert ex_on.stats()["flop_executed"] == c["prefix"]
        assert ex_off.stats()["flop_executed"] == c["e_flsl"]


def test_contract_host_and_amplitude_api(jet):
    circ, bits = workload("C1")
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=1, trials=8, n_sliced=2)
    ref = contract.amplitude(build_network(circ, bits), plan.ssa_path, plan.sliced_labels)
    ex = jet.Exec(plan, "c128")
    assert rel(ex.contract_host(0, 4), ref) < 1e-10
    assert rel(jet.amplitude(plan, "c128"), ref) < 1e-10
    assert rel(jet.amplitude(plan, "c64"), ref) < 1e-4


def test_errors(jet):
    import torch

    circ, bits = workload("C1")
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=1, trials=8, n_sliced=2)
    import ctypes
    from paper_2107_09793_b200.jet import _check, _lib, c_vp

    small = torch.empty(256, dtype=torch.uint8, device="cuda")
    h = c_vp()
    with pytest.raises(jet.JetError) as e:
        _check(_lib.jt_exec_create(plan._h, 0, 0, c_vp(small.data_ptr()), 256, None, ctypes.byref(h)))
    assert e.value.code == 4
    ex = jet.Exec(plan, "c64")
    acc = torch.zeros(2, dtype=torch.float64, device="cuda")
    with pytest.raises(jet.JetError) as e:
        ex.contract(0, 5, acc)
    assert e.value.code == 2
    q = Circuit(2, 3)
    q.add((0, 1), np.eye(9))
    qnet = jet.Network.from_circuit(q, [0, 0])
    qplan = jet.Plan.greedy(qnet)
    with pytest.raises(jet.JetError) as e:
        jet.Exec(qplan, "c64")
    assert e.value.code == 2


# ----------------------------------------------------------------------------- GBS (qudits, d=4)
@pytest.mark.parametrize("dim,width", [(2, 2), (3, 2)])
def test_gbs_parity_and_closed_forms(jet, dim, width):
    r, d = 0.5, 4
    circ = generate_gbs(dim, width, 1, r, d, seed=9)
    M = circ.n_wires
    cases = [[0] * M, random_bitstring(M, d, 1), random_bitstring(M, d, 2)]
    x = [0] * M
    x[0] = x[M - 1] = 1
    cases.append(x)
    for k, bits in enumerate(cases):
        net = jet.Network.from_circuit(circ, bits)
        plan = jet.Plan.greedy(net, seed=k, trials=16, n_sliced=min(k, 2))
        ref = contract.amplitude(build_network(circ, bits), plan.ssa_path, plan.sliced_labels)
        amp, _, _ = run(jet, plan, "c128")
        if abs(ref) < 1e-14:
            assert abs(amp) < 1e-14
        else:
            assert rel(amp, ref) < 1e-10
        if bits == [0] * M:
            assert abs(amp - math.cosh(r) ** (-M / 2)) < 1e-12            # P8 vacuum


# ----------------------------------------------------------------------------- K4 (c128 DMMA)
@pytest.mark.parametrize("form", ["3M", "4M"])
@pytest.mark.parametrize("dim,width,d,k", [(2, 3, 4, 0), (2, 4, 4, 2), (2, 2, 8, 1), (3, 2, 4, 1), (2, 4, 4, 3)])
def test_k4_dmma_parity_vs_oracle_and_k2(jet, monkeypatch, dim, width, d, k, form):
    """c128 contractions on the FP64 tensor cores (K4: the 4M form by default and the 3M Gauss
    form with JETB200_K4_3M=1) against the oracle (1e-10) and against the CUDA-core K2 path
    (JETB200_DMMA=0) on the same plan."""
    monkeypatch.setenv("JETB200_K4_3M", "1" if form == "3M" else "0")
    circ = generate_gbs(dim, width, 1, 0.5, d, seed=5)
    M = circ.n_wires
    bits = random_bitstring(M, d, 11)
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=1, trials=16, n_sliced=k)
    k4 = [n for n in plan.describe_exec("c128")["nodes"] if n["kind"] == 3]
    assert k4
    assert any(n["gauss"] for n in k4) == (form == "3M")
    ref_vals = np.array(contract.slice_values(build_network(circ, bits), plan.ssa_path, plan.sliced_labels))
    ref = complex(np.sum(ref_vals))
    amp, vals, _ = run(jet, plan, "c128")
    scale = np.max(np.abs(ref_vals))
    assert np.max(np.abs(vals - ref_vals)) <= 1e-10 * scale
    if abs(ref) <= 1e-14 * scale:   # odd total photon number: exactly 0 (P8)
        assert abs(amp) <= 1e-12 * scale
    else:
        assert rel(amp, ref) < 1e-10
    monkeypatch.setenv("JETB200_DMMA", "0")
    assert not any(n["kind"] == 3 for n in plan.describe_exec("c128")["nodes"])
    amp2, vals2, _ = run(jet, plan, "c128")
    assert np.max(np.abs(vals2 - vals)) <= 1e-12 * scale


@pytest.mark.parametrize("name", ["G88d4"])
def test_gbs88_closed_forms_full_size(jet, name):
    """f4: GBS-88-m1 (64 modes, cutoff 4) at full size on K4/K2, pinned by the
    P8 closed forms (vacuum, sampled two-photon outputs, odd photon numbers) within 1e-10."""
    from gbs_closed import p8_cases

    circ, _ = workload(name)
    cases = p8_cases(circ, 0.5, max_pairs=12, seed=3)
    plan = None
    for bits, want in cases:
        net = jet.Network.from_circuit(circ, bits)
        if plan is None:
            plan = jet.Plan.greedy(net, seed=1, trials=64)
            assert any(n["kind"] == 3 for n in plan.describe_exec("c128")["nodes"])
            ssa, sl = plan.ssa_path, plan.sliced_labels
        else:   # same network shape, new bra digits: the same path
            plan = jet.Plan.create(net, ssa, sl)
        amp, _, _ = run(jet, plan, "c128")
        if want == 0.0:
            assert abs(amp) < 1e-14
        else:
            assert rel(amp, want) < 1e-10, (bits, amp, want)


# ----------------------------------------------------------------------------- C2 (Sycamore-53 m=10)
@pytest.fixture(scope="module")
def c2_plan(jet):
    circ, bits = workload("C2")
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=1, trials=256, n_sliced=6, bytes_weight=5.0)
    kinds = [n["kind"] for n in plan.describe_exec("c64")["nodes"]]
    assert sum(kinds) >= 10, "the C2 plan should exercise the K3 tensor-core kernel"
    return circ, bits, net, plan


@pytest.fixture(scope="module")
def c2_ref(c2_plan):
    circ, bits, net, plan = c2_plan
    return contract.slice_values(build_network(circ, bits), plan.ssa_path, plan.sliced_labels)


def test_c2_full_parity(jet, c2_plan, c2_ref):
    circ, bits, net, plan = c2_plan
    ref_vals = c2_ref
    ref = sum(ref_vals)
    assert abs(ref) ** 2 * 2 ** 53 > 0.01                                    # reading A13
    amp, vals, ex = run(jet, plan, "c64")
    assert rel(amp, ref) < 1e-4
    for v, r in zip(vals, ref_vals):
        assert abs(v - r) <= 1e-4 * abs(r)
    assert ex.stats()["flop_executed"] == plan.cost()["prefix"]


def test_c2_full_parity_c128(jet, c2_plan, c2_ref):
    """The same 64 slices in complex128 (K2 FP64 + K4 DMMA on the Sycamore shapes) at 1e-10."""
    circ, bits, net, plan = c2_plan
    assert any(n["kind"] == 3 for n in plan.describe_exec("c128")["nodes"])
    amp, vals, ex = run(jet, plan, "c128")
    ref = sum(c2_ref)
    assert rel(amp, ref) < 1e-10
    for v, r in zip(vals, c2_ref):
        assert abs(v - r) <= 1e-10 * abs(r)


def test_c2_fsim_identity_closed_form(jet):
    """P7: fSim(0,0) = I makes the 53-qubit circuit a product of 1-qubit chains, so
    <x|U|0> = prod_q <x_q|V_q|0>; same network structure and cost as C2."""
    qs = sycamore_qubits(53)
    circ = random_circuit(qs, 10, seed=1, theta=0.0, phi=0.0)
    bits = random_bitstring(53, 2, 1)
    want = 1 + 0j
    for q in range(53):
        v = np.array([1, 0], dtype=np.complex128)
        for g in circ.gates:
            if g.wires == (q,):
                v = g.u @ v
        want *= v[bits[q]]
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=1, trials=64, n_sliced=6)
    for dtype in ("c64", "c128"):
        amp, _, _ = run(jet, plan, dtype)
        assert rel(amp, want) < TOL[dtype]


def test_k3_tensor_cores_vs_cuda_cores(jet, c2_plan, monkeypatch):
    """K3 (tcgen05 3xTF32) and K2 (CUDA-core FP32) give the same slices within c64 rounding."""
    circ, bits, net, plan = c2_plan
    monkeypatch.setenv("JETB200_TC", "0")
    assert sum(n["kind"] for n in plan.describe_exec("c64")["nodes"]) == 0
    amp0, v0, _ = run(jet, plan, "c64", ranges=[(0, 8)])
    monkeypatch.setenv("JETB200_TC", "1")
    amp1, v1, _ = run(jet, plan, "c64", ranges=[(0, 8)])
    # both are complex64 evaluations of a ~40-deep tree; each is within ~2e-5 of the oracle
    # (the parity bar is 1e-4), so they agree to within the sum
    assert np.max(np.abs(v1 - v0) / np.abs(v0)) < 5e-5
    assert rel(amp1, amp0) < 5e-5


def test_k3_consumer_layout_and_pair_gathers_parity(jet, monkeypatch):
    """Opt-in paths: consumer-ordered output layouts (a bit the parent contracts at stride 1) and
    K3's 16-B k-pair gathers, against the oracle on the full C2 slice set (1e-4)."""
    circ, bits = workload("C2")
    net = jet.Network.from_circuit(circ, bits)
    monkeypatch.setenv("JETB200_CONSUMER_LAYOUT", "1")
    monkeypatch.setenv("JETB200_K3_VEC", "1")
    monkeypatch.setenv("JETB200_K3_TMA", "0")   # the pair gathers belong to the cp.async path
    plan = jet.Plan.greedy(net, seed=1, trials=256, n_sliced=6, bytes_weight=5.0)
    nodes = plan.describe_exec("c64")["nodes"]
    assert any(n["kind"] == 1 and n["vecB"] == 1 for n in nodes)
    ref = np.array(contract.slice_values(build_network(circ, bits), plan.ssa_path, plan.sliced_labels))
    amp, vals, _ = run(jet, plan, "c64")
    assert np.max(np.abs(vals - ref) / np.abs(ref).max()) < 1e-4
    assert rel(amp, complex(np.sum(ref))) < 1e-4


def test_cuda_graph_replay_bitwise(jet, monkeypatch):
    """Per-level CUDA graphs (device-side slice digits) give the same s_sigma bit for bit as
    direct launches, across split ranges, and count the same executed FLOP."""
    import torch

    circ, bits = workload("C1")
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=4, trials=16, n_sliced=5)
    n = plan.cost()["n_sl"]
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("JETB200_GRAPHS", mode)
        stream = torch.cuda.Stream()
        ex = jet.Exec(plan, "c64", stream=stream)
        acc = torch.zeros(2, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        vals = np.concatenate([ex.contract(0, 11, acc, slice_values=True),
                               ex.contract(11, n, acc, slice_values=True)])
        torch.cuda.synchronize()
        out[mode] = (vals, ex.stats()["flop_executed"])
    assert np.array_equal(out["0"][0], out["1"][0])
    assert out["0"][1] == out["1"][1] == plan.cost()["prefix"]


# ----------------------------------------------------------------------------- C3 (Sycamore-53 m=14)
@pytest.fixture(scope="module")
def c3_plan(jet):
    from paper_2107_09793_b200.runtime import plan_best

    circ, bits = workload("C3")
    net = jet.Network.from_circuit(circ, bits)
    plan, _ = plan_best(net, 10, trials=1024, seed=1)
    return circ, bits, net, plan


def test_c3_full_size_sampled_slices(jet, c3_plan):
    """BASELINE config C3 at full size, in the bench's launch configuration: the oracle
    contracts two seeded slices of the same plan one by one and every s_sigma matches."""
    import torch

    circ, bits, net, plan = c3_plan
    n_sl = plan.cost()["n_sl"]
    picks = [0, int(np.random.default_rng(3).integers(1, n_sl))]
    onet = build_network(circ, bits)
    ref = contract.slice_values(onet, plan.ssa_path, plan.sliced_labels, indices=picks)
    stream = torch.cuda.Stream()
    ex = jet.Exec(plan, "c64", stream=stream)
    acc = torch.zeros(2, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for p_, r in zip(picks, ref):
        v = ex.contract(p_, p_ + 1, acc, slice_values=True)[0]
        assert abs(v - r) <= 1e-4 * abs(r), (p_, v, r)


def test_c3_fsim_identity_closed_form_full_amplitude(jet):
    """P7 at C3 scale: with fSim(0, 0) = I the full 1024-slice m=14 amplitude is the product
    of 53 one-qubit chains."""
    import torch

    from paper_2107_09793_b200.runtime import plan_best

    qs = sycamore_qubits(53)
    circ = random_circuit(qs, 14, seed=1, theta=0.0, phi=0.0)
    bits = random_bitstring(53, 2, 1)
    want = 1 + 0j
    for q in range(53):
        v = np.array([1, 0], dtype=np.complex128)
        for g in circ.gates:
            if g.wires == (q,):
                v = g.u @ v
        want *= v[bits[q]]
    net = jet.Network.from_circuit(circ, bits)
    plan, _ = plan_best(net, 10, trials=256, seed=1)
    stream = torch.cuda.Stream()
    ex = jet.Exec(plan, "c64", stream=stream)
    acc = torch.zeros(2, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ex.contract(0, plan.cost()["n_sl"], acc)
    torch.cuda.synchronize()
    amp = complex(acc[0].item(), acc[1].item())
    assert rel(amp, want) < 1e-4


@pytest.mark.parametrize("tmt_max,mincopy,seg,perm", [("6", "4096", "4", "1"), ("7", "4096", "4", "1"),
                                                      ("7", "16", "4", "1"), ("7", "16", "0", "1"),
                                                      ("6", "4096", "1", "1"), ("7", "4096", "4", "force"),
                                                      ("7", "4096", "0", "force")])
def test_k3g_streamed_operands_parity(jet, c2_plan, monkeypatch, tmt_max, mincopy, seg, perm):
    """K3g (tcgen05 with both operands streamed, K in 16-complex chunks): force the C2 nodes
    K3 would take onto K3g and compare 8 slices with the oracle (tile columns up to 64 complex
    with two accumulators, or up to 128 with one; seg 0 / 1: accumulation segments of 1 / 2
    chunks, i.e. the epilogue's bulk FP32 add-reductions of later segments; perm force: every
    operand whose chunk is not one TMA box bit-gathered into the K3g layout first)."""
    circ, bits, net, plan = c2_plan
    monkeypatch.setenv("JETB200_TCG_FORCE", "1")
    monkeypatch.setenv("JETB200_TCG_SEG", seg)
    monkeypatch.setenv("JETB200_TCG_PERM", perm)
    monkeypatch.setenv("JETB200_TCG_TMT", tmt_max)
    monkeypatch.setenv("JETB200_TMA_MINCOPY", mincopy)   # 16: every chunk on the TMA engine
    nodes = plan.describe_exec("c64")["nodes"]
    if mincopy == "16":
        assert any(n["kind"] == 2 and n["tma"] for n in nodes)
    if perm == "force":
        assert any(n["kind"] == 2 and (n["permA"] or n["permB"]) and n["tma"] for n in nodes)
    assert [n["kind"] for n in nodes].count(2) >= 10
    assert max(n["tc_tm"] for n in nodes if n["kind"] == 2) == int(tmt_max)
    idx = list(range(0, 64, 8))
    ref = contract.slice_values(build_network(circ, bits), plan.ssa_path, plan.sliced_labels, indices=idx)
    import torch

    ex = jet.Exec(plan, "c64")
    acc = torch.zeros(2, dtype=torch.float64, device="cuda")
    for i, r in zip(idx, ref):
        v = ex.contract(i, i + 1, acc, slice_values=True)[0]
        assert abs(v - r) <= 1e-4 * abs(r), (i, v, r)


# ------------------------------------------------------------- f1 batches of amplitudes
def run_batch(jet, plan, dtype, ranges):
    import torch

    c = plan.cost()
    ex = jet.Exec(plan, dtype)
    acc = torch.zeros(2 * c["n_batch"], dtype=torch.float64, device="cuda")
    vals = [ex.contract(b, e, acc, slice_values=True) for b, e in ranges]
    torch.cuda.synchronize()
    return acc.cpu().numpy().view(np.complex128), np.concatenate(vals), ex


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_c1_batch_all_512_amplitudes(jet, dtype):
    """Every wire open: one batch plan yields all 512 amplitudes of C1, each against the state
    vector and the oracle (f1); split ranges agree with one range."""
    circ, _ = workload("C1")
    psi = statevector.final_state(circ).reshape(-1)
    bits = [0] * 9
    net = jet.Network.from_circuit(circ, bits, open_wires=list(range(9)))
    plan = jet.Plan.greedy(net, seed=2, trials=16, n_sliced=2)
    n = plan.cost()["n_sl"] * 512
    amps, vals, ex = run_batch(jet, plan, dtype, [(0, 700), (700, n)])
    ref = np.array(contract.batch_amplitudes(circ, bits, list(range(9)), plan.ssa_path, plan.sliced_labels))
    assert np.max(np.abs(ref - psi)) < 1e-12
    assert np.max(np.abs(amps - ref) / np.abs(ref)) < TOL[dtype]
    assert ex.stats()["flop_executed"] == plan.prefix_flop(0, n)
    amps1 = jet.amplitude(plan, dtype)
    assert np.max(np.abs(amps1 - ref) / np.abs(ref)) < TOL[dtype]


def test_c2_batch_sampled_runs(jet):
    """Sycamore-53 m=10 batch over 4 open wires (16 bitstrings) x 2^6 slices: sampled runs
    s_(sigma, y) against the oracle, c64 on the tensor-core path."""
    circ, bits = workload("C2")
    ow = [3, 17, 30, 52]
    net = jet.Network.from_circuit(circ, bits, open_wires=ow)
    plan = jet.Plan.greedy(net, seed=1, trials=128, n_sliced=6, bytes_weight=5.0)
    n = plan.cost()["n_sl"] * 16
    amps, vals, ex = run_batch(jet, plan, "c64", [(0, n)])
    sample = [0, 1, 15, 16, 17, 500, n - 1]
    ref = contract.batch_run_values(circ, bits, ow, plan.ssa_path, plan.sliced_labels, sample)
    for r, want in zip(sample, ref):
        assert abs(vals[r] - want) <= 1e-4 * abs(want)
    # amplitudes are the per-bitstring sums of the runs (canonical order, complex128)
    for y in range(16):
        assert abs(amps[y] - sum(vals[y::16])) <= 1e-12 * abs(amps[y])
    # prefix cache: nodes off the bra-attached subtrees are shared across the 16 bitstrings
    assert ex.stats()["flop_executed"] == plan.prefix_flop(0, n) < plan.cost()["e_flsl"]
