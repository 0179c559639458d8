"""f3 memory report (fig. m10_memory): peak memory with and without deletion of
intermediates and the extra memory shared work costs, checked against an independent recomputation
from the compiled launch plan (host only)."""

import pytest

from circuits import workload


@pytest.fixture(scope="module")
def jet():
    import __graft_entry__

    __graft_entry__.build()
    from paper_2107_09793_b200 import jet as j

    return j


def align(x):
    return (x + 255) // 256 * 256


def recompute(plan, dtype):
    """Peak of live intermediates over the execution order, from describe_exec: a node output lives
    from its own position to its parent's; prefix-cache entries (parent recomputed more often,
    maxpos(parent) > maxpos(v)) and the root live for the whole run."""
    d = plan.describe_exec(dtype)
    es = 8 if dtype == "c64" else 16
    nodes = d["nodes"]
    by_v = {n["v"]: n for n in nodes}
    n_pos = len(nodes)
    live = [0] * n_pos
    live_ns = [0] * n_pos
    no_del = cache = 0
    for n in nodes:
        size = align(n["n_out"] * es)
        no_del += size
        par = by_v.get(n["parent"])
        persistent = par is None or par["maxpos"] > n["maxpos"]
        if par is not None and par["maxpos"] > n["maxpos"]:
            cache += size
        lo, hi = (0, n_pos - 1) if persistent else (n["pos"], par["pos"])
        for q in range(lo, hi + 1):
            live[q] += size
        lo, hi = (0, n_pos - 1) if par is None else (n["pos"], par["pos"])
        for q in range(lo, hi + 1):
            live_ns[q] += size
    return max(live), max(live_ns), no_del, cache, d


@pytest.mark.parametrize("name,k,dtype", [("C1", 0, "c128"), ("C1", 3, "c64"), ("C2", 6, "c64"), ("C2", 0, "c64")])
def test_memory_report_matches_recomputation(jet, name, k, dtype):
    circ, bits = workload(name)
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=1, trials=32, n_sliced=k)
    m = plan.memory(dtype)
    peak, peak_ns, no_del, cache, d = recompute(plan, dtype)
    assert m["total_bytes"] == plan.workspace_bytes(dtype) == d["total_bytes"]
    assert m["peak_live_bytes"] == peak
    assert m["peak_live_noshare_bytes"] == peak_ns
    assert m["no_deletion_bytes"] == no_del
    assert m["cache_bytes"] == cache
    assert m["arena_bytes"] == d["inter_bytes"]
    assert peak_ns <= peak <= m["arena_bytes"] <= no_del
    assert m["leaf_bytes"] + m["arena_bytes"] + m["scratch_bytes"] <= m["total_bytes"]
    if k == 0:
        assert cache == 0 and peak == peak_ns


def test_memory_deletion_and_shared_work_shape(jet):
    """The qualitative findings of fig. m10_memory on the synthetic m=10 circuit: deleting
    intermediates saves a large factor; the sliced run with shared work needs more memory than the
    sliced run without it (the cached intermediates), and slicing shrinks the peak."""
    circ, bits = workload("C2")
    net = jet.Network.from_circuit(circ, bits)
    sl = jet.Plan.greedy(net, seed=1, trials=64, n_sliced=6).memory("c64")
    full = jet.Plan.greedy(net, seed=1, trials=64, n_sliced=0).memory("c64")
    assert sl["no_deletion_bytes"] >= 5 * sl["peak_live_bytes"]
    assert full["no_deletion_bytes"] >= 5 * full["peak_live_bytes"]
    assert sl["cache_bytes"] > 0 and sl["peak_live_bytes"] > sl["peak_live_noshare_bytes"]
    assert sl["peak_live_bytes"] < full["peak_live_bytes"]


def test_concurrent_slice_subsets(jet):
    circ, bits = workload("C2")
    net = jet.Network.from_circuit(circ, bits)
    plan = jet.Plan.greedy(net, seed=1, trials=32, n_sliced=6)
    m = plan.memory("c64")
    per = m["total_bytes"] - m["leaf_bytes"]
    for budget in (m["total_bytes"] - 1, m["total_bytes"], m["total_bytes"] + 3 * per, 180 * 10**9):
        n = plan.concurrent_slices(budget, "c64")
        assert m["leaf_bytes"] + n * per <= budget < m["leaf_bytes"] + (n + 1) * per
