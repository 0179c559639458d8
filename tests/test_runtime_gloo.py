"""Multi-rank host logic on CPU (gloo, world size 2): slice sharding and the single
all-reduce.  The per-rank partial sums come from the oracle, so this checks the
partition + reduction, not the kernels."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2107_09793_b200.runtime import host_shard_sum, shard_range


def test_shard_range_disjoint_cover():
    for n in (1, 2, 7, 64, 1024, 4096):
        for g in (1, 2, 3, 4, 8):
            got = []
            for r in range(g):
                b, e = shard_range(n, r, g)
                assert 0 <= b <= e <= n
                got.extend(range(b, e))
            assert got == list(range(n))
    # d^k slices over d^j ranks: rank block = slices whose outer j digits equal the rank
    b, e = shard_range(1024, 3, 8)
    assert (b, e) == (384, 512) and all((s >> 7) == 3 for s in range(b, e))
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from circuits import workload
    from oracle import contract
    from oracle.network import build_network
    from oracle.path import greedy_path
    from paper_2107_09793_b200.runtime import allreduce_amplitude

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    circ, bits = workload("C1")
    net = build_network(circ, bits)
    p = greedy_path(net)
    sliced = sorted(net.dims)[20:24]
    n = 2 ** len(sliced)
    b, e = shard_range(n, rank, world)
    vals = contract.slice_values(net, p, sliced, indices=range(b, e))
    part = 0j
    for v in vals:
        part += v
    acc = torch.tensor([part.real, part.imag], dtype=torch.float64)
    allreduce_amplitude(acc)
    out[rank] = (complex(acc[0].item(), acc[1].item()), [complex(v) for v in vals])
    dist.destroy_process_group()


def test_gloo_two_ranks_single_allreduce():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    from circuits import workload
    from oracle import contract
    from oracle.network import build_network
    from oracle.path import greedy_path

    circ, bits = workload("C1")
    net = build_network(circ, bits)
    full = contract.amplitude(net, greedy_path(net))
    tot, _ = host_shard_sum([out[r][1] for r in range(world)])
    for r in range(world):
        assert abs(out[r][0] - full) < 1e-12          # every rank holds the reduced amplitude
    assert abs(tot - full) < 1e-12


def _plan_worker(rank, world, port, out):
    import torch.distributed as dist

    import __graft_entry__
    from circuits import workload
    from paper_2107_09793_b200 import jet
    from paper_2107_09793_b200.runtime import plan_shared

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    __graft_entry__.build() if rank == 0 else None
    dist.barrier()
    circ, bits = workload("C2")
    net = jet.Network.from_circuit(circ, bits)
    calls = []

    def make():
        calls.append(1)
        return jet.Plan.greedy(net, seed=3, trials=32, n_sliced=6, slice_objective=1), {"who": rank}

    plan, info = plan_shared(net, make)
    out[rank] = (list(plan.ssa_path), list(plan.sliced_labels), plan.cost()["prefix"], len(calls), info["who"])
    dist.destroy_process_group()


def test_gloo_plan_once_broadcast():
    """Rank 0 plans, rank 1 rebuilds the identical plan from the broadcast path + sliced labels."""
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_plan_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0][3] == 1 and out[1][3] == 0          # only rank 0 ran the planner
    assert out[0][:3] == out[1][:3]                   # same path, slices and executed FLOP
    assert out[1][4] == 0
