"""Pairwise contraction along an SSA path, with slicing (oracle).

PAPER.md l.92-105 (Eq. sequence): contract two tensors at a time, summing over
the labels they share; the result carries the remaining labels.  Output label
order: free labels of A in A's order, then free labels of B in B's order
(SPEC.md l.53).  PAPER.md l.116-133 (Eq. sliced_sum): slicing fixes a shared
index to each of its values; each assignment sigma gives a partial sum s_sigma
and <x|U|0> = sum_sigma s_sigma.  Slice assignments are enumerated
lexicographically with sliced_labels[0] most significant (reading A12) and
summed in that canonical order in complex128.

The "sum over shared labels" step uses numpy.tensordot as the library
primitive (a matmul); ``contract_pair_loops`` is the same definition written as
nested loops, used by the tests to pin ``contract_pair`` on small operands.
"""

import itertools

import numpy as np


def contract_pair(a, la, b, lb):
    """C = sum over labels shared by (a, la) and (b, lb); returns (C, lc)."""
    shared = [l for l in la if l in lb]
    ia = [la.index(l) for l in shared]
    ib = [lb.index(l) for l in shared]
    for x, y in zip(ia, ib):
        if a.shape[x] != b.shape[y]:
            raise ValueError("shared label with mismatched dimension")
    c = np.tensordot(a, b, axes=(ia, ib))
    lc = tuple(l for l in la if l not in shared) + tuple(l for l in lb if l not in shared)
    return c, lc


def contract_pair_loops(a, la, b, lb):
    """Same definition as contract_pair, as explicit nested loops (small inputs only)."""
    shared = [l for l in la if l in lb]
    fa = [l for l in la if l not in shared]
    fb = [l for l in lb if l not in shared]
    dim = {}
    for l, s in zip(la, a.shape):
        dim[l] = s
    for l, s in zip(lb, b.shape):
        dim[l] = s
    lc = tuple(fa) + tuple(fb)
    c = np.zeros(tuple(dim[l] for l in lc), dtype=np.complex128)
    for out in itertools.product(*[range(dim[l]) for l in lc]):
        val = dict(zip(lc, out))
        acc = 0j
        for sh in itertools.product(*[range(dim[l]) for l in shared]):
            val.update(zip(shared, sh))
            acc += a[tuple(val[l] for l in la)] * b[tuple(val[l] for l in lb)]
        c[out] = acc
    return c, lc


def validate_path(n_tensors, ssa_path):
    """SSA path: step s consumes two live ids and creates id n_tensors + s; ends in one tensor."""
    live = set(range(n_tensors))
    for s, (i, j) in enumerate(ssa_path):
        if i == j or i not in live or j not in live:
            raise ValueError(f"step {s}: ids ({i},{j}) not both live")
        live.discard(i)
        live.discard(j)
        live.add(n_tensors + s)
    if len(live) != 1:
        raise ValueError(f"path leaves {len(live)} tensors")


def validate_slices(net, sliced_labels):
    car = net.carriers()
    for l in sliced_labels:
        if len(car.get(l, [])) != 2:
            raise ValueError(f"sliced label {l} is not a bond")
    if len(set(sliced_labels)) != len(sliced_labels):
        raise ValueError("duplicate sliced label")


def restrict(t, lt, assignment):
    """Leaf restricted at sigma: drop each sliced axis by fixing its value (l.120)."""
    idx = []
    keep = []
    for l in lt:
        if l in assignment:
            idx.append(assignment[l])
        else:
            idx.append(slice(None))
            keep.append(l)
    return t[tuple(idx)], tuple(keep)


def contract_along(net, ssa_path, assignment=None):
    """Scalar obtained by contracting the (sigma-restricted) network along ssa_path."""
    assignment = assignment or {}
    vals = {}
    labs = {}
    for t in range(net.n_tensors):
        vals[t], labs[t] = restrict(net.tensors[t], net.labels[t], assignment)
    nid = net.n_tensors
    for (i, j) in ssa_path:
        vals[nid], labs[nid] = contract_pair(vals.pop(i), labs.pop(i), vals.pop(j), labs.pop(j))
        nid += 1
    (root,) = vals.keys()
    if labs[root]:
        raise ValueError("network is not closed")
    return complex(vals[root])


def slice_assignments(net, sliced_labels):
    """Lexicographic enumeration, sliced_labels[0] most significant (reading A12)."""
    dims = [net.dims[l] for l in sliced_labels]
    for digits in itertools.product(*[range(dd) for dd in dims]):
        yield dict(zip(sliced_labels, digits))


def slice_assignment(net, sliced_labels, index):
    """The index-th assignment of slice_assignments (mixed radix, sliced_labels[0] most
    significant), without enumerating the ones before it (N_sl reaches 2^36 at C4)."""
    n = 1
    for l in sliced_labels:
        n *= net.dims[l]
    if not 0 <= index < n:
        raise ValueError(f"slice index {index} out of range [0, {n})")
    digits = {}
    for l in reversed(list(sliced_labels)):
        index, digits[l] = divmod(index, net.dims[l])
    return {l: digits[l] for l in sliced_labels}


def slice_values(net, ssa_path, sliced_labels, indices=None):
    """s_sigma for each slice index (all, or the given subset), in canonical order."""
    validate_path(net.n_tensors, ssa_path)
    validate_slices(net, sliced_labels)
    if indices is None:
        return [contract_along(net, ssa_path, sig) for sig in slice_assignments(net, sliced_labels)]
    return [contract_along(net, ssa_path, slice_assignment(net, sliced_labels, i)) for i in indices]


def amplitude(net, ssa_path, sliced_labels=()):
    """<x|U|0> = sum_sigma s_sigma (Eq. sliced_sum 3), plain double summation in order."""
    vals = slice_values(net, ssa_path, list(sliced_labels))
    acc = 0j
    for v in vals:
        acc += v
    return acc


def batch_bitstrings(bitstring, open_wires, d):
    """The bitstrings of a batch of amplitudes: bitstring with the digits of open_wires
    enumerated lexicographically, open_wires[0] most significant (reading A23)."""
    out = []
    for digits in itertools.product(range(d), repeat=len(open_wires)):
        x = [int(v) for v in bitstring]
        for w, v in zip(open_wires, digits):
            x[w] = v
        out.append(x)
    return out


def batch_run_values(circuit, bitstring, open_wires, ssa_path, sliced_labels, runs):
    """Batch of amplitudes as a multi-contraction ("computing batches of
    amplitudes"): run r = sigma * n_batch + y is s_sigma of the amplitude of the y-th batch
    bitstring, each a plain closed network contracted along the same SSA path (the tensor
    ids do not depend on the bra digits, so one path serves every bitstring)."""
    from .network import build_network

    xs = batch_bitstrings(bitstring, open_wires, circuit.d)
    nb = len(xs)
    nets = {}
    out = []
    for r in runs:
        sig, y = divmod(int(r), nb)
        if y not in nets:
            nets[y] = build_network(circuit, xs[y])
        out.append(slice_values(nets[y], ssa_path, list(sliced_labels), [sig])[0])
    return out


def batch_amplitudes(circuit, bitstring, open_wires, ssa_path, sliced_labels=()):
    """Every amplitude of the batch, y-indexed: Eq. sliced_sum per bitstring."""
    from .network import build_network

    return [amplitude(build_network(circuit, x), ssa_path, sliced_labels)
            for x in batch_bitstrings(bitstring, open_wires, circuit.d)]
