"""FLOP counters of the sliced contraction (oracle).

Convention (reading A11): one pairwise step costs
8 * prod(dims of the distinct labels of both operands) real FLOP, on the
sigma-restricted network (sliced labels are fixed, so they do not count).

  FLOP_sl   = sum of step costs of one slice
  E-flsl    = N_sl * FLOP_sl                                   (Eq. sliced_flops)
  f_sl      = FLOP of nodes whose subtree carries no sliced label / FLOP_sl
  E-fltask  = f_sl FLOP_sl + N_sl (1 - f_sl) FLOP_sl           (Eq. task_based_amplitude_flops)
  exact     = sum_v flop_v * prod_{l in S(v)} d_l               (dedup by task name, reading A9)
  prefix    = executed FLOP of a slice loop over [begin, end) with one cached
              copy per node: at each slice, recompute every node v whose
              max position of S(v) in the loop order is >= the highest
              changed digit (reading A10).
S(v) = the sliced labels carried by the leaves under v ("sliced or the
result of a contraction involving a sliced tensor").
"""

import itertools


def tree_info(net, ssa_path, sliced_labels):
    """Per step: (flop, S(v) as frozenset).  Integers only."""
    sl = set(sliced_labels)
    labs = {t: [l for l in net.labels[t] if l not in sl] for t in range(net.n_tensors)}
    ss = {t: frozenset(l for l in net.labels[t] if l in sl) for t in range(net.n_tensors)}
    nid = net.n_tensors
    steps = []
    for (i, j) in ssa_path:
        la, lb = labs.pop(i), labs.pop(j)
        union = set(la) | set(lb)
        flop = 8
        for l in union:
            flop *= net.dims[l]
        out = [l for l in la if l not in lb] + [l for l in lb if l not in la]
        labs[nid] = out
        ss[nid] = ss.pop(i) | ss.pop(j)
        steps.append((flop, ss[nid]))
        nid += 1
    return steps


def cost_report(net, ssa_path, sliced_labels):
    steps = tree_info(net, ssa_path, sliced_labels)
    n_sl = 1
    for l in sliced_labels:
        n_sl *= net.dims[l]
    flop_sl = sum(f for f, _ in steps)
    shared = sum(f for f, s in steps if not s)
    exact = 0
    for f, s in steps:
        m = 1
        for l in s:
            m *= net.dims[l]
        exact += f * m
    return {
        "n_sl": n_sl,
        "flop_sl": flop_sl,
        "flop_shared": shared,
        "e_flsl": n_sl * flop_sl,
        "e_fltask": shared + n_sl * (flop_sl - shared),
        "exact_reuse": exact,
        "prefix": prefix_flop(net, ssa_path, sliced_labels, 0, n_sl),
    }


def prefix_flop(net, ssa_path, sliced_labels, begin, end):
    """Executed FLOP of the one-copy prefix cache over slices [begin, end)."""
    steps = tree_info(net, ssa_path, sliced_labels)
    pos = {l: p for p, l in enumerate(sliced_labels)}
    maxpos = [max((pos[l] for l in s), default=-1) for _, s in steps]
    dims = [net.dims[l] for l in sliced_labels]
    total = 0
    prev = None
    for idx, digits in enumerate(itertools.product(*[range(d) for d in dims])):
        if idx < begin:
            continue
        if idx >= end:
            break
        if prev is None:
            j = -1                       # first slice of the range: everything
        else:
            j = next(p for p in range(len(dims)) if digits[p] != prev[p])
        total += sum(f for f, mp in zip((f for f, _ in steps), maxpos) if mp >= j)
        prev = digits
    return total
