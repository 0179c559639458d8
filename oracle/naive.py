"""Naive full summation (Eq. naive_summation).

<a|U|0> = sum over every joint assignment of every index of the product of all
tensor entries.  Exponential: refuses networks with more than 2^22 joint
assignments.
"""

import itertools

import numpy as np


def full_sum(net, max_states=1 << 22):
    labels = sorted(net.dims)
    total = 1
    for l in labels:
        total *= net.dims[l]
    if total > max_states:
        raise ValueError(f"network too large for exhaustive sum ({total} assignments)")
    acc = 0j
    for vals in itertools.product(*[range(net.dims[l]) for l in labels]):
        v = dict(zip(labels, vals))
        p = 1 + 0j
        for t, ls in zip(net.tensors, net.labels):
            p *= t[tuple(v[l] for l in ls)]
            if p == 0:
                break
        acc += p
    return complex(acc)
