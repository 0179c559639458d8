"""P8 closed forms of GBS amplitudes (SURVEY.md 8c, P:310-312 hafnian context), independent of
any tensor network: beam splitters preserve the vacuum and map the single-photon subspace by
the M x M matrix W; after S(r) on every mode, <0|U|0> = cosh(r)^(-M/2), odd photon numbers give
0, and with B = tanh(r) W W^T: <1_i 1_j|U|0> = pref * B_ij, <2_i|U|0> = pref * B_ii / sqrt(2).
Exact under Fock truncation when the total photon number is <= d - 1."""

import math

import numpy as np


def single_photon_matrix(circ):
    """W[j][i] = <1_j|U|1_i>, the product of the BS single-photon blocks (l.219-246)."""
    m, d = circ.n_wires, circ.d
    W = np.eye(m, dtype=np.complex128)
    for g in circ.gates:
        if len(g.wires) != 2:
            continue
        a, b = g.wires
        blk = np.array([[g.u[d * 1 + 0, d * 1 + 0], g.u[d * 1 + 0, d * 0 + 1]],
                        [g.u[d * 0 + 1, d * 1 + 0], g.u[d * 0 + 1, d * 0 + 1]]])
        e = np.eye(m, dtype=np.complex128)
        e[np.ix_([a, b], [a, b])] = blk
        W = e @ W
    return W


def p8_cases(circ, r, max_pairs=None, seed=0):
    """(bitstring, exact amplitude) pairs: vacuum, two-photon outputs, odd photon numbers."""
    M = circ.n_wires
    pref = math.cosh(r) ** (-M / 2)
    B = math.tanh(r) * single_photon_matrix(circ) @ single_photon_matrix(circ).T
    pairs = [(i, j) for i in range(M) for j in range(i, M)]
    if max_pairs is not None and len(pairs) > max_pairs:
        rng = np.random.default_rng(seed)
        pairs = [pairs[t] for t in sorted(rng.choice(len(pairs), max_pairs, replace=False))]
    cases = [([0] * M, pref)]
    for i, j in pairs:
        x = [0] * M
        if i == j:
            x[i] = 2
            cases.append((x, pref * B[i, i] / math.sqrt(2)))
        else:
            x[i] = x[j] = 1
            cases.append((x, pref * B[i, j]))
    x = [0] * M
    x[0] = 1
    cases.append((x, 0.0))
    x = [0] * M
    x[-1] = 3
    cases.append((x, 0.0))
    return cases
