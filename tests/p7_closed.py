"""P7 closed form: with fSim(0, 0) = I every two-qubit gate is the identity, so the
closed network factorises into 53 one-qubit chains and each slice value is a product of
chain values:

    s_sigma = prod_q <x_q| V_q,last ... P_a ... V_q,1 |0>

where P_a = |a><a| is inserted wherever sigma fixes a wire segment of qubit q (a sliced label).
Labels follow the id convention of PAPER.md l.72-85 / DESIGN.md "ids": labels 0..n-1 are the
ket legs, then every gate creates one new label per wire in its `wires` order.  Independent of
the oracle and of the product (plain 2-vectors), so it pins the GPU path at full size.
"""

import numpy as np


def slice_closed_form(circ, bits, sliced_labels, index, absolute=False):
    """s_sigma of the P7 circuit; absolute=True evaluates the same chains with |U| entries (and
    real |.| vectors): the sum of the magnitudes of every product term of s_sigma, the scale of the
    forward rounding error of any summation order (reading A13d)."""
    n, d = circ.n_wires, circ.d
    digits = {}
    rem = index
    for l in reversed(list(sliced_labels)):
        rem, digits[l] = divmod(rem, d)
    v = [np.eye(d, dtype=np.complex128)[0] for _ in range(n)]

    def project(q, label):
        if label in digits:
            p = np.zeros(d, dtype=np.complex128)
            p[digits[label]] = v[q][digits[label]]
            v[q] = p

    for q in range(n):
        project(q, q)
    nxt = n
    for g in circ.gates:
        if len(g.wires) == 1:
            q = g.wires[0]
            v[q] = (np.abs(g.u) @ np.abs(v[q])) if absolute else (g.u @ v[q])
            project(q, nxt)
            nxt += 1
        else:
            if not np.array_equal(g.u, np.eye(d ** len(g.wires))):
                raise ValueError("P7 needs identity two-qubit gates")
            for q in g.wires:
                project(q, nxt)
                nxt += 1
    out = 1 + 0j
    for q in range(n):
        out *= abs(v[q][bits[q]]) if absolute else v[q][bits[q]]
    return out.real if absolute else out
