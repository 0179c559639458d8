"""Dense state-vector brute force (independent pin, not the paper's method).

psi = |0...0> in C^{d^n}; apply each gate matrix U[out][in] in circuit order to
its wires (wires[0] most significant digit of U's index); amplitude(x) =
psi[x] with x[0] (wire 0) the most significant digit (reading A6).  Shares no
code with oracle.contract.
"""

import numpy as np


def final_state(circuit, max_wires=None):
    n, d = circuit.n_wires, circuit.d
    if d ** n > (1 << 24):
        raise ValueError("state too large")
    psi = np.zeros((d,) * n, dtype=np.complex128)
    psi[(0,) * n] = 1.0
    for g in circuit.gates:
        k = len(g.wires)
        u = np.asarray(g.u).reshape((d,) * (2 * k))
        # contract U's input axes (k..2k-1) with psi's wire axes, then move outputs back
        psi = np.tensordot(u, psi, axes=(list(range(k, 2 * k)), list(g.wires)))
        # result axes: U outputs (k of them) then the remaining wires in order
        rest = [w for w in range(n) if w not in g.wires]
        order = list(g.wires) + rest
        inv = np.argsort(order)
        psi = np.transpose(psi, inv)
    return psi


def amplitude(circuit, bitstring):
    return complex(final_state(circuit)[tuple(int(x) for x in bitstring)])
