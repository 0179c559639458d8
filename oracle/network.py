"""Circuit -> closed tensor network (Sec. II.B.1 "Example Circuit").

Follows the paper's mapping: "the initial state is the product of rank-one
tensors |0>_a |0>_d" (l.81); a one-qudit gate is a rank-2 tensor S_ba with b the
output and a the input index; a two-qudit gate is a rank-4 tensor B_cfbe with
outputs (c, f) then inputs (b, e) (l.81, reading A7); "to compute the amplitude
of |a_1 a_2> we attach the rank-1 <a_1|_c and <a_2|_f tensors" (l.83).

Id conventions (shared *by definition* with the C ABI):
  tensors: 0..n-1 = kets of wires 0..n-1; n+g = gate g; n+G+w = bra of wire w.
  labels:  0..n-1 = the wire labels entering the circuit (ket legs); then each
           gate g, in order, creates one new label per wire in gates[g].wires order.
"""

import numpy as np


class Network:
    def __init__(self):
        self.tensors = []   # list of np.ndarray (complex128), one axis per label
        self.labels = []    # list of tuple of label ids
        self.dims = {}      # label -> dimension

    @property
    def n_tensors(self):
        return len(self.tensors)

    def carriers(self):
        car = {}
        for t, ls in enumerate(self.labels):
            for l in ls:
                car.setdefault(l, []).append(t)
        return car


def build_network(circuit, bitstring):
    """Closed network whose full contraction is <x|U|0...0> (Eq. naive_summation)."""
    n, d = circuit.n_wires, circuit.d
    net = Network()
    cur = list(range(n))            # current open label of each wire
    next_label = n
    for w in range(n):              # |0>_w, rank 1
        ket = np.zeros(d, dtype=np.complex128)
        ket[0] = 1.0
        net.tensors.append(ket)
        net.labels.append((w,))
        net.dims[w] = d
    for g in circuit.gates:
        k = len(g.wires)
        outs = []
        for w in g.wires:
            outs.append(next_label)
            net.dims[next_label] = d
            next_label += 1
        ins = [cur[w] for w in g.wires]
        # U[out][in] with wires[0] most significant -> axes (out_0..out_{k-1}, in_0..in_{k-1})
        t = np.asarray(g.u, dtype=np.complex128).reshape((d,) * (2 * k))
        net.tensors.append(t)
        net.labels.append(tuple(outs) + tuple(ins))
        for w, o in zip(g.wires, outs):
            cur[w] = o
    assert len(bitstring) == n
    for w in range(n):              # <x_w|, rank 1
        xw = int(bitstring[w])
        assert 0 <= xw < d
        bra = np.zeros(d, dtype=np.complex128)
        bra[xw] = 1.0
        net.tensors.append(bra)
        net.labels.append((cur[w],))
    validate_closed(net)
    return net


def validate_closed(net):
    """Every label on exactly two tensors with agreeing dimension (closed network)."""
    for l, ts in net.carriers().items():
        if len(ts) != 2:
            raise ValueError(f"label {l} carried by {len(ts)} tensors")
    for t, ls in zip(net.tensors, net.labels):
        if t.shape != tuple(net.dims[l] for l in ls):
            raise ValueError("tensor shape does not match its labels")
