"""Plain circuit container shared by the oracle and the product path (inputs only)."""

from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np


@dataclass
class Gate:
    wires: Tuple[int, ...]          # wires[0] is the most significant digit of U's index
    u: np.ndarray                   # (d^k, d^k) complex128, U[out][in]
    name: str = ""


@dataclass
class Circuit:
    n_wires: int
    d: int
    gates: List[Gate] = field(default_factory=list)
    meta: dict = field(default_factory=dict)

    def add(self, wires, u, name=""):
        wires = tuple(int(w) for w in wires)
        k = len(wires)
        u = np.asarray(u, dtype=np.complex128)
        assert u.shape == (self.d ** k, self.d ** k), (u.shape, self.d, k)
        assert all(0 <= w < self.n_wires for w in wires) and len(set(wires)) == k
        self.gates.append(Gate(wires, u, name))

    def inverse(self) -> "Circuit":
        """U^dagger: gates in reverse order, each conjugate-transposed."""
        c = Circuit(self.n_wires, self.d, meta=dict(self.meta, inverse=True))
        for g in reversed(self.gates):
            c.add(g.wires, g.u.conj().T, g.name + "^dag")
        return c

    def then(self, other: "Circuit") -> "Circuit":
        assert other.n_wires == self.n_wires and other.d == self.d
        c = Circuit(self.n_wires, self.d, meta=dict(self.meta))
        for g in self.gates + other.gates:
            c.add(g.wires, g.u, g.name)
        return c

    @property
    def n_two_qudit(self) -> int:
        return sum(1 for g in self.gates if len(g.wires) == 2)


def random_bitstring(n_wires: int, d: int, seed: int):
    """Output digits x[0..n-1], uniform in [0, d) (A6, A19)."""
    from .rng import SplitMix64

    r = SplitMix64(seed ^ 0xB175_7121_6000_0001)
    return [r.randint(d) for _ in range(n_wires)]
