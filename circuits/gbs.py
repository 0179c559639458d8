"""Alg. 1 of the paper: random n-dimensional GBS circuit.

Reading A16/A17: loops exactly as written (1-based in the paper, 0-based wires
here): llens[l] = width^(l-1); S(r) on every mode; then for each cycle, each
l = 1..dim, each i = 1..modes-llens[l]: draw theta then phi uniformly in
[0, 2 pi) and apply BS(theta, phi) on modes (i, i + llens[l]).
"""

import math

from .circuit import Circuit
from .gates import beamsplitter, squeezer
from .rng import SplitMix64


def generate_gbs(dim: int, width: int, cycles: int, r: float, d: int, seed: int) -> Circuit:
    modes = width ** dim
    llens = [width ** (i - 1) for i in range(1, dim + 1)]
    rng = SplitMix64(seed)
    circ = Circuit(modes, d, meta={"kind": "gbs", "dim": dim, "width": width, "cycles": cycles,
                                   "r": r, "d": d, "seed": seed,
                                   "name": f"gbs{width}^{dim}_m{cycles}_d{d}"})
    s = squeezer(r, d)
    for k in range(1, modes + 1):
        circ.add((k - 1,), s, "S")
    for _c in range(1, cycles + 1):
        for l in range(1, dim + 1):
            for i in range(1, modes - llens[l - 1] + 1):
                theta = 2.0 * math.pi * rng.uniform()
                phi = 2.0 * math.pi * rng.uniform()
                circ.add((i - 1, i - 1 + llens[l - 1]), beamsplitter(theta, phi, d), "BS")
    return circ
