"""Synthetic Sycamore-style random quantum circuits (readings A1-A5).

The paper uses Arute et al.'s circuit files for Sycamore-53 (PAPER.md l.217,
l.267: "the only two qubit gate is fSim"); those are not available, so this is a
seeded generator of the same structure:

  * layout: the 54-qubit Sycamore grid, rows of 2,4,6,8,9,9,7,5,3,1 qubits on
    GridQubit coordinates (row r, col c); couplers join (r,c)-(r+1,c) and
    (r,c)-(r,c+1).  Sycamore-53 removes qubit (0,5) (reading A1).
  * coupler patterns: A = vertical, (r+c) even; B = vertical, (r+c) odd;
    C = horizontal, (r+c) even; D = horizontal, (r+c) odd -- each a matching.
    Cycle k uses pattern "ABCDCDAB"[k % 8].
  * cycle = one 1-qubit layer on every qubit (sqrt X/Y/W, uniformly random,
    never the same gate twice in a row on a qubit), then fSim(pi/2, pi/6) on
    the cycle's pattern; after m cycles one final 1-qubit layer (A2-A4).
  * wires are the qubits sorted by (r, c); wire 0 is the most significant digit.
"""

import math

from .circuit import Circuit
from .gates import SYC_1Q, SYC_1Q_NAMES, fsim
from .rng import SplitMix64

SYCAMORE_ROWS = {0: (5, 6), 1: (4, 7), 2: (3, 8), 3: (2, 9), 4: (1, 9),
                 5: (0, 8), 6: (1, 7), 7: (2, 6), 8: (3, 5), 9: (4, 4)}
REMOVED_53 = (0, 5)
PATTERN_SEQ = "ABCDCDAB"
FSIM_THETA = math.pi / 2
FSIM_PHI = math.pi / 6


def sycamore_qubits(n_qubits: int = 53):
    qs = [(r, c) for r in range(10) for c in range(SYCAMORE_ROWS[r][0], SYCAMORE_ROWS[r][1] + 1)]
    assert len(qs) == 54
    if n_qubits == 53:
        qs.remove(REMOVED_53)
    else:
        assert n_qubits == 54
    return sorted(qs)


def grid_qubits(rows: int, cols: int):
    return [(r, c) for r in range(rows) for c in range(cols)]


def coupler_patterns(qubits):
    """Return dict pattern -> list of (q_a, q_b) wire pairs (q_a < q_b)."""
    idx = {q: i for i, q in enumerate(qubits)}
    pats = {"A": [], "B": [], "C": [], "D": []}
    for (r, c) in qubits:
        if (r + 1, c) in idx:
            pats["A" if (r + c) % 2 == 0 else "B"].append((idx[(r, c)], idx[(r + 1, c)]))
        if (r, c + 1) in idx:
            pats["C" if (r + c) % 2 == 0 else "D"].append((idx[(r, c)], idx[(r, c + 1)]))
    for p in pats.values():
        used = [w for pair in p for w in pair]
        assert len(used) == len(set(used)), "pattern is not a matching"
    return pats


def random_circuit(qubits, m: int, seed: int, theta: float = FSIM_THETA,
                   phi: float = FSIM_PHI, name: str = "rqc") -> Circuit:
    n = len(qubits)
    pats = coupler_patterns(qubits)
    rng = SplitMix64(seed)
    circ = Circuit(n, 2, meta={"kind": "sycamore", "name": name, "m": m, "seed": seed,
                               "qubits": list(qubits)})
    last = [-1] * n
    u2 = fsim(theta, phi)

    def one_qubit_layer():
        for w in range(n):
            if last[w] < 0:
                g = rng.randint(3)
            else:
                g = (last[w] + 1 + rng.randint(2)) % 3
            last[w] = g
            circ.add((w,), SYC_1Q[g], SYC_1Q_NAMES[g])

    for k in range(m):
        one_qubit_layer()
        for (a, b) in pats[PATTERN_SEQ[k % len(PATTERN_SEQ)]]:
            circ.add((a, b), u2, "fSim")
    one_qubit_layer()
    return circ


def sycamore53(m: int, seed: int = 1) -> Circuit:
    return random_circuit(sycamore_qubits(53), m, seed, name=f"syc53_m{m}")


def grid_rqc(rows: int, cols: int, m: int, seed: int = 1) -> Circuit:
    return random_circuit(grid_qubits(rows, cols), m, seed, name=f"grid{rows}x{cols}_m{m}")
