"""Seeded synthetic input generators shared by the oracle and the product path.

Holds no tensor-network arithmetic (no network build, no contraction, no slicing):
only circuits (gate matrices + wires) and output digits, drawn from splitmix64.
"""

from .circuit import Circuit, Gate, random_bitstring
from .gbs import generate_gbs
from .rng import SplitMix64
from .sycamore import grid_rqc, random_circuit, sycamore53, sycamore_qubits, grid_qubits

__all__ = ["Circuit", "Gate", "random_bitstring", "generate_gbs", "SplitMix64",
           "grid_rqc", "random_circuit", "sycamore53", "sycamore_qubits", "grid_qubits",
           "workload"]


def workload(name: str, seed: int = 1):
    """The BASELINE.json configs as (circuit, bitstring) pairs."""
    if name == "C1":
        c = grid_rqc(3, 3, 8, seed)
    elif name == "C2":
        c = sycamore53(10, seed)
    elif name == "C3":
        c = sycamore53(14, seed)
    elif name == "C5":
        c = sycamore53(20, seed)
    elif name == "C4":
        c = generate_gbs(3, 4, 1, 0.5, 4, seed)
    elif name == "G88d4":     # GBS-88-m1 (2-D 8x8 modes, one cycle), cutoff 4
        c = generate_gbs(2, 8, 1, 0.5, 4, seed)
    elif name == "G88d8":     # the same circuit at cutoff 8 (qudits of 3 address bits)
        c = generate_gbs(2, 8, 1, 0.5, 8, seed)
    else:
        raise ValueError(name)
    bs = seed
    bits = random_bitstring(c.n_wires, c.d, bs)
    if name in ("C4", "G88d4", "G88d8"):
        # reading A19b: a GBS output with an odd total photon number has amplitude exactly 0
        # (P8: the squeezers emit photon pairs, the beam splitters conserve photon number), so
        # the bitstring seed is advanced until the digit sum is even
        while sum(bits) % 2:
            bs += 1
            bits = random_bitstring(c.n_wires, c.d, bs)
    return c, bits
