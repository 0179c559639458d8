"""Counter-based seeded RNG shared by every input generator (reading A21).

splitmix64 with a documented draw order.  This module holds no tensor-network
arithmetic; it exists so that the oracle (``oracle/``) and the product path
(``paper_2107_09793_b200``) receive *identical* synthetic inputs.
"""

MASK64 = (1 << 64) - 1


class SplitMix64:
    """splitmix64: state += golden; mix(state).  uniform() = top 53 bits / 2^53."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        """Uniform double in [0, 1)."""
        return (self.next_u64() >> 11) * (1.0 / (1 << 53))

    def randint(self, n: int) -> int:
        """Integer in [0, n) as floor(uniform * n)."""
        return min(int(self.uniform() * n), n - 1)
