"""B200-native hot path of Jet (arXiv 2107.09793): sliced pairwise tensor-network
contraction of random quantum circuits into amplitudes, behind the C ABI in
include/jetb200.h.  ``jet`` is the ctypes binding; ``runtime`` adds the multi-GPU
driver (slice sharding + one NCCL all-reduce)."""

from . import jet  # noqa: F401  (fails loudly if libjetb200.so is missing)
from .jet import Exec, Network, Plan, amplitude, permute, version  # noqa: F401
