"""CPU oracle for the Jet hot path -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct complex128 implementation of what the product
path computes, written from the paper (arXiv 2107.09793, PAPER.md).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  It shares no code with
``paper_2107_09793_b200`` (the only common dependency is the seeded input
generator package ``circuits``, which holds no method arithmetic).

Modules and the passages they follow:
  network      circuit -> tensor network + amplitude closure      PAPER.md l.72-85 (Sec. II.B.1)
  contract     pairwise contraction along an SSA path, slicing    l.92-105 (Eq. seq), l.116-133 (Eq. sliced_sum)
  naive        full summation over every index                    l.85-90 (Eq. naive_summation)
  statevector  dense state-vector brute force                     (independent pin, not the method)
  cost         FLOP_amp counters                                  l.140-146 (Eq. sliced_flops), l.205-212 (Eq. task_based)
  path         a plain greedy path for cases with no given path   (plumbing; the paper takes paths as input, l.176)

Pins (tests/test_oracle_*.py, all ``-m "not gpu"``): the worked example with
S=H, B=CZ (P1), state vector (P2), normalisation (P3), slice-sum identity (P4),
path independence (P5), GBS closed forms (P8), gate closed forms (P9),
Alg. 1 counts (P11), FLOP identities (P12).  Parity-unpinned: none of the
functions here; the paper's own m=10 FLOP figures (45.2/97.2 GFLOP) are
context only (path unpublished) and are not used.
"""
