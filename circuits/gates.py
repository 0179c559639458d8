"""Gate matrices for the synthetic workloads (inputs, not method arithmetic).

Conventions (readings A3, A4, A7, A15):
  * every matrix is U[out][in], row-major; for a 2-qudit gate on wires
    (w0, w1) the row/column index is d*digit(w0) + digit(w1) (w0 most significant).
  * Sycamore-style 1-qubit set: sqrt(X), sqrt(Y), sqrt(W), W = (X+Y)/sqrt(2),
    each written exp(-i pi/4 P) = (I - iP)/sqrt(2).
  * fSim(theta, phi) = [[1,0,0,0],[0,c,-is,0],[0,-is,c,0],[0,0,0,e^{-i phi}]].
  * S(r) = exp(r/2 (a^dag^2 - a^2)), exact matrix elements from a working
    cutoff of 96, cropped to d (A15).
  * BS(theta, phi) = exp(theta (e^{i phi} a^dag b - e^{-i phi} a b^dag)), built
    exactly per photon-number block N (the generator conserves N), then cropped
    to in/out states with both occupations < d (A15).
"""

import math

import numpy as np
from scipy.linalg import expm

_X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
_Y = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
_W = (_X + _Y) / math.sqrt(2.0)
_I2 = np.eye(2, dtype=np.complex128)


def _sqrt_pauli(p):
    return (_I2 - 1j * p) / math.sqrt(2.0)


SQRT_X = _sqrt_pauli(_X)
SQRT_Y = _sqrt_pauli(_Y)
SQRT_W = _sqrt_pauli(_W)
SYC_1Q = (SQRT_X, SQRT_Y, SQRT_W)
SYC_1Q_NAMES = ("sqrtX", "sqrtY", "sqrtW")


def fsim(theta: float, phi: float) -> np.ndarray:
    c, s = math.cos(theta), math.sin(theta)
    u = np.zeros((4, 4), dtype=np.complex128)
    u[0, 0] = 1.0
    u[1, 1] = c
    u[1, 2] = -1j * s
    u[2, 1] = -1j * s
    u[2, 2] = c
    u[3, 3] = np.exp(-1j * phi)
    return u


HADAMARD = np.array([[1, 1], [1, -1]], dtype=np.complex128) / math.sqrt(2.0)
CZ = np.diag([1, 1, 1, -1]).astype(np.complex128)

SQUEEZE_WORK_CUTOFF = 96


def squeezer(r: float, d: int, work_cutoff: int = SQUEEZE_WORK_CUTOFF) -> np.ndarray:
    """d x d matrix <m|S(r)|n>, S(r) = exp(r/2 (a^dag^2 - a^2))."""
    n = max(work_cutoff, d)
    a = np.diag(np.sqrt(np.arange(1, n, dtype=np.float64)), 1)  # a|k> = sqrt(k)|k-1>
    ad = a.T
    gen = 0.5 * r * (ad @ ad - a @ a)
    s = expm(gen)
    return s[:d, :d].astype(np.complex128)


def beamsplitter(theta: float, phi: float, d: int) -> np.ndarray:
    """d^2 x d^2 matrix <p q|BS|n m>, row index d*p + q, column d*n + m.

    Built per photon-number block: on span{|k, N-k>} the generator
    theta (e^{i phi} a^dag b - e^{-i phi} a b^dag) is a (N+1)x(N+1) matrix,
    exponentiated exactly (no truncation inside the block).
    """
    u = np.zeros((d * d, d * d), dtype=np.complex128)
    ephi = np.exp(1j * phi)
    for N in range(0, 2 * (d - 1) + 1):
        # basis |k, N-k>, k = 0..N
        g = np.zeros((N + 1, N + 1), dtype=np.complex128)
        for k in range(N + 1):
            # a^dag b |k, N-k> = sqrt(k+1) sqrt(N-k) |k+1, N-k-1>
            if k + 1 <= N:
                g[k + 1, k] += theta * ephi * math.sqrt(k + 1) * math.sqrt(N - k)
            # a b^dag |k, N-k> = sqrt(k) sqrt(N-k+1) |k-1, N-k+1>
            if k >= 1:
                g[k - 1, k] -= theta * np.conj(ephi) * math.sqrt(k) * math.sqrt(N - k + 1)
        blk = expm(g)
        for kin in range(N + 1):
            nin, min_ = kin, N - kin
            if nin >= d or min_ >= d:
                continue
            for kout in range(N + 1):
                p, q = kout, N - kout
                if p >= d or q >= d:
                    continue
                u[d * p + q, d * nin + min_] = blk[kout, kin]
    return u
