"""oracle.fct2 -- TEST INFRASTRUCTURE ONLY: the fp64 CPU oracle of NEXT-3, the FCT2 sketch (Sec. 3.2).

    Pi1 = (8 / r1) sqrt(pi t / (2 s)) * C * H~
    H~  = blockdiag(G, ..., G), n/t blocks, G the s x t FJLT      (the SAME G in every block)
    C   = r1 x (n s / t) i.i.d. standard Cauchy

G is the paper's FJLT implementation, the SRHT, in its standard form
    G = sqrt(t / s) * R * (H_t / sqrt(t)) * D_t
D_t: t Rademacher signs; H_t: Sylvester Hadamard, H[r][l] = (-1)^popcount(r & l); R: s of the t rows
(indices `sel`, distinct).  n is zero-padded to a multiple of t (as FCT1's Q7).  Parameters (reading of the
garbled P:L1447-1449): s = ceil(2 d ln d), t = 2 d^2 rounded up to a power of two, r1 = ceil(2 d ln d).

Written as the definition: explicit Hadamard matrix (no FWHT), one block at a time, then a dense matrix
product with C (numpy, fp64).  Pinned in tests/test_oracle_fct2.py.  Shares no code with paper_1207_4684_b200.
"""
from __future__ import annotations

import math

import numpy as np


def params(d: int):
    """(s, t, r1) of PAPER.md P:L1447-1449 for FCT2 (reading: s = r1 = ceil(2 d ln d), t = 2 d^2 -> power of 2)."""
    s = max(1, math.ceil(2 * d * math.log(d))) if d > 1 else 1
    t = 1 << max(1, math.ceil(math.log2(2 * d * d)))
    return min(s, t), t, s


def hadamard(t: int) -> np.ndarray:
    """Sylvester Hadamard of order t (unnormalised), H[r][l] = (-1)^popcount(r & l)."""
    r = np.arange(t)
    pc = np.vectorize(lambda v: bin(v).count("1"))(r[:, None] & r[None, :])
    return np.where(pc % 2 == 0, 1.0, -1.0)


def hadamard_apply(X: np.ndarray) -> np.ndarray:
    """H_t X (unnormalised, X: t x d).  t <= 1024: the explicit matrix; larger t: the Sylvester identity
    H_{2^(a+b)} = H_{2^a} kron H_{2^b} (popcount(r & l) splits over the high and low index bits), i.e.
    H_t X = H_{2^a} [X reshaped 2^a x 2^b x d] H_{2^b}^T, with both factors explicit."""
    t = X.shape[0]
    if t <= 1024:
        return hadamard(t) @ X
    a = (t.bit_length() - 1) // 2
    ta, tb = 1 << a, t >> a
    Y1 = (hadamard(ta) @ X.reshape(ta, -1)).reshape(ta, tb, -1)     # high index bits
    return np.matmul(hadamard(tb), Y1).reshape(t, -1)                  # low index bits


def scale(t: int, s: int, r1: int) -> float:
    """(8 / r1) sqrt(pi t / (2 s))."""
    return 8.0 / r1 * math.sqrt(math.pi * t / (2.0 * s))


def srht(A: np.ndarray, signs_t: np.ndarray, sel: np.ndarray, t: int, s: int) -> np.ndarray:
    """Z = H~ A: block b of t rows (zero-padded) -> s rows  sqrt(t/s) * (H_t / sqrt t) (D_t A_b) [sel]."""
    A = np.asarray(A, dtype=np.float64)
    n, d = A.shape
    nb = -(-n // t)
    D = np.asarray(signs_t, dtype=np.float64)
    Z = np.zeros((nb * s, d))
    for b in range(nb):
        Ab = np.zeros((t, d))
        rows = A[b * t:(b + 1) * t]
        Ab[:rows.shape[0]] = rows
        Z[b * s:(b + 1) * s] = math.sqrt(t / s) / math.sqrt(t) * hadamard_apply(D[:, None] * Ab)[np.asarray(sel)]
    return Z


def sketch(A: np.ndarray, signs_t: np.ndarray, sel: np.ndarray, C: np.ndarray, t: int, s: int, r1: int,
           with_bound: bool = True):
    """Y = Pi1 A (r1 x d, fp64) and the entrywise magnitude bound Mbound = kappa |C| |H~| |A| (|H~| with the
    absolute values of G's entries, sqrt(t/s) / sqrt(t) = 1 / sqrt(s) each)."""
    Z = srht(A, signs_t, sel, t, s)
    C = np.asarray(C, dtype=np.float64)
    assert C.shape == (r1, Z.shape[0])
    k = scale(t, s, r1)
    Y = k * (C @ Z)
    if not with_bound:
        return Y
    A = np.abs(np.asarray(A, dtype=np.float64))
    n, d = A.shape
    nb = -(-n // t)
    Zb = np.zeros_like(Z)
    for b in range(nb):
        colsum = A[b * t:(b + 1) * t].sum(axis=0) / math.sqrt(s)    # |G| |A_b| rows: all equal
        Zb[b * s:(b + 1) * s] = colsum[None, :]
    return Y, k * (np.abs(C) @ Zb)
