"""oracle.dense -- TEST INFRASTRUCTURE ONLY: FCT1 by explicitly materialised matrices (tiny n).

Pi1 = 4 B C H~ (Sec. 3.1), with the north_star Rademacher D on the
right.  H_s is built by the paper's recursion H_n = [[H, H], [H, -H]], H_2 = [[1,1],[1,-1]]
(P:L2273-2281), normalised by 1/sqrt(s) -- a different construction from the
popcount formula used by oracle.c, so the two pin each other.
"""
from __future__ import annotations

import numpy as np


def hadamard_recursive(s: int) -> np.ndarray:
    """Unnormalised Sylvester Hadamard matrix by the recursion of P:L2273-2281."""
    assert s >= 1 and (s & (s - 1)) == 0
    H = np.ones((1, 1))
    while H.shape[0] < s:
        H = np.block([[H, H], [H, -H]])
    return H


def G_block(s: int) -> np.ndarray:
    """G_s = [H_s; I_s] (2s x s), H_s normalised."""
    return np.vstack([hadamard_recursive(s) / np.sqrt(s), np.eye(s)])


def H_tilde(n_pad: int, s: int) -> np.ndarray:
    """Block-diagonal H~ (2n' x n') of n'/s copies of G_s."""
    return np.kron(np.eye(n_pad // s), G_block(s))


def materialise(n: int, signs, cauchy, hash_rows, s: int, r1: int):
    """Return dense (B, C, H~, D) for an n-row problem zero-padded to n' = s*ceil(n/s)."""
    n_pad = -(-n // s) * s
    D = np.diag(np.concatenate([np.asarray(signs[:n], np.float64), np.ones(n_pad - n)]))
    C = np.diag(np.asarray(cauchy[: 2 * n_pad], np.float64))
    B = np.zeros((r1, 2 * n_pad))
    B[np.asarray(hash_rows[: 2 * n_pad]), np.arange(2 * n_pad)] = 1.0   # one e_h per column
    return B, C, H_tilde(n_pad, s), D


def dense_sketch(A: np.ndarray, signs, cauchy, hash_rows, s: int, r1: int) -> np.ndarray:
    """Y = 4 B C H~ D A_pad with every factor materialised (n <= a few hundred)."""
    A = np.asarray(A, np.float64)
    n = A.shape[0]
    B, C, Ht, D = materialise(n, signs, cauchy, hash_rows, s, r1)
    A_pad = np.vstack([A, np.zeros((D.shape[0] - n, A.shape[1]))])
    return 4.0 * (B @ (C @ (Ht @ (D @ A_pad))))


def dense_magnitude_bound(A: np.ndarray, signs, cauchy, hash_rows, s: int, r1: int) -> np.ndarray:
    """north_star's entrywise tolerance yardstick 4 |B| |C| |H~| |D| |A_pad|, every factor materialised and
    replaced by its entrywise absolute value before the products (the same matrices as dense_sketch)."""
    A = np.asarray(A, np.float64)
    n = A.shape[0]
    B, C, Ht, D = materialise(n, signs, cauchy, hash_rows, s, r1)
    A_pad = np.vstack([A, np.zeros((D.shape[0] - n, A.shape[1]))])
    return 4.0 * (np.abs(B) @ (np.abs(C) @ (np.abs(Ht) @ (np.abs(D) @ np.abs(A_pad)))))
