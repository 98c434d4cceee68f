"""oracle.lad -- TEST INFRASTRUCTURE ONLY: the fp64 CPU oracle of NEXT-2, the coreset l1 regression.

FastCauchyRegression steps 6-8 (Thm P:L2955-2980): with X = [A, -b]
 and the diagonal sampling matrix D (idx, weight from the sampler),
build DA, Db and return x_hat = argmin_x ||D(Ax - b)||_1.

Written as the plain definition:
  coreset_rows  Z_j = weight_j * X[idx_j]   (fp64: (double)weight * (double)X, one rounding)
                so that Z_j . [x; 1] = weight_j * (A_j x - b_j)
  lad           min_x sum_j |Z_j . [x; 1]| as the textbook LP
                    min 1'u + 1'v  s.t.  Z[:, :p] x + u - v = -Z[:, p],  u, v >= 0
                solved by a library LP solver (scipy HiGHS dual simplex, a library primitive).
  objective     sum_j |Z_j . [x; 1]| in fp64 (math.fsum, exactly rounded sum).
Pinned in tests/test_oracle_lad.py by the weighted median (p = 1), brute-force vertex enumeration
(an l1 optimum interpolates p rows), exact fits, equivariance and a subgradient optimality certificate.
Shares no code with paper_1207_4684_b200.
"""
from __future__ import annotations

import math

import numpy as np


def coreset_rows(X: np.ndarray, idx: np.ndarray, weight: np.ndarray, row_base: int = 0) -> np.ndarray:
    """Z = D X restricted to the sampled rows: Z_j = weight_j * X[idx_j - row_base] (fp64)."""
    X = np.asarray(X)
    rows = np.asarray(idx, dtype=np.int64) - int(row_base)
    return np.asarray(weight, dtype=np.float64)[:, None] * X[rows].astype(np.float64)


def objective(Z: np.ndarray, x: np.ndarray) -> float:
    """sum_j |Z_j . [x; 1]|  (residual per row in fp64, exactly rounded sum)."""
    Z = np.asarray(Z, dtype=np.float64)
    r = Z[:, :-1] @ np.asarray(x, dtype=np.float64) + Z[:, -1]
    return math.fsum(np.abs(r).tolist())


def lad(Z: np.ndarray):
    """argmin_x sum_j |Z_j . [x; 1]| via the LP; returns (x, f) with f = objective(Z, x)."""
    import scipy.sparse as sp
    from scipy.optimize import linprog

    Z = np.asarray(Z, dtype=np.float64)
    m, q = Z.shape
    p = q - 1
    if m == 0 or p == 0:
        x = np.zeros(p)
        return x, objective(Z, x) if m else 0.0
    Aeq = sp.hstack([sp.csr_matrix(Z[:, :p]), sp.identity(m, format="csr"), -sp.identity(m, format="csr")],
                    format="csr")
    c = np.concatenate([np.zeros(p), np.ones(2 * m)])
    bounds = [(None, None)] * p + [(0, None)] * (2 * m)
    res = linprog(c, A_eq=Aeq, b_eq=-Z[:, p], bounds=bounds, method="highs-ds",
                  options={"primal_feasibility_tolerance": 1e-10, "dual_feasibility_tolerance": 1e-10})
    if res.status != 0:
        raise RuntimeError(f"oracle.lad: LP failed: {res.message}")
    x = np.asarray(res.x[:p], dtype=np.float64)
    return x, objective(Z, x)


def coreset_regression(X: np.ndarray, idx: np.ndarray, weight: np.ndarray, row_base: int = 0):
    """x_hat = argmin ||D(Ax - b)||_1 for X = [A, -b]; returns (x_hat, f_coreset, Z)."""
    Z = coreset_rows(X, idx, weight, row_base)
    x, f = lad(Z)
    return x, f, Z
