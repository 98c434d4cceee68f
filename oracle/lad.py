"""oracle.lad -- TEST INFRASTRUCTURE ONLY: the fp64 CPU oracle of NEXT-2, the coreset l1 regression.

FastCauchyRegression steps 6-8 (Thm P:L2955-2980): with X = [A, -b]
 and the diagonal sampling matrix D (idx, weight from the sampler),
build DA, Db and return x_hat = argmin_x ||D(Ax - b)||_1.

Written as the plain definition:
  coreset_rows  Z_j = weight_j * X[idx_j]   (fp64: (double)weight * (double)X, one rounding)
                so that Z_j . [x; 1] = weight_j * (A_j x - b_j)
  lad           min_x sum_j |Z_j . [x; 1]| as the textbook LP
                    min 1'u + 1'v  s.t.  Z[:, :p] x + u - v = -Z[:, p],  u, v >= 0
                solved through its dual (p equality rows) by a library LP solver (scipy HiGHS dual
                simplex, a library primitive); x from the dual's multipliers, strong duality checked.
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
    """argmin_x sum_j |Z_j . [x; 1]| via LP duality; returns (x, f) with f = objective(Z, x).

    The l1 regression  min_x ||At x - bt||_1  (At = Z[:, :p], bt = -Z[:, p]) is the LP
    min 1'u + 1'v s.t. At x + u - v = bt, u, v >= 0, whose dual is  max bt'y s.t. At'y = 0, -1 <= y <= 1.
    The dual has p equality rows, so the library LP solver (HiGHS dual simplex) is fast on it; x is the
    multiplier of At'y = 0: with V(c) = min {-bt'y : At'y = c, |y| <= 1} = -min_x (||At x - bt||_1 + c'x),
    dV/dc = -x*, i.e. x = -(eqlin marginals).  Strong duality f(x) = bt'y* is checked on every call.
    """
    from scipy.optimize import linprog

    Z = np.asarray(Z, dtype=np.float64)
    m, q = Z.shape
    p = q - 1
    if m == 0 or p == 0:
        x = np.zeros(p)
        return x, objective(Z, x) if m else 0.0
    bt = -Z[:, p]
    res = linprog(-bt, A_eq=Z[:, :p].T, b_eq=np.zeros(p), bounds=(-1, 1), method="highs-ds",
                  options={"primal_feasibility_tolerance": 1e-10, "dual_feasibility_tolerance": 1e-10})
    if res.status != 0:
        raise RuntimeError(f"oracle.lad: LP failed: {res.message}")
    x = -np.asarray(res.eqlin.marginals, dtype=np.float64)
    f = objective(Z, x)
    if not abs(f - (-res.fun)) <= 1e-9 * max(f, 1e-300) + 1e-12 * math.fsum(np.abs(bt).tolist()):
        raise RuntimeError(f"oracle.lad: strong duality check failed: f(x) = {f!r}, dual = {-res.fun!r}")
    return x, f


def coreset_regression(X: np.ndarray, idx: np.ndarray, weight: np.ndarray, row_base: int = 0):
    """x_hat = argmin ||D(Ax - b)||_1 for X = [A, -b]; returns (x_hat, f_coreset, Z)."""
    Z = coreset_rows(X, idx, weight, row_base)
    x, f = lad(Z)
    return x, f, Z
