"""Pins for oracle.lad (NEXT-2: coreset l1 regression, FastCauchyRegression steps 6-8).

Each pin fixes the LP oracle against something other than itself: the weighted median (the p = 1 case of
l1 regression), brute-force enumeration of interpolating vertices, exact fits, equivariance, and the
subgradient optimality condition of the l1 objective.
"""
import itertools
import math

import numpy as np
import pytest

from oracle import lad as L


def _wmedian_objective(b, w):
    """Textbook weighted median of b with weights w and sum_i w_i |b_i - med| (sorted cumulative weights)."""
    o = np.argsort(b, kind="stable")
    bs, ws = b[o], w[o]
    c = np.cumsum(ws)
    med = bs[np.searchsorted(c, 0.5 * c[-1])]
    return med, math.fsum((w * np.abs(b - med)).tolist())


@pytest.mark.parametrize("seed", range(4))
def test_p1_is_weighted_median(seed):
    """min_x sum_i w_i |b_i - x| (rows Z_i = w_i [1, -b_i]) is attained at the weighted median."""
    rng = np.random.default_rng(seed)
    m = 101 + 17 * seed
    b = rng.standard_cauchy(m)
    w = rng.uniform(1.0, 50.0, m)
    Z = np.stack([w, -w * b], axis=1)
    x, f = L.lad(Z)
    med, fmed = _wmedian_objective(b, w)
    assert f == pytest.approx(fmed, rel=1e-12)
    assert x[0] == pytest.approx(med, rel=1e-9, abs=1e-12)


def _brute_force(Z):
    """An l1 optimum interpolates p rows (A of full column rank): min over all p-subsets of the
    objective at the solution of the square system (P:L2178-2188's LP has a vertex optimum)."""
    m, q = Z.shape
    p = q - 1
    best = math.inf
    for S in itertools.combinations(range(m), p):
        M = Z[list(S), :p]
        if abs(np.linalg.det(M)) < 1e-12:
            continue
        x = np.linalg.solve(M, -Z[list(S), p])
        best = min(best, L.objective(Z, x))
    return best


@pytest.mark.parametrize("m,p,seed", [(7, 1, 0), (8, 2, 1), (9, 3, 2), (9, 2, 3), (6, 3, 4)])
def test_brute_force_vertices(m, p, seed):
    rng = np.random.default_rng(seed)
    Z = rng.standard_normal((m, p + 1)) * rng.uniform(0.5, 3.0, (m, 1))
    _, f = L.lad(Z)
    assert f == pytest.approx(_brute_force(Z), rel=1e-10)


def test_exact_fit_recovers_x():
    rng = np.random.default_rng(5)
    A = rng.standard_normal((200, 6))
    xs = rng.standard_normal(6)
    w = rng.uniform(1, 4, 200)
    Z = w[:, None] * np.concatenate([A, -(A @ xs)[:, None]], axis=1)
    x, f = L.lad(Z)
    assert f < 1e-9
    np.testing.assert_allclose(x, xs, rtol=1e-8, atol=1e-9)


def test_equivariance():
    """b -> c b + A z  gives  x -> c x + z and f -> |c| f (the objective only sees A x - b)."""
    rng = np.random.default_rng(6)
    m, p = 300, 4
    A = rng.standard_normal((m, p))
    b = A @ rng.standard_normal(p) + rng.standard_cauchy(m)
    x0, f0 = L.lad(np.concatenate([A, -b[:, None]], axis=1))
    z, c = rng.standard_normal(p), -2.5
    x1, f1 = L.lad(np.concatenate([A, -(c * b + A @ z)[:, None]], axis=1))
    assert f1 == pytest.approx(abs(c) * f0, rel=1e-10)
    np.testing.assert_allclose(x1, c * x0 + z, rtol=1e-7, atol=1e-8)


@pytest.mark.parametrize("seed", range(3))
def test_subgradient_certificate(seed):
    """x is optimal iff 0 is in sum_{r_i != 0} sign(r_i) a_i + sum_{r_i = 0} [-1, 1] a_i.  With continuous
    data the optimum has exactly p zero residuals: solve for their multipliers and check |xi| <= 1."""
    rng = np.random.default_rng(10 + seed)
    m, p = 1500, 5
    A = rng.standard_normal((m, p)) * rng.uniform(0.2, 5, (m, 1))
    b = A @ rng.standard_normal(p) + 0.1 * rng.standard_normal(m)
    out = rng.random(m) < 0.05
    b[out] += 100 * rng.standard_cauchy(int(out.sum()))
    Z = np.concatenate([A, -b[:, None]], axis=1)
    x, f = L.lad(Z)
    r = A @ x - b
    scale = np.abs(A).sum(axis=1) * (np.abs(x).max() + 1) + np.abs(b)
    zero = np.abs(r) <= 1e-9 * scale
    assert zero.sum() == p
    g = (np.sign(r[~zero])[:, None] * A[~zero]).sum(axis=0)
    xi = np.linalg.solve(A[zero].T, -g)
    assert np.all(np.abs(xi) <= 1 + 1e-9)
    # a perturbation in any direction does not decrease the objective
    for _ in range(20):
        dx = 1e-4 * rng.standard_normal(p)
        assert L.objective(Z, x + dx) >= f - 1e-9 * f


def test_coreset_rows_scaling():
    rng = np.random.default_rng(7)
    X = rng.standard_normal((50, 4)).astype(np.float32)
    idx = np.array([103, 110, 149], dtype=np.int64)
    w = np.array([1.0, 2.5, 1e3])
    Z = L.coreset_rows(X, idx, w, row_base=100)
    np.testing.assert_array_equal(Z, w[:, None] * X[[3, 10, 49]].astype(np.float64))
    # ||D(Ax - b)||_1 == sum_j w_j |A_j x - b_j| for X = [A, -b]
    x = rng.standard_normal(3)
    A, b = X[[3, 10, 49], :3].astype(np.float64), -X[[3, 10, 49], 3].astype(np.float64)
    assert L.objective(Z, x) == pytest.approx(float((w * np.abs(A @ x - b)).sum()), rel=1e-14)
