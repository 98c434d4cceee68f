"""Pins for oracle.fct2 (NEXT-3: the FCT2 sketch Pi1 = (8/r1) sqrt(pi t/(2s)) C H~, Sec. 3.2).

Each pin fixes the oracle against something other than itself: the library Sylvester Hadamard, the orthogonality
of G when s = t, a dense assembly of Pi1 from scipy's Hadamard and np.kron, the exact expectation
E||G x||^2 = ||x||^2 of the SRHT, the 1-stability of C (exact Cauchy law of every entry of Y), linearity over
t-aligned shards, and the lower distortion side of Thm FCT2 on small problems.
"""
import math

import numpy as np
import pytest
from scipy import linalg, stats

import fctgen
from oracle import fct2 as F


def test_params_reading():
    # s = r1 = ceil(2 d ln d), t = 2 d^2 rounded up to a power of two (reading of P:L1447-1449)
    want = {8: (34, 128, 34), 16: (89, 512, 89), 32: (222, 2048, 222), 64: (533, 8192, 533), 100: (922, 32768, 922)}
    for d, v in want.items():
        assert F.params(d) == v


@pytest.mark.parametrize("t", [1, 2, 4, 8, 64, 256])
def test_hadamard_is_sylvester(t):
    np.testing.assert_array_equal(F.hadamard(t), linalg.hadamard(t))


@pytest.mark.parametrize("t", [2048, 4096])
def test_kronecker_apply_matches_explicit(t):
    """The large-t path (H_{2^a} kron H_{2^b}) equals the explicit Sylvester matrix (scipy)."""
    X = np.random.default_rng(t).standard_normal((t, 3))
    np.testing.assert_allclose(F.hadamard_apply(X), linalg.hadamard(t) @ X, rtol=1e-12, atol=1e-9)


def test_s_equals_t_is_orthogonal():
    """R = identity (s = t): G = H_t/sqrt(t) D_t is orthogonal, so every column keeps its 2-norm per block."""
    rng = np.random.default_rng(0)
    t, n, d = 64, 3 * 64 + 17, 5
    A = rng.standard_normal((n, d))
    sg = rng.choice([-1, 1], t).astype(np.int8)
    Z = F.srht(A, sg, np.arange(t), t, t)
    Ap = np.zeros((3 * t + t, d))
    Ap[:n] = A
    for b in range(4):
        np.testing.assert_allclose(np.linalg.norm(Z[b * t:(b + 1) * t], axis=0),
                                   np.linalg.norm(Ap[b * t:(b + 1) * t], axis=0), rtol=1e-12)


def test_dense_assembly():
    """Pi1 assembled as a dense matrix from scipy's Hadamard, a selection matrix and np.kron equals the oracle."""
    t, s, r1, d = 16, 5, 7, 3
    n = 3 * t - 4
    inp = fctgen.fct2_inputs(9, n, t, s, r1)
    A = np.random.default_rng(1).standard_normal((n, d))
    Rsel = np.eye(t)[inp.sel]
    G = math.sqrt(t / s) * Rsel @ (linalg.hadamard(t) / math.sqrt(t)) @ np.diag(inp.signs_t.astype(float))
    nb = 3
    Ht = np.kron(np.eye(nb), G)
    Pi1 = (8.0 / r1) * math.sqrt(math.pi * t / (2 * s)) * inp.C.astype(np.float64) @ Ht
    Ap = np.zeros((nb * t, d))
    Ap[:n] = A
    Y, Mb = F.sketch(A, inp.signs_t, inp.sel, inp.C, t, s, r1)
    np.testing.assert_allclose(Y, Pi1 @ Ap, rtol=1e-12, atol=1e-12 * np.abs(Y).max())
    assert (np.abs(Y) <= Mb * (1 + 1e-12)).all()


def test_srht_norm_expectation():
    """E_R ||G x||_2^2 = ||x||_2^2 for R uniform over s-subsets (the SRHT's isometry in expectation)."""
    rng = np.random.default_rng(2)
    t, s = 64, 9
    x = rng.standard_normal((t, 1))
    sg = rng.choice([-1, 1], t).astype(np.int8)
    vals = np.array([float((F.srht(x, sg, np.sort(rng.choice(t, s, replace=False)), t, s) ** 2).sum())
                     for _ in range(3000)])
    se = vals.std() / math.sqrt(len(vals))
    assert abs(vals.mean() - float((x ** 2).sum())) < 4 * se


def test_cauchy_one_stability():
    """For fixed A (one column) and G, every Y_k / kappa = sum_i C_ki Z_i is Cauchy with scale sum_i |Z_i|
    (P:L1186-1189): KS test over independent draws of C."""
    rng = np.random.default_rng(3)
    t, s, r1 = 32, 6, 4
    n = 4 * t
    A = rng.standard_normal((n, 1))
    sg = rng.choice([-1, 1], t).astype(np.int8)
    sel = np.sort(rng.choice(t, s, replace=False))
    Z = F.srht(A, sg, sel, t, s)[:, 0]
    gam = np.abs(Z).sum()
    k = F.scale(t, s, r1)
    draws = []
    for _ in range(1500):
        C = rng.standard_cauchy((r1, Z.size))
        draws.append(F.sketch(A, sg, sel, C, t, s, r1, with_bound=False)[:, 0] / (k * gam))
    p = stats.kstest(np.concatenate(draws), "cauchy").pvalue
    assert p > 1e-3


def test_shard_additivity():
    t, s, r1, d = 32, 7, 11, 4
    n = 5 * t
    inp = fctgen.fct2_inputs(4, n, t, s, r1)
    A = np.random.default_rng(5).standard_normal((n, d))
    Y = F.sketch(A, inp.signs_t, inp.sel, inp.C, t, s, r1, with_bound=False)
    Y2 = (F.sketch(A[:2 * t], inp.signs_t, inp.sel, inp.C[:, :2 * s], t, s, r1, with_bound=False)
          + F.sketch(A[2 * t:], inp.signs_t, inp.sel, inp.C[:, 2 * s:], t, s, r1, with_bound=False))
    np.testing.assert_allclose(Y, Y2, rtol=1e-12, atol=1e-12 * np.abs(Y).max())


def test_lower_distortion_side():
    """Thm FCT2 lower side ||Ax||_1 <= ||Pi1 A x||_1: the constant (8/r1) sqrt(pi t/2s) makes
    it hold for nearly all x on small problems with the paper's parameters (empirical gate, like FCT1's)."""
    rng = np.random.default_rng(6)
    d = 6
    s, t, r1 = F.params(d)
    n = 64 * t
    ok = 0
    total = 0
    for seed in range(3):
        inp = fctgen.fct2_inputs(20 + seed, n, t, s, r1)
        A = rng.standard_normal((n, d))
        Y = F.sketch(A, inp.signs_t, inp.sel, inp.C, t, s, r1, with_bound=False)
        X = rng.standard_normal((d, 300))
        ok += int((np.abs(A @ X).sum(axis=0) <= np.abs(Y @ X).sum(axis=0)).sum())
        total += X.shape[1]
    assert ok >= 0.95 * total
