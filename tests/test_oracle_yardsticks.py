"""Pins for the oracle's tolerance yardsticks (round-2 VERDICT item 1).

Every GPU parity bound is a multiple of one of these magnitude bounds, so each is pinned here against
a source other than the formula that computes it:
  * FCT1 Mbound = 4 |B||C||H~||D||A| (north_star) == the product of the materialised, entrywise-|.|
    factors (oracle.dense.dense_magnitude_bound), for every s in 1..64, several r1, ragged n;
  * the row-norm bounds max_j sum_l |A_il||M_lj| and sum_j sum_l |A_il||Rinv_lj| == exactly rounded
    (math.fsum) brute force;
  * FCT2 Mbound = kappa |C||H~||A| == the materialised |C| |kron(I, G)| |A|, with G built from the
    explicit Hadamard matrix, selection and signs;
  * FCT2's kappa (8/r1) sqrt(pi t/2s) == the constant the paper's proof assembles (P:L816-827:
    4/r1 from the Cauchy embedding times (2/c3) sqrt(t/s) with c3 = sqrt(2/pi)), and its
    sqrt(pi t/2s) factor == the exact expectation identity E[sqrt(pi t/2s) ||G z||_1] -> ||z||_1 for
    flat z (E|sum of t Rademachers| in closed form).
Each pin fails under the corresponding mutation of the oracle (1/sqrt(s) dropped, a bound scaled).
"""
import math

import numpy as np
import pytest
import scipy.linalg

import fctgen
import oracle
from oracle import dense
from oracle import fct2 as F


def _inputs(n, d, s, r1, seed):
    rng = np.random.default_rng(seed)
    n_pad = -(-n // s) * s
    A = (rng.standard_normal((n, d)) * rng.choice([1.0, 1e3], (n, 1), p=[0.9, 0.1])).astype(np.float32)
    sg = rng.choice(np.array([-1, 1], np.int8), n_pad)
    c = rng.standard_cauchy(2 * n_pad).astype(np.float32)
    h = rng.integers(0, r1, 2 * n_pad).astype(np.int32)
    return A, sg, c, h


@pytest.mark.parametrize("s", [1, 2, 4, 8, 16, 32, 64])
@pytest.mark.parametrize("r1", [1, 5, 16])
@pytest.mark.parametrize("n_extra", [0, 3])
def test_fct1_mbound_equals_materialised_abs_product(s, r1, n_extra):
    n = 3 * s + n_extra if s > 1 else 9 + n_extra
    d = 3
    A, sg, c, h = _inputs(n, d, s, r1, seed=7 * s + r1 + 1000 * n_extra)
    _, Mb = oracle.sketch(A, sg, c, h, s, r1)
    want = dense.dense_magnitude_bound(A, sg, c, h, s, r1)
    np.testing.assert_allclose(Mb, want, rtol=1e-12, atol=0)


def test_fct1_mbound_hadamard_half_scaling():
    """One block, one nonzero input row, identity half routed to its own bucket: the Hadamard-half bucket
    holds exactly 4|c| |a| / sqrt(s) (|H_s| entries are 1/sqrt(s))."""
    for s in (4, 64, 1024):
        A = np.zeros((s, 1), np.float32)
        A[s // 3, 0] = -3.0
        sg = np.ones(s, np.int8)
        c = np.full(2 * s, 0.5, np.float32)
        h = np.zeros(2 * s, np.int32)
        h[s:] = 1                                     # identity half -> bucket 1, Hadamard half -> bucket 0
        _, Mb = oracle.sketch(A, sg, c, h, s, 2)
        assert Mb[1, 0] == pytest.approx(4 * 0.5 * 3.0, rel=1e-15)
        assert Mb[0, 0] == pytest.approx(s * 4 * 0.5 * 3.0 / math.sqrt(s), rel=1e-13)


def test_rownorm_bound_fsum_brute_force():
    rng = np.random.default_rng(21)
    n, d, k = 40, 7, 5
    A = rng.standard_normal((n, d)).astype(np.float32)
    Rinv = np.triu(rng.standard_normal((d, d))) + 2 * np.eye(d)
    Pi2 = rng.standard_cauchy((d, k)).astype(np.float32)
    _, _, bnd = oracle.rownorm(A, Rinv, Pi2, with_bound=True)
    M = [[math.fsum(Rinv[l, m] * float(Pi2[m, j]) for m in range(d)) for j in range(k)] for l in range(d)]
    for i in range(n):
        want = max(math.fsum(abs(float(A[i, l])) * abs(M[l][j]) for l in range(d)) for j in range(k))
        assert bnd[i] == pytest.approx(want, rel=1e-13)


def test_rownorm_exact_bound_fsum_brute_force():
    rng = np.random.default_rng(22)
    n, d = 40, 9
    A = rng.standard_normal((n, d)).astype(np.float32)
    Rinv = np.triu(rng.standard_normal((d, d))) + 2 * np.eye(d)
    _, _, bnd = oracle.rownorm_exact(A, Rinv, with_bound=True)
    for i in range(n):
        want = math.fsum(abs(float(A[i, l])) * abs(Rinv[l, j]) for j in range(d) for l in range(d))
        assert bnd[i] == pytest.approx(want, rel=1e-14)


def _G_explicit(signs_t, sel, t, s):
    """G = sqrt(t/s) R (H_t / sqrt t) D_t, materialised from scipy's Hadamard matrix."""
    H = scipy.linalg.hadamard(t).astype(np.float64)
    return math.sqrt(t / s) / math.sqrt(t) * H[np.asarray(sel)] * np.asarray(signs_t, np.float64)[None, :]


@pytest.mark.parametrize("t,s,r1,nb", [(16, 5, 3, 3), (64, 9, 7, 2), (128, 128, 4, 2), (32, 1, 2, 4)])
def test_fct2_mbound_equals_materialised_abs_product(t, s, r1, nb):
    d = 3
    n = nb * t - 5
    inp = fctgen.fct2_inputs(9, n, t, s, r1)
    A = np.random.default_rng(t + s).standard_normal((n, d))
    _, Mb = F.sketch(A, inp.signs_t, inp.sel, inp.C, t, s, r1)
    G = _G_explicit(inp.signs_t, inp.sel, t, s)
    Ht = np.kron(np.eye(nb), np.abs(G))
    Ap = np.zeros((nb * t, d))
    Ap[:n] = np.abs(A)
    kappa = 4.0 / r1 * (2.0 / math.sqrt(2.0 / math.pi)) * math.sqrt(t / s)
    np.testing.assert_allclose(Mb, kappa * (np.abs(inp.C.astype(np.float64)) @ (Ht @ Ap)), rtol=1e-12, atol=0)


@pytest.mark.parametrize("t,s,r1", [(8192, 533, 533), (128, 20, 7), (2, 1, 1)])
def test_fct2_kappa_is_the_constant_the_proof_assembles(t, s, r1):
    """Appendix FCT2: (4/r1)||C H~ A x||_1 lower-bounds ||H~Ax||_1 (Thm sw) and
    ||H~ y||_1 >= (1/2) c3 sqrt(s/t) ||y||_1 (eq. Hlower); multiplying by (2/c3) sqrt(t/s) with
    c3 = sqrt(2/pi) gives Pi1's scale.  Independent of the printed formula at P:L2363."""
    c3 = math.sqrt(2.0 / math.pi)
    assert F.scale(t, s, r1) == pytest.approx((4.0 / r1) * (2.0 / c3) * math.sqrt(t / s), rel=1e-14)


def test_fct2_sqrt_pi_t_over_2s_flat_vector_expectation():
    """For flat z (all ones) and random D_t, (G z)_r = s^(-1/2) sum_l H[sel_r, l] D_l is a sum of t
    Rademachers / sqrt(s), so E ||G z||_1 = s E|S_t| / sqrt(s) with E|S_t| = t C(t-1, floor((t-1)/2)) / 2^(t-1)
    exactly; sqrt(pi t / 2s) is the factor that maps it to ||z||_1 = t as t grows (c3 = E|N(0,1)|).
    Checks the sqrt(pi t/2s) part of F.scale against a Monte-Carlo mean over D_t draws (4 s.e.)."""
    rng = np.random.default_rng(31)
    t, s, r1 = 256, 16, 1
    sel = np.sort(rng.choice(t, s, replace=False))
    e_abs = t * math.comb(t - 1, (t - 1) // 2) / 2.0 ** (t - 1)
    want = math.sqrt(s) * e_abs                    # E ||G z||_1
    # D_t 1 = the sign vector itself: one srht call over 4000 sign-vector columns with D = I
    Dcols = rng.choice([-1.0, 1.0], (t, 4000))
    vals = np.abs(F.srht(Dcols, np.ones(t, np.int8), sel, t, s)).sum(axis=0)
    assert abs(vals.mean() - want) < 4 * vals.std() / math.sqrt(len(vals))
    fjlt_factor = F.scale(t, s, r1) * r1 / 8.0      # sqrt(pi t / 2s)
    assert fjlt_factor * want / t == pytest.approx(1.0, abs=2e-3)   # -> ||z||_1 (Cauchy-Schwarz tight for flat z)
