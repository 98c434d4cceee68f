"""Pins for oracle O2 (conditioning), O3 (row-norm estimator) and O4 (l1 sampling)."""
import math

import numpy as np
import pytest
from scipy import special, stats

import fctgen
import oracle


# ---------------------------------------------------------------- O2: R from Pi1 A = QR
def test_condition_invariants():
    rng = np.random.default_rng(0)
    Y = rng.standard_normal((256, 12)) * np.logspace(0, 3, 12)
    R, Rinv, _ = oracle.condition(Y)
    assert np.allclose(np.tril(R, -1), 0) and (np.diag(R) > 0).all()
    np.testing.assert_allclose(R.T @ R, Y.T @ Y, rtol=1e-11, atol=1e-11 * np.abs(Y.T @ Y).max())
    Q = Y @ Rinv
    np.testing.assert_allclose(Q.T @ Q, np.eye(12), atol=1e-10)       # orthonormal columns
    np.testing.assert_allclose(R @ Rinv, np.eye(12), atol=1e-10)


# ---------------------------------------------------------------- O3: lambda_i = median_j |Lambda_ij|
def test_rownorm_identity_reduces_to_textbook_median():
    """Rinv = I, Pi2 = I_d (k = d): lambda_i = median_j |A_ij| (numpy.median)."""
    rng = np.random.default_rng(1)
    for d in (5, 8):   # odd and even k
        A = rng.standard_normal((500, d)).astype(np.float32)
        lam, tot = oracle.rownorm(A, np.eye(d), np.eye(d, dtype=np.float32))
        np.testing.assert_allclose(lam, np.median(np.abs(A.astype(np.float64)), axis=1), rtol=1e-15)
        np.testing.assert_allclose(tot, lam.sum(), rtol=1e-12)


def test_rownorm_invariants():
    rng = np.random.default_rng(2)
    n, d, k = 400, 6, 9
    A = rng.standard_normal((n, d)).astype(np.float32)
    A[7] = 0.0
    Rinv = np.triu(rng.standard_normal((d, d))) + 3 * np.eye(d)
    Pi2 = rng.standard_cauchy((d, k)).astype(np.float32)
    lam, tot = oracle.rownorm(A, Rinv, Pi2)
    assert lam[7] == 0.0                                        # zero row -> 0
    lam2, _ = oracle.rownorm(A * np.float32(-4.0), Rinv, Pi2)    # |alpha| homogeneity (exact power of 2)
    np.testing.assert_allclose(lam2, 4.0 * lam, rtol=1e-14)
    p = oracle.probs(lam, tot)
    p2 = oracle.probs(lam2, lam2.sum())
    np.testing.assert_allclose(p, p2, rtol=1e-12)               # p invariant to scaling of A
    # A (R^-1 Pi2) = (A R^-1) Pi2   (associativity used by P:L2170-2171)
    U = A.astype(np.float64) @ Rinv
    want = np.median(np.abs(U @ Pi2.astype(np.float64)), axis=1)
    np.testing.assert_allclose(lam, want, rtol=1e-12, atol=1e-14)


def test_rownorm_brute_force_tiny():
    """Pure-Python loops with math.fsum (exactly rounded sums) and sorted() medians, n <= 64, k <= 7."""
    rng = np.random.default_rng(3)
    for k in (1, 2, 3, 6, 7):
        n, d = 40, 3
        A = rng.standard_normal((n, d)).astype(np.float32)
        Rinv = np.triu(rng.standard_normal((d, d))) + 2 * np.eye(d)
        Pi2 = rng.standard_cauchy((d, k)).astype(np.float32)
        lam, _ = oracle.rownorm(A, Rinv, Pi2)
        M = [[math.fsum(float(Rinv[l, m]) * float(Pi2[m, j]) for m in range(d)) for j in range(k)] for l in range(d)]
        for i in range(n):
            v = sorted(abs(math.fsum(float(A[i, l]) * M[l][j] for l in range(d))) for j in range(k))
            med = v[k // 2] if k % 2 else 0.5 * (v[k // 2 - 1] + v[k // 2])
            assert abs(lam[i] - med) <= 1e-12 * max(med, 1e-300)


@pytest.mark.parametrize("k", [27, 29, 16])
def test_median_of_half_cauchys_distribution(k):
    """For fixed U_(i), lambda_i / ||U_(i)||_1 = median of k i.i.d. half-Cauchys (1-stability,
    Lemma medCauchy).  Odd k = 2h+1: CDF I_{F(x)}(h+1, h+1), F(x) = (2/pi) arctan x.
    KS over 3000 independent draws of Pi2 for one row (Rinv = I)."""
    d = 5
    rng = np.random.default_rng(k)
    a = rng.standard_normal((1, d)).astype(np.float32)
    l1 = float(np.abs(a.astype(np.float64)).sum())
    ratios = np.empty(3000)
    for t in range(ratios.size):
        Pi2 = rng.standard_cauchy((d, k)).astype(np.float32)
        lam, _ = oracle.rownorm(a, np.eye(d), Pi2)
        ratios[t] = lam[0] / l1
    if k % 2:
        h = k // 2
        cdf = lambda x: special.betainc(h + 1, h + 1, (2 / np.pi) * np.arctan(x))
        assert stats.kstest(ratios, cdf).pvalue > 1e-3
        # P[1/2 <= ratio <= 3/2] (the event of Lemma medCauchy), exact vs empirical
        pexact = cdf(1.5) - cdf(0.5)
        pemp = ((ratios >= 0.5) & (ratios <= 1.5)).mean()
        assert abs(pemp - pexact) < 4 * math.sqrt(pexact * (1 - pexact) / ratios.size)
        assert pexact >= 1 - 2 * math.exp(-0.07 * k)           # the lemma's (weak) bound holds
    else:
        # even k: compare with an independent simulation of the half-Cauchy median
        sim = np.median(np.abs(rng.standard_cauchy((20000, k))), axis=1)
        assert stats.ks_2samp(ratios, sim).pvalue > 1e-3


@pytest.mark.parametrize("k", [9, 27])
def test_median_of_half_normals_gaussian_pi2(k):
    """NEXT-1's Gaussian-Pi2 estimator (OptimizedFastCauchyRegression): with Pi2 i.i.d. N(0,1),
    lambda_i / ||U_(i)||_2 is the median of k i.i.d. half-normals (2-stability).  Odd k = 2h+1: exact CDF
    I_{F(x)}(h+1, h+1) with F(x) = erf(x / sqrt 2); KS over 3000 draws of Pi2 for one row (Rinv = I)."""
    d = 6
    rng = np.random.default_rng(100 + k)
    a = rng.standard_normal((1, d)).astype(np.float32)
    l2 = float(np.linalg.norm(a.astype(np.float64)))
    ratios = np.empty(3000)
    for t in range(ratios.size):
        Pi2 = rng.standard_normal((d, k)).astype(np.float32)
        lam, _ = oracle.rownorm(a, np.eye(d), Pi2)
        ratios[t] = lam[0] / l2
    h = k // 2
    cdf = lambda x: special.betainc(h + 1, h + 1, special.erf(x / math.sqrt(2)))
    assert stats.kstest(ratios, cdf).pvalue > 1e-3


# ---------------------------------------------------------------- O4: Bernoulli l1 sampling
def test_sample_extremes_and_weights():
    n = 1000
    p = np.zeros(n, np.float32)
    p[:10] = 1.0                    # m p >= 1 -> phat = 1 -> always in, weight 1
    p[10:20] = 1e-9
    idx, w, cnt = oracle.sample(p, m=5, seed=3)
    assert set(range(10)).issubset(set(idx.tolist()))
    assert not set(range(20, n)) & set(idx.tolist())         # p = 0 -> never in
    assert (np.diff(idx) > 0).all()
    np.testing.assert_array_equal(w[idx < 10], 1.0)
    # weights are 1/phat with phat = min(1, m p) in fp64 from the fp32 p
    for i, wi in zip(idx, w):
        assert wi == 1.0 / min(1.0, 5 * float(p[i]))
    # an undefined probability (NaN) is never sampled, even with explicit uniforms of 0 (R31); +inf is
    # p_hat = 1
    p2 = np.full(64, np.nan, np.float32)
    p2[5] = np.inf
    idx2, w2, cnt2 = oracle.sample(p2, m=5, seed=3, u=np.zeros(64))
    assert cnt2 == 1 and idx2.tolist() == [5] and w2.tolist() == [1.0]


def test_sample_explicit_uniforms_rule():
    rng = np.random.default_rng(4)
    n, m = 5000, 300
    p = rng.random(n).astype(np.float32)
    p /= p.sum(dtype=np.float64)
    p = p.astype(np.float32)
    u = rng.random(n)
    idx, w, cnt = oracle.sample(p, m, u=u, row_base=1000)
    phat = np.minimum(1.0, m * p.astype(np.float64))
    want = np.nonzero(u < phat)[0] + 1000
    np.testing.assert_array_equal(idx, want)
    np.testing.assert_array_equal(w, 1.0 / phat[want - 1000])
    # the generated uniforms are u53(rng(seed, 9, row)): same decisions as passing them explicitly
    uu = fctgen.uniforms(77, 1000, n)
    a = oracle.sample(p, m, seed=77, row_base=1000)
    b = oracle.sample(p, m, u=uu, row_base=1000)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


def test_sample_expectations():
    """E[count] = sum phat; E ||D Z x||_1 = ||Z x||_1 (unbiased); count <= 2m."""
    rng = np.random.default_rng(5)
    n, m, T = 4000, 200, 300
    Z = rng.standard_cauchy((n, 3))
    x = rng.standard_normal(3)
    lam = np.abs(Z).sum(axis=1)
    p = (lam / lam.sum()).astype(np.float32)
    phat = np.minimum(1.0, m * p.astype(np.float64))
    zx = np.abs(Z @ x)
    counts, ests = [], []
    for t in range(T):
        idx, w, cnt = oracle.sample(p, m, seed=1000 + t)
        counts.append(cnt)
        ests.append((w * zx[idx]).sum())
        assert cnt <= 2 * m
    counts = np.array(counts)
    var_c = (phat * (1 - phat)).sum()
    assert abs(counts.mean() - phat.sum()) < 4 * math.sqrt(var_c / T)
    var_e = ((1 - phat) / np.maximum(phat, 1e-300) * zx ** 2).sum()
    assert abs(np.mean(ests) - zx.sum()) < 4 * math.sqrt(var_e / T)


def test_sample_tie_rule_is_strict():
    """Reading R14: keep iff u < phat (strict); u = phat is out, u just below phat is in."""
    rng = np.random.default_rng(6)
    n, m = 2000, 100
    p = (rng.random(n) / n).astype(np.float32)
    phat = np.minimum(1.0, m * p.astype(np.float64))
    u_eq = phat.copy()
    u_below = np.nextafter(phat, 0.0)
    assert oracle.sample(p, m, u=u_eq)[2] == 0
    np.testing.assert_array_equal(oracle.sample(p, m, u=u_below)[0], np.arange(n))


# ---------------------------------------------------------------- NEXT-1: exact l1 row norms of U = A R^-1
def test_rownorm_exact_closed_forms():
    """lambda_i = ||(A R^-1)_i||_1.  Closed forms that catch a transposed R^-1, a dropped
    absolute value or a wrong index: Rinv = I -> ||a_i||_1; Rinv = diag(r) -> sum_l |a_il r_l|; a signed
    permutation -> ||a_i||_1; A = e_l rows -> the l1 norm of ROW l of Rinv (not column l); d = 1 -> |a r|."""
    rng = np.random.default_rng(11)
    n, d = 300, 7
    A = rng.standard_normal((n, d)).astype(np.float32)
    A64 = A.astype(np.float64)
    lam, tot = oracle.rownorm_exact(A, np.eye(d))
    np.testing.assert_allclose(lam, np.abs(A64).sum(1), rtol=1e-15)
    assert math.isclose(tot, float(np.abs(A64).sum()), rel_tol=1e-12)
    r = rng.standard_normal(d) * 3
    lam, _ = oracle.rownorm_exact(A, np.diag(r))
    np.testing.assert_allclose(lam, np.abs(A64 * r).sum(1), rtol=1e-14)
    P = np.eye(d)[rng.permutation(d)] * rng.choice([-1.0, 1.0], d)
    lam, _ = oracle.rownorm_exact(A, P)
    np.testing.assert_allclose(lam, np.abs(A64).sum(1), rtol=1e-14)
    Rinv = np.triu(rng.standard_normal((d, d))) + 2 * np.eye(d)
    E = np.eye(d, dtype=np.float32)
    lam, _ = oracle.rownorm_exact(E, Rinv)
    want = [math.fsum(abs(x) for x in Rinv[l, :]) for l in range(d)]
    np.testing.assert_allclose(lam, want, rtol=1e-15)
    assert not np.allclose(lam, np.abs(Rinv).sum(0))            # the column sums differ: orientation is pinned
    lam, _ = oracle.rownorm_exact(A[:, :1].copy(), np.array([[-2.5]]))
    np.testing.assert_allclose(lam, 2.5 * np.abs(A64[:, 0]), rtol=1e-15)


def test_rownorm_exact_invariants_and_bound():
    rng = np.random.default_rng(12)
    n, d = 256, 6
    A = rng.standard_normal((n, d)).astype(np.float32)
    A[3] = 0.0
    Rinv = np.triu(rng.standard_normal((d, d))) + 2 * np.eye(d)
    lam, tot, bnd = oracle.rownorm_exact(A, Rinv, with_bound=True)
    assert lam[3] == 0.0 and bnd[3] == 0.0
    lam2, _ = oracle.rownorm_exact(A * np.float32(-8.0), Rinv)
    np.testing.assert_allclose(lam2, 8.0 * lam, rtol=1e-14)          # |alpha| homogeneity
    lam3, _ = oracle.rownorm_exact(A, 0.5 * Rinv)
    np.testing.assert_allclose(lam3, 0.5 * lam, rtol=1e-14)
    assert (lam <= bnd * (1 + 1e-12)).all()                            # triangle inequality
    # brute force with exactly rounded sums on a few rows
    for i in (0, 1, 100):
        want = math.fsum(abs(math.fsum(float(A[i, l]) * Rinv[l, j] for l in range(d))) for j in range(d))
        assert math.isclose(lam[i], want, rel_tol=1e-14)


# ---------------------------------------------------------------- NEXT-4: multinomial m-draw sampling
def test_multinomial_point_mass_and_zero_rows():
    p = np.zeros(1000, np.float32)
    p[417] = 0.25
    idx, w, T, F = oracle.sample_multinomial(p, 64, seed=3)
    assert (idx == 417).all() and np.all(w == 1.0 / 64)          # weight = 1 / (m * phat), phat = 1
    rng = np.random.default_rng(5)
    p = rng.random(5000).astype(np.float32)
    p[::3] = 0.0
    idx, w, T, F = oracle.sample_multinomial(p, 20000, seed=4, row_base=100)
    assert (p[idx - 100] > 0).all()                                # zero rows never drawn
    assert T < 2 ** 62 and T > 0


def test_multinomial_uniform_closed_form():
    """n a power of two, all p equal: every W_i is equal, so draw j is exactly floor(X_j n / 2^53) with
    X_j the top 53 bits of the stream-10 generator (fctgen's independent copy of rng_u64)."""
    n, m, seed = 1 << 12, 3000, 77
    p = np.full(n, 1.0 / n, np.float32)
    idx, w, T, F = oracle.sample_multinomial(p, m, seed=seed)
    want = [(fctgen.rng_u64(seed, 10, j) >> 11) * n >> 53 for j in range(m)]
    np.testing.assert_array_equal(idx, want)
    np.testing.assert_allclose(w, n / m, rtol=1e-15)


def test_multinomial_distribution_and_unbiased():
    rng = np.random.default_rng(6)
    n = 25
    p = (rng.random(n) ** 3 + 0.01).astype(np.float32)      # every expected count >= 5 for the chi-square
    idx, w, T, F = oracle.sample_multinomial(p, 200000, seed=9)
    counts = np.bincount(idx, minlength=n)
    expected = 200000 * p.astype(np.float64) / p.astype(np.float64).sum()
    chi2 = ((counts - expected) ** 2 / expected).sum()
    assert stats.chi2.sf(chi2, n - 1) > 1e-3
    # Horvitz-Thompson: sum_j weight_j f(idx_j) is unbiased for sum_i f(i) (f = p-independent values)
    f = rng.standard_normal(n) + 3.0
    est = []
    for s in range(300):
        i2, w2, _, _ = oracle.sample_multinomial(p, 50, seed=1000 + s)
        est.append(float((w2 * f[i2]).sum()))
    est = np.array(est)
    assert abs(est.mean() - f.sum()) < 3 * est.std(ddof=1) / math.sqrt(len(est)) + 1e-9
