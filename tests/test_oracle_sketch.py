"""Pins for oracle O1 (Y = 4 B C H~ D A, Sec. 3.1) against sources other than itself."""
import os

import numpy as np
import pytest
import scipy.linalg
from scipy import stats

import fctgen
import oracle
from oracle import dense

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rand_inputs(n, d, s, r1, seed):
    rng = np.random.default_rng(seed)
    n_pad = -(-n // s) * s
    A = rng.standard_normal((n, d)).astype(np.float32)
    sg = rng.choice(np.array([-1, 1], np.int8), n_pad)
    c = rng.standard_cauchy(2 * n_pad).astype(np.float32)
    h = rng.integers(0, r1, 2 * n_pad).astype(np.int32)
    return A, sg, c, h


def unit_probe(s, A, n_pad=None):
    """Inputs that make Y expose H~ A itself: D = I, c = 1/4, bucket(H~-row t) = t (r1 = 2n')."""
    n = A.shape[0]
    n_pad = n_pad or -(-n // s) * s
    sg = np.ones(n_pad, np.int8)
    c = np.full(2 * n_pad, 0.25, np.float32)
    h = np.arange(2 * n_pad, dtype=np.int32)
    Y, _ = oracle.sketch(A, sg, c, h, s, 2 * n_pad)
    return Y


# ---------------------------------------------------------------- definition (dense materialisation)
@pytest.mark.parametrize("s", [1, 2, 4, 8, 16, 32, 64])
@pytest.mark.parametrize("r1", [1, 3, 16])
@pytest.mark.parametrize("n_extra", [0, 5])
def test_sketch_equals_dense_definition(s, r1, n_extra):
    n = 2 * s + n_extra if s > 1 else 7 + n_extra
    d = 4
    A, sg, c, h = rand_inputs(n, d, s, r1, seed=s * 100 + r1 + n_extra)
    Y, _ = oracle.sketch(A, sg, c, h, s, r1)
    Yd = dense.dense_sketch(A, sg, c, h, s, r1)
    np.testing.assert_allclose(Y, Yd, rtol=1e-12, atol=1e-12 * np.abs(Yd).max())


# ---------------------------------------------------------------- Hadamard closed forms
def _golden_hadamard():
    H = {"H2": [], "H4": []}
    with open(os.path.join(GOLDEN, "hadamard_paper.txt")) as f:
        for line in f:
            t = line.split()
            if t and t[0] in H:
                H[t[0]].append([int(x) for x in t[1:]])
    return {k: np.array(v, np.float64) for k, v in H.items()}


def test_hadamard_golden_from_paper():
    g = _golden_hadamard()
    np.testing.assert_array_equal(dense.hadamard_recursive(2), g["H2"])
    np.testing.assert_array_equal(dense.hadamard_recursive(4), g["H4"])
    for s, H in [(2, g["H2"]), (4, g["H4"])]:
        Y = unit_probe(s, np.eye(s, dtype=np.float32))
        np.testing.assert_allclose(Y[:s], H / np.sqrt(s), rtol=0, atol=1e-15)


@pytest.mark.parametrize("lg", range(0, 10))
def test_oracle_hadamard_full_matrix(lg):
    """Oracle's explicit H_s == recursive construction == scipy.linalg.hadamard (Sylvester), s <= 512."""
    s = 1 << lg
    Y = unit_probe(s, np.eye(s, dtype=np.float32))
    Hs = scipy.linalg.hadamard(s).astype(np.float64)
    np.testing.assert_array_equal(dense.hadamard_recursive(s), Hs)
    np.testing.assert_allclose(Y[:s], Hs / np.sqrt(s), rtol=0, atol=1e-14)
    np.testing.assert_allclose(Y[s:2 * s], np.eye(s), rtol=0, atol=0)     # identity half of G_s


@pytest.mark.parametrize("lg", [10, 11, 12])
def test_oracle_hadamard_columns_large(lg):
    s = 1 << lg
    cols = [0, 1, s // 2 + 3, s - 1]
    A = np.zeros((s, len(cols)), np.float32)
    A[cols, np.arange(len(cols))] = 1.0
    Y = unit_probe(s, A)
    Hs = scipy.linalg.hadamard(s)[:, cols].astype(np.float64)
    np.testing.assert_allclose(Y[:s], Hs / np.sqrt(s), rtol=0, atol=1e-14)


@pytest.mark.parametrize("j", [1, 2, 3, 4, 5, 6])
def test_comb_witness(j):
    """s = 4^j, z = 1{i = 0 mod sqrt(s)} / s^(1/4):  H_s z = 1{i < sqrt(s)} / s^(1/4),
    ||G_s z||_1 = 2 s^(1/4)  (tightness example of the uncertainty lemma)."""
    s = 4 ** j
    rs = int(round(np.sqrt(s)))
    z = np.zeros((s, 1), np.float64)
    z[::rs, 0] = 1.0
    z /= s ** 0.25
    Y = unit_probe(s, z.astype(np.float32))
    want = np.zeros(s)
    want[:rs] = 1.0 / s ** 0.25
    np.testing.assert_allclose(Y[:s, 0], want, rtol=1e-6, atol=1e-7 / s ** 0.25)
    np.testing.assert_allclose(np.abs(Y[:, 0]).sum(), 2 * s ** 0.25, rtol=1e-6)


@pytest.mark.parametrize("s", [1, 4, 16, 64, 256])
def test_e1_l1_norm(s):
    """||H~ e_1||_1 = sqrt(s) + 1; with r1 = 1, c = 1, D = I: Y = 4 (sqrt(s) + 1)."""
    A = np.zeros((s, 1), np.float32)
    A[0, 0] = 1.0
    Y, _ = oracle.sketch(A, np.ones(s, np.int8), np.ones(2 * s, np.float32), np.zeros(2 * s, np.int32), s, 1)
    assert Y.shape == (1, 1)
    np.testing.assert_allclose(Y[0, 0], 4 * (np.sqrt(s) + 1), rtol=1e-13)


# ---------------------------------------------------------------- invariants of H~
@pytest.mark.parametrize("s", [2, 16, 128])
def test_Htilde_isometry_and_l1_bounds(s):
    rng = np.random.default_rng(s)
    n = 4 * s
    for trial in range(3):
        y = rng.standard_normal((n, 1)).astype(np.float32)
        Hy = unit_probe(s, y)[:, 0]
        y64 = y[:, 0].astype(np.float64)
        # H~^T H~ = 2I  =>  ||H~ y||_2^2 = 2 ||y||_2^2
        np.testing.assert_allclose((Hy ** 2).sum(), 2 * (y64 ** 2).sum(), rtol=1e-12)
        # ||H~ y||_1 <= sqrt(4 s) ||y||_1
        assert np.abs(Hy).sum() <= np.sqrt(4 * s) * np.abs(y64).sum() * (1 + 1e-12)
        # uncertainty principle per block: ||G_s z||_1 >= 1/2 s^(1/4) ||z||_2
        for b in range(n // s):
            z = y64[b * s:(b + 1) * s]
            g = np.concatenate([Hy[2 * s * b: 2 * s * b + 2 * s]])
            assert np.abs(g).sum() >= 0.5 * s ** 0.25 * np.linalg.norm(z)


def test_column_sum_identity_integer_exact():
    """C = I: 1^T Y = 4 sum_b (sum_l (DA)_{bs+l} + sqrt(s) (DA)_{bs})  -- 1^T B = 1^T,
    1^T H_s = sqrt(s) e_0^T.  Exact on integer-valued A with s a power of 4."""
    s, n, d, r1 = 16, 16 * 9, 5, 8
    rng = np.random.default_rng(1)
    A = rng.integers(-50, 50, (n, d)).astype(np.float32)
    sg = rng.choice(np.array([-1, 1], np.int8), n)
    h = rng.integers(0, r1, 2 * n).astype(np.int32)
    Y, _ = oracle.sketch(A, sg, np.ones(2 * n, np.float32), h, s, r1)
    DA = sg[:, None].astype(np.float64) * A
    want = 4 * (DA.sum(axis=0) + np.sqrt(s) * DA[::s].sum(axis=0))
    np.testing.assert_array_equal(Y.sum(axis=0), want)


def test_linearity_homogeneity_shards():
    s, r1, d = 32, 8, 3
    A1, sg, c, h = rand_inputs(256, d, s, r1, 5)
    A2 = np.random.default_rng(6).standard_normal(A1.shape).astype(np.float32)
    Y1, _ = oracle.sketch(A1, sg, c, h, s, r1)
    Y2, _ = oracle.sketch(A2, sg, c, h, s, r1)
    Y12, _ = oracle.sketch((A1.astype(np.float64) + A2).astype(np.float32), sg, c, h, s, r1)
    np.testing.assert_allclose(Y12, Y1 + Y2, rtol=1e-6, atol=1e-6 * np.abs(Y12).max())
    Y3, _ = oracle.sketch(A1 * np.float32(-2.0), sg, c, h, s, r1)
    np.testing.assert_allclose(Y3, -2.0 * Y1, rtol=1e-13, atol=0)
    # shard additivity: s-aligned row shards, aux arrays sliced by 2*row0
    Ys = sum(oracle.sketch(A1[r0:r0 + 64], sg[r0:r0 + 64], c[2 * r0:2 * r0 + 128], h[2 * r0:2 * r0 + 128], s, r1)[0]
             for r0 in range(0, 256, 64))
    np.testing.assert_allclose(Ys, Y1, rtol=1e-12, atol=1e-12 * np.abs(Y1).max())


def test_r1_equals_1_is_a_gemv():
    """r1 = 1: Y = 4 c^T (H~ D A) -- blockwise with scipy.linalg.hadamard (library routine)."""
    s, n, d = 64, 64 * 5, 6
    A, sg, c, h = rand_inputs(n, d, s, 1, 9)
    Y, _ = oracle.sketch(A, sg, c, np.zeros_like(h), s, 1)
    H = scipy.linalg.hadamard(s) / np.sqrt(s)
    DA = sg[:, None].astype(np.float64) * A
    want = np.zeros(d)
    for b in range(n // s):
        z = DA[b * s:(b + 1) * s]
        want += c[2 * s * b: 2 * s * b + s].astype(np.float64) @ (H @ z)
        want += c[2 * s * b + s: 2 * s * b + 2 * s].astype(np.float64) @ z
    np.testing.assert_allclose(Y[0], 4 * want, rtol=1e-12, atol=1e-12 * np.abs(want).max())


def test_s_equals_1_brute_force():
    """s = 1: row i contributes 4 d_i (c_2i e_h(2i) + c_2i+1 e_h(2i+1)) A_i."""
    n, d, r1 = 50, 3, 7
    A, sg, c, h = rand_inputs(n, d, 1, r1, 11)
    Y, M = oracle.sketch(A, sg, c, h, 1, r1)
    want = np.zeros((r1, d))
    wabs = np.zeros((r1, d))
    for i in range(n):
        for t in (2 * i, 2 * i + 1):
            want[h[t]] += 4.0 * float(sg[i]) * float(c[t]) * A[i].astype(np.float64)
            wabs[h[t]] += 4.0 * abs(float(c[t])) * np.abs(A[i].astype(np.float64))
    np.testing.assert_allclose(Y, want, rtol=1e-12, atol=1e-12 * np.abs(want).max())
    np.testing.assert_allclose(M, wabs, rtol=1e-12)


def test_magnitude_bound_dominates():
    A, sg, c, h = rand_inputs(300, 4, 16, 8, 13)
    Y, M = oracle.sketch(A, sg, c, h, 16, 8)
    assert (np.abs(Y) <= M * (1 + 1e-12)).all()
    Yabs, _ = oracle.sketch(np.abs(A), np.ones_like(sg), np.abs(c), h, 16, 8)
    assert (Yabs <= M * (1 + 1e-12) + 1e-12).all()      # |H| entries replace +-1/sqrt(s) by 1/sqrt(s)


# ---------------------------------------------------------------- distributional / statistical pins
def test_one_stability_of_bucket_values():
    """For fixed y and B, (Pi1 y)_k / (4 gamma_k) ~ standard Cauchy with gamma_k = sum_{h(i)=k} |(H~Dy)_i|
    (1-stability P:L1186-1189; bucket scales P:L4011-4029).  KS over 4000 draws of C."""
    n, s, r1 = 256, 64, 16
    rng = np.random.default_rng(2)
    y = rng.standard_normal((n, 1)).astype(np.float32)
    sg = rng.choice(np.array([-1, 1], np.int8), n)
    h = rng.integers(0, r1, 2 * n).astype(np.int32)
    g = unit_probe(s, (sg[:, None] * y).astype(np.float32))[:, 0]          # H~ D y
    gamma = np.bincount(h, weights=np.abs(g), minlength=r1)
    np.testing.assert_allclose(gamma.sum(), np.abs(g).sum(), rtol=1e-12)
    ratios = []
    for t in range(4000):
        c = rng.standard_cauchy(2 * n).astype(np.float32)
        Y, _ = oracle.sketch(y, sg, c, h, s, r1, with_bound=True)
        ratios.append(Y[:, 0] / (4 * gamma))
    ratios = np.concatenate(ratios)
    # the fp32 rounding of c perturbs each ratio by <= 6e-8 relative: invisible to the KS test
    assert stats.kstest(ratios, "cauchy").pvalue > 1e-3
    assert abs(np.median(np.abs(ratios)) - 1.0) < 0.02


def test_distortion_lower_side_empirical():
    """||Ax||_1 <= ||Pi1 A x||_1 (Thm FCT1) for >= 99% of random x (empirical gate;
    the paper's probability bound is vacuous at practical s)."""
    n, d, s, r1 = 1 << 13, 4, 64, 64
    cfg = fctgen.CONFIGS[1]
    ok = 0
    total = 0
    for seed in range(3):
        inp = fctgen.make_inputs(cfg, n=n, d=d, s=s, r1=r1, seed=100 + seed)
        Y, _ = oracle.sketch(inp.A, inp.signs, inp.cauchy, inp.hash, s, r1)
        X = np.random.default_rng(seed).standard_normal((d, 300))
        lhs = np.abs(inp.A.astype(np.float64) @ X).sum(axis=0)
        rhs = np.abs(Y @ X).sum(axis=0)
        ok += int((lhs <= rhs).sum())
        total += X.shape[1]
    assert ok / total >= 0.99
