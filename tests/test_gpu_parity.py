"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded inputs.

Tolerances:
  sketch   |Y_gpu - Y_oracle| <= 1e-5 * Mbound entrywise, Mbound = 4|B||C||H~||D||A| (north_star)
  lambda   |lambda_gpu - lambda_oracle| <= 1e-5 * lambda_oracle per row, same Rinv and Pi2 (north_star)
  sample   idx / weight bit-exact given identical p and uniforms (north_star)
  R, Rinv  1e-9 relative to the matrix norm x cond, same fp32 Y (CholeskyQR2 vs Householder)
"""
import numpy as np
import pytest

import fctgen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SK_TOL = 1e-5
LAM_TOL = 1e-5
# NEXT-1 (exact l1 norms on the tensor cores, reading R28): every row of the 9042-row config samples
# meets north_star's 1e-5 relative lambda bar (measured r02: max 8.5e-6 at the cfg-4 shape, median 4e-7);
# held at that bar.  The full-size fraction is measured in test_gpu_fullsize.py.
EXACT_FAIL_FRAC = {1: 0.0, 2: 0.0, 3: 0.0, 4: 0.0, 5: 0.0}
EXACT_MAX_REL = 1e-5


@pytest.fixture(scope="module")
def fct():
    import paper_1207_4684_b200 as m
    from paper_1207_4684_b200 import build
    build.build()
    m.load()
    return m


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def sketch_gpu(fct, inp, s=None, r1=None):
    s = inp.s if s is None else s
    r1 = inp.r1 if r1 is None else r1
    Y = fct.fct_sketch(dev(inp.A), dev(inp.signs), dev(inp.cauchy), dev(inp.hash), s, r1)
    return Y.cpu().numpy().astype(np.float64)


def assert_sketch_close(Yg, Yo, Mb, tol=SK_TOL):
    err = np.abs(Yg - Yo)
    ratio = err / np.maximum(Mb, 1e-300)
    worst = np.unravel_index(np.argmax(ratio), ratio.shape)
    assert (err <= tol * Mb + 1e-30).all(), f"max err/Mbound = {ratio.max():.3e} at {worst}"


# ---------------------------------------------------------------- K1 sketch
@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_sketch_configs_ragged(fct, c):
    """Each config's (d, s, r1, data kind) at a size spanning several blocks plus a ragged tail."""
    cfg = fctgen.CONFIGS[c]
    nblocks = {1: 40, 2: 20, 3: 9, 4: 6, 5: 3}[c]
    n = nblocks * cfg.s + 37
    inp = fctgen.make_inputs(cfg, n=n)
    Yo, Mb = oracle.sketch(inp.A, inp.signs, inp.cauchy, inp.hash, cfg.s, cfg.r1)
    Yg = sketch_gpu(fct, inp)
    assert_sketch_close(Yg, Yo, Mb)


@pytest.mark.parametrize("n,d,s,r1", [
    (1, 1, 1, 1), (5, 3, 8, 2), (63, 7, 64, 16), (1000, 13, 16, 1), (1000, 33, 4, 128), (300, 1, 256, 64),
    (4096, 130, 32, 8), (2048 + 5, 8, 2048, 64), (4096 + 1, 4, 4096, 32), (777, 5, 1, 4096), (2000, 40, 128, 20000),
])
def test_sketch_edge_shapes(fct, n, d, s, r1):
    rng = np.random.default_rng(n * 31 + d)
    n_pad = -(-n // s) * s
    A = (rng.standard_normal((n, d)) * rng.choice([1e-3, 1.0, 1e3], (n, 1))).astype(np.float32)
    sg = rng.choice(np.array([-1, 1], np.int8), n_pad)
    c = rng.standard_cauchy(2 * n_pad).astype(np.float32)
    h = rng.integers(0, r1, 2 * n_pad).astype(np.int32)
    Yo, Mb = oracle.sketch(A, sg, c, h, s, r1)
    Yg = fct.fct_sketch(dev(A), dev(sg), dev(c), dev(h), s, r1).cpu().numpy().astype(np.float64)
    assert_sketch_close(Yg, Yo, Mb)


@pytest.mark.parametrize("noextra", [False, True])
def test_sketch_extra_ctas_tail(fct, noextra, monkeypatch):
    """K1's leftover SMs (5 slices of 16 columns fill 145 of 148 SMs; the 3 left over run one extra CTA that takes
    a tail of the blocks in 5 passes, one slice per pass, flushing its partial between passes), with a partly
    empty last slice (d = 72) and a ragged tail block; the same input with the extra CTAs switched off."""
    if noextra:
        monkeypatch.setenv("FCT_SKETCH_NOEXTRA", "1")
    cfg = fctgen.CONFIGS[2]
    inp = fctgen.make_inputs(cfg, n=1200 * 256 + 77, s=256, r1=1024, d=72)
    Yo, Mb = oracle.sketch(inp.A, inp.signs, inp.cauchy, inp.hash, 256, 1024)
    Yg = sketch_gpu(fct, inp)
    assert_sketch_close(Yg, Yo, Mb)


@pytest.mark.parametrize("onewave", [False, True])
def test_sketch_multiwave_grid(fct, onewave, monkeypatch):
    """K1's multi-wave grid: 19 slices of 4 columns (d = 76, r1 = 8192) fill only 134 of 148 SMs in one wave, so
    the launch runs several unpaced waves of one CTA per SM (capped here by the 48 blocks); FCT_SKETCH_ONEWAVE=1
    keeps the paced single wave with its extra CTA. Ragged tail block included."""
    if onewave:
        monkeypatch.setenv("FCT_SKETCH_ONEWAVE", "1")
    cfg = fctgen.CONFIGS[5]
    inp = fctgen.make_inputs(cfg, n=48 * 1024 + 33, s=1024, r1=8192, d=76)
    Yo, Mb = oracle.sketch(inp.A, inp.signs, inp.cauchy, inp.hash, 1024, 8192)
    Yg = sketch_gpu(fct, inp)
    assert_sketch_close(Yg, Yo, Mb)


def test_sketch_strided_accumulate_and_shards(fct):
    """lda > d (a column slice of a wider matrix), accumulate=1, and s-aligned row shards."""
    cfg = fctgen.CONFIGS[2]
    inp = fctgen.make_inputs(cfg, n=8 * cfg.s)
    wide = np.zeros((inp.A.shape[0], 24), np.float32)
    wide[:, 3:3 + 16] = inp.A
    Aw = dev(wide)[:, 3:3 + 16]
    assert Aw.stride(0) == 24
    sg, c, h = dev(inp.signs), dev(inp.cauchy), dev(inp.hash)
    Yo, Mb = oracle.sketch(inp.A, inp.signs, inp.cauchy, inp.hash, cfg.s, cfg.r1)
    Y = fct.fct_sketch(Aw, sg, c, h, cfg.s, cfg.r1)
    assert_sketch_close(Y.cpu().numpy().astype(np.float64), Yo, Mb)
    # shards with accumulate: Pi1 A = sum_g Pi1_g A_g
    Ys = torch.zeros_like(Y)
    for r0 in range(0, inp.A.shape[0], 3 * cfg.s):
        r1_ = min(r0 + 3 * cfg.s, inp.A.shape[0])
        fct.fct_sketch(Aw[r0:r1_], sg[r0:], c[2 * r0:], h[2 * r0:], cfg.s, cfg.r1, Y=Ys, accumulate=True)
    assert_sketch_close(Ys.cpu().numpy().astype(np.float64), Yo, Mb)


def test_sketch_errors(fct):
    A = torch.zeros((10, 4), device="cuda")
    sg = torch.ones(16, dtype=torch.int8, device="cuda")
    c = torch.ones(32, device="cuda")
    h = torch.full((32,), 99, dtype=torch.int32, device="cuda")
    with pytest.raises(fct.FctError, match="FCT_ERR_ARG"):
        fct.fct_sketch(A, sg, c, h, 3, 8)


# ---------------------------------------------------------------- K5 conditioning
@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_condition_matches_householder(fct, c):
    cfg = fctgen.CONFIGS[c]
    inp = fctgen.make_inputs(cfg, n=2 * cfg.s)
    Y32 = oracle.sketch(inp.A, inp.signs, inp.cauchy, inp.hash, cfg.s, cfg.r1, with_bound=False).astype(np.float32)
    R_o, Rinv_o, _ = oracle.condition(Y32.astype(np.float64))
    R, Rinv, info = fct.fct_condition(dev(Y32))
    R, Rinv = R.cpu().numpy(), Rinv.cpu().numpy()
    cond = np.linalg.cond(Y32.astype(np.float64))
    assert np.abs(R - R_o).max() <= 1e-12 * cond * np.abs(R_o).max()
    assert np.abs(Rinv - Rinv_o).max() <= 1e-12 * cond * np.abs(Rinv_o).max()
    assert (np.diag(R) > 0).all() and np.allclose(np.tril(R, -1), 0)


def test_condition_singular_reports_info(fct):
    Y = np.zeros((64, 4), np.float32)
    Y[:, 0] = 1.0
    Y[:, 1] = 1.0     # two equal columns -> rank deficient
    with pytest.raises(fct.FctError, match="SINGULAR"):
        fct.fct_condition(dev(Y))


def _ill_conditioned_Y(r1, d, delta, seed):
    """Exactly representable fp32 Y of full rank with cond ~ ||Y|| / delta: small-integer columns, the last
    column = col0 + col1 except a single entry delta in row 0 (where every other column is 0)."""
    rng = np.random.default_rng(seed)
    Y = rng.integers(-8, 9, (r1, d)).astype(np.float32)
    Y[0] = 0.0
    Y[:, d - 1] = Y[:, 0] + Y[:, 1]
    Y[0, d - 1] = delta
    return Y


@pytest.mark.parametrize("delta,path", [(2.0 ** -30, -1), (2.0 ** -4, 0)])
def test_condition_shifted_cholqr3_fallback(fct, delta, path):
    """cond(Y) ~ 1e11 breaks CholeskyQR2 (Gram cond ~ 1e22 > 1/u): the device restarts with shifted CholeskyQR3
    (info = -1) and still matches Householder QR ("for example using a QR-factorization");
    a moderately conditioned Y stays on CholeskyQR2 (info = 0)."""
    r1, d = 512, 16
    Y = _ill_conditioned_Y(r1, d, delta, seed=3)
    Y64 = Y.astype(np.float64)
    cond = np.linalg.cond(Y64)
    R_o, Rinv_o, _ = oracle.condition(Y64)
    R, Rinv, info = fct.fct_condition(dev(Y))
    assert int(info.item()) == path
    R, Rinv = R.cpu().numpy(), Rinv.cpu().numpy()
    assert (np.diag(R) > 0).all() and np.allclose(np.tril(R, -1), 0)
    assert np.abs(R - R_o).max() <= 1e-12 * cond * np.abs(R_o).max()
    assert abs(R[-1, -1] - R_o[-1, -1]) <= 1e-4 * R_o[-1, -1]
    orth = lambda Ri: np.abs((Y64 @ Ri).T @ (Y64 @ Ri) - np.eye(d)).max()   # evaluated in fp64 on the host
    assert orth(Rinv) <= max(1e-10, 10 * orth(Rinv_o))
    np.testing.assert_allclose(R @ Rinv, np.eye(d), atol=1e-8 * cond ** 0.5)


def test_condition_nonfinite_is_nan_not_garbage(fct):
    """Even the shifted fallback fails on a non-finite Y: info > 0 and R, Rinv are NaN (no silent
    garbage flows into the row norms)."""
    Y = np.random.default_rng(4).standard_normal((256, 8)).astype(np.float32)
    Y[17, 3] = np.inf
    R, Rinv, info = fct.fct_condition(dev(Y), check=False)
    assert int(info.item()) > 0
    assert torch.isnan(R).all() and torch.isnan(Rinv).all()


@pytest.mark.parametrize("r1,d", [(64, 64), (20000, 3), (300, 128), (128, 1), (8192, 100)])
def test_condition_shapes(fct, r1, d):
    Y = np.random.default_rng(r1 + d).standard_normal((r1, d)).astype(np.float32)
    R_o, Rinv_o, _ = oracle.condition(Y.astype(np.float64))
    R, Rinv, info = fct.fct_condition(dev(Y))
    assert int(info.item()) == 0
    cond = np.linalg.cond(Y.astype(np.float64))
    R, Rinv = R.cpu().numpy(), Rinv.cpu().numpy()
    assert np.abs(R - R_o).max() <= 1e-12 * cond * np.abs(R_o).max()
    assert np.abs(Rinv - Rinv_o).max() <= 1e-12 * cond * np.abs(Rinv_o).max()


@pytest.mark.parametrize("r1,d", [(64, 8), (1024, 32), (4096, 64), (8192, 100), (300, 128)])
def test_condition_series_pass_equals_cholesky_pass(fct, r1, d, monkeypatch):
    """Passes >= 1 factor a near-identity Gram (|G - I| <= 2^-26 entrywise) by its second-order series
    (R32) instead of d serial Cholesky steps: R and R^-1 agree with the serial path
    (FCT_COND_NOSERIES=1) to fp64 rounding, and both match Householder QR."""
    Y = np.random.default_rng(r1 * 7 + d).standard_normal((r1, d)).astype(np.float32)
    R_s, Ri_s, info_s = fct.fct_condition(dev(Y))
    monkeypatch.setenv("FCT_COND_NOSERIES", "1")
    R_c, Ri_c, info_c = fct.fct_condition(dev(Y))
    assert int(info_s.item()) == 0 and int(info_c.item()) == 0
    R_s, Ri_s, R_c, Ri_c = (t.cpu().numpy() for t in (R_s, Ri_s, R_c, Ri_c))
    assert np.abs(R_s - R_c).max() <= 64 * d * 2.0 ** -53 * np.abs(R_c).max()
    assert np.abs(Ri_s - Ri_c).max() <= 64 * d * 2.0 ** -53 * np.abs(Ri_c).max()
    R_o, Rinv_o, _ = oracle.condition(Y.astype(np.float64))
    cond = np.linalg.cond(Y.astype(np.float64))
    assert np.abs(R_s - R_o).max() <= 1e-12 * cond * np.abs(R_o).max()
    assert np.abs(Ri_s - Rinv_o).max() <= 1e-12 * cond * np.abs(Rinv_o).max()


# ---------------------------------------------------------------- K2 row-norm
def _rinv_for(inp):
    """Rinv from the oracle's own conditioning of the oracle sketch (stage-wise parity input)."""
    Y, _ = oracle.sketch(inp.A, inp.signs, inp.cauchy, inp.hash, inp.s, inp.r1)
    R, Rinv, _ = oracle.condition(Y.astype(np.float32).astype(np.float64))
    return Rinv


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_rownorm_configs(fct, c):
    cfg = fctgen.CONFIGS[c]
    inp = fctgen.make_inputs(cfg, n=2 * cfg.s)
    Rinv = _rinv_for(inp)
    # rows to score: a larger slice of the same matrix kind (ragged: not a multiple of 32)
    B = fctgen.matrix(cfg.kind, cfg.seed, max(cfg.n, 20013), cfg.d, 0, 20000 + 13)
    B[5] = 0.0
    lam_o, tot_o = oracle.rownorm(B, Rinv, inp.pi2)
    lam, tot = fct.l1_rownorm(dev(B), dev(Rinv), dev(inp.pi2))
    lam = lam.cpu().numpy().astype(np.float64)
    rel = np.abs(lam - lam_o) / np.maximum(lam_o, 1e-300)
    assert lam[5] == 0.0
    assert (np.abs(lam - lam_o) <= LAM_TOL * lam_o).all(), f"max rel {rel.max():.3e}"
    np.testing.assert_allclose(float(tot.item()), lam.sum(), rtol=1e-12)


@pytest.mark.parametrize("c", [2, 4])
def test_rownorm_gaussian_pi2(fct, c):
    """NEXT-1's Gaussian-Pi2 estimator is the same kernel with Gaussian Pi2: parity at 1e-5."""
    cfg = fctgen.CONFIGS[c]
    inp = fctgen.make_inputs(cfg, n=2 * cfg.s)
    Rinv = _rinv_for(inp)
    Pi2 = fctgen.normals(cfg.seed, fctgen.ST_PI2, 0, cfg.d * cfg.k).reshape(cfg.d, cfg.k).astype(np.float32)
    B = fctgen.matrix(cfg.kind, cfg.seed, max(cfg.n, 6000), cfg.d, 0, 6000 + 11)
    lam_o, _ = oracle.rownorm(B, Rinv, Pi2)
    lam, _ = fct.l1_rownorm(dev(B), dev(Rinv), dev(Pi2))
    lam = lam.cpu().numpy().astype(np.float64)
    assert (np.abs(lam - lam_o) <= LAM_TOL * lam_o + 1e-30).all()


@pytest.mark.parametrize("k", [1, 2, 3, 7, 8, 16, 20, 27, 29, 32])
def test_rownorm_all_k_and_identity(fct, k):
    rng = np.random.default_rng(k)
    d = 9
    A = rng.standard_normal((1000, d)).astype(np.float32)
    Rinv = np.triu(rng.standard_normal((d, d))) + 4 * np.eye(d)
    Pi2 = rng.standard_cauchy((d, k)).astype(np.float32)
    lam_o, _ = oracle.rownorm(A, Rinv, Pi2)
    lam, _ = fct.l1_rownorm(dev(A), dev(Rinv), dev(Pi2))
    lam = lam.cpu().numpy().astype(np.float64)
    assert (np.abs(lam - lam_o) <= LAM_TOL * lam_o).all()
    # identity: Rinv = I, Pi2 = I -> textbook median of |A| (many exact ties in the candidates)
    I = np.eye(d, dtype=np.float32)
    lam_i, _ = fct.l1_rownorm(dev(A), dev(np.eye(d)), dev(I))
    np.testing.assert_allclose(lam_i.cpu().numpy(), np.median(np.abs(A.astype(np.float64)), axis=1),
                               rtol=1e-7, atol=0)


def test_probs_and_rownorm_probs(fct):
    cfg = fctgen.CONFIGS[2]
    inp = fctgen.make_inputs(cfg, n=4 * cfg.s)
    Rinv = _rinv_for(inp)
    lam_o, tot_o = oracle.rownorm(inp.A, Rinv, inp.pi2)
    lam, p, tot = fct.l1_rownorm_probs(dev(inp.A), dev(Rinv), dev(inp.pi2))
    lam = lam.cpu().numpy()
    # p = (float)(lambda / total) from the GPU's own fp32 lambdas and fp64 total
    want = (lam.astype(np.float64) / lam.astype(np.float64).sum()).astype(np.float32)
    np.testing.assert_array_equal(p.cpu().numpy(), want)
    np.testing.assert_allclose(float(tot.item()), tot_o, rtol=1e-6)


# ---------------------------------------------------------------- K4 sampling (bit-exact)
def _probs(n, seed, heavy=True):
    rng = np.random.default_rng(seed)
    lam = np.abs(rng.standard_cauchy(n)) if heavy else rng.random(n)
    return (lam / lam.sum()).astype(np.float32)


@pytest.mark.parametrize("n,m,row_base", [(1, 1, 0), (2047, 100, 0), (2049, 100, 7), (100000, 4096, 123456),
                                          (1 << 20, 65536, 1 << 30)])
def test_sample_bit_exact(fct, n, m, row_base):
    p = _probs(n, n)
    p[:3] = 1.0                                   # phat = 1 rows
    idx, w, cnt = fct.l1_sample(dev(p), m, seed=99, row_base=row_base, capacity=2 * m + n // 10 + 64)
    gi, gw, gc = fct.trim(idx, w, cnt)
    oi, ow, oc = oracle.sample(p, m, seed=99, row_base=row_base)
    assert gc == oc
    np.testing.assert_array_equal(gi.numpy(), oi)
    np.testing.assert_array_equal(gw.numpy(), ow)       # bitwise: 1/phat in IEEE fp64


def test_device_uniforms_match_host_generator(fct):
    """the device's u_i (rng_u64(seed, 9, row_base + i) >> 11) * 2^-53 equals fctgen's host copy
    for 10^7 rows.  With m = 1: p_i = fp32(u_i) rounded down keeps no row iff every u_dev >= p_i, and p_i rounded
    up keeps every row iff every u_dev < p_i -- together u_dev lies in u_host's fp32 interval on every row."""
    n, seed, rb = 10_000_000, 77, 123457
    u = fctgen.uniforms(seed, rb, n)
    f = u.astype(np.float32)
    lo = np.where(f.astype(np.float64) > u, np.nextafter(f, np.float32(0)), f)
    hi = np.where(f.astype(np.float64) > u, f, np.nextafter(f, np.float32(2)))
    assert (lo.astype(np.float64) <= u).all() and (hi.astype(np.float64) > u).all()
    _, _, c_lo = fct.l1_sample(dev(lo), 1, seed, row_base=rb, capacity=16)
    assert int(c_lo.item()) == 0
    idx, w, c_hi = fct.l1_sample(dev(hi), 1, seed, row_base=rb, capacity=n)
    assert int(c_hi.item()) == n
    np.testing.assert_array_equal(idx.cpu().numpy(), rb + np.arange(n))


def test_sample_explicit_uniforms_and_capacity(fct):
    n, m = 50000, 3000
    p = _probs(n, 5, heavy=False)
    u = fctgen.uniforms(17, 0, n)
    idx, w, cnt = fct.l1_sample_u(dev(p), dev(u), m, capacity=100)
    oi, ow, oc = oracle.sample(p, m, u=u)
    c = int(cnt.item())
    assert c == oc > 100                                  # count is exact even when it exceeds capacity
    np.testing.assert_array_equal(idx.cpu().numpy()[:100], oi[:100])
    np.testing.assert_array_equal(w.cpu().numpy()[:100], ow[:100])
    # generator uniforms == the same uniforms passed explicitly
    a = fct.trim(*fct.l1_sample(dev(p), m, seed=17, capacity=2 * m + 64))
    b = fct.trim(*fct.l1_sample_u(dev(p), dev(u), m, capacity=2 * m + 64))
    np.testing.assert_array_equal(a[0].numpy(), b[0].numpy())


@pytest.mark.parametrize("n,m,row_base,cap", [(1, 1, 0, None), (2047, 100, 0, None), (2049, 100, 7, None),
                                              (300001, 4096, 123456, None), (1 << 20, 65536, 1 << 30, None),
                                              (50000, 3000, 5, 100)])
def test_probs_sample_fused_bit_exact(fct, n, m, row_base, cap):
    """Fused single-pass probabilities + sampling (decoupled look-back) == oracle probabilities and
    sampler bit for bit; == the unfused l1_probs -> l1_sample path."""
    rng = np.random.default_rng(n)
    lam = np.abs(rng.standard_cauchy(n)).astype(np.float32)
    lam[:2] = 0.0
    tot = np.array([lam.astype(np.float64).sum()])
    capacity = 2 * m + n // 10 + 64 if cap is None else cap
    p, idx, w, cnt = fct.l1_probs_sample(dev(lam), dev(tot), m, seed=3, row_base=row_base, capacity=capacity)
    p_o = (lam.astype(np.float64) / tot[0]).astype(np.float32)
    np.testing.assert_array_equal(p.cpu().numpy(), p_o)
    oi, ow, oc = oracle.sample(p_o, m, seed=3, row_base=row_base)
    c = int(cnt.item())
    assert c == oc
    k = min(c, capacity)
    np.testing.assert_array_equal(idx.cpu().numpy()[:k], oi[:k])
    np.testing.assert_array_equal(w.cpu().numpy()[:k], ow[:k])
    p2 = fct.l1_probs(dev(lam), dev(tot))
    i2, w2, c2 = fct.l1_sample(p2, m, seed=3, row_base=row_base, capacity=capacity)
    assert int(c2.item()) == c
    np.testing.assert_array_equal(i2.cpu().numpy()[:k], idx.cpu().numpy()[:k])


def test_sample_nan_probabilities_are_never_sampled(fct):
    """NaN p (e.g. after a conditioning failure) -> p_hat = 0 on both sides (R31); bit-exact."""
    p = np.abs(np.random.default_rng(8).standard_cauchy(5000)).astype(np.float32) * 1e-4
    p[::3] = np.nan
    p[7] = np.inf
    oi, ow, oc = oracle.sample(p, 300, seed=4)
    idx, w, cnt = fct.l1_sample(dev(p), 300, seed=4)
    gi, gw, gc = fct.trim(idx, w, cnt)
    assert gc == oc and not np.isnan(p[oi]).any()
    np.testing.assert_array_equal(gi.numpy(), oi)
    np.testing.assert_array_equal(gw.numpy(), ow)


# ---------------------------------------------------------------- whole pipeline vs oracle pipeline
@pytest.mark.parametrize("c", [1, 2])
def test_pipeline_end_to_end(fct, c):
    cfg = fctgen.CONFIGS[c]
    n = min(cfg.n, 64 * cfg.s)
    inp = fctgen.make_inputs(cfg, n=n)
    P = fct.Pipeline(n, cfg.d, cfg.s, cfg.r1, cfg.k, cfg.m, seed=11)
    P.run(dev(inp.A), dev(inp.signs), dev(inp.cauchy), dev(inp.hash), dev(inp.pi2))
    torch.cuda.synchronize()
    assert int(P.info.item()) == 0
    Yo, Mb = oracle.sketch(inp.A, inp.signs, inp.cauchy, inp.hash, cfg.s, cfg.r1)
    assert_sketch_close(P.Y.cpu().numpy().astype(np.float64), Yo, Mb)
    _, Rinv_o, _ = oracle.condition(Yo)
    lam_o, tot_o = oracle.rownorm(inp.A, Rinv_o, inp.pi2)
    lam = P.lam.cpu().numpy().astype(np.float64)
    # end-to-end (oracle's own R from its own fp64 Y): looser bound, DESIGN.md "Parity bar"
    assert (np.abs(lam - lam_o) <= 1e-3 * lam_o + 1e-30).all()
    p_o = oracle.probs(lam_o, tot_o)
    oi, ow, oc = oracle.sample(p_o.astype(np.float32), cfg.m, seed=11)
    gi, gw, gc = fct.trim(P.idx, P.weight, P.count)
    # decisions may differ only where u is within the probability discrepancy of phat
    u = fctgen.uniforms(11, 0, n)
    phat = np.minimum(1.0, cfg.m * P.p.cpu().numpy().astype(np.float64))
    diff = np.setxor1d(gi.numpy(), oi)
    assert all(abs(u[i] - phat[i]) <= 2e-3 * phat[i] for i in diff)
    # and the GPU's own decisions are exactly the Bernoulli rule on its p
    oi2, ow2, _ = oracle.sample(P.p.cpu().numpy(), cfg.m, seed=11)
    np.testing.assert_array_equal(gi.numpy(), oi2)
    np.testing.assert_array_equal(gw.numpy(), ow2)


def test_host_pipeline_matches_device_pipeline(fct):
    cfg = fctgen.CONFIGS[2]
    n = 32 * cfg.s
    inp = fctgen.make_inputs(cfg, n=n)
    H = fct.HostPipeline(n, cfg.d, cfg.s, cfg.r1, cfg.k, cfg.m, seed=5)
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
    hi, hw, hc = H.run(pin(inp.A), pin(inp.signs), pin(inp.cauchy), pin(inp.hash), pin(inp.pi2))
    P = fct.Pipeline(n, cfg.d, cfg.s, cfg.r1, cfg.k, cfg.m, seed=5)
    P.run(dev(inp.A), dev(inp.signs), dev(inp.cauchy), dev(inp.hash), dev(inp.pi2))
    di, dw, dc = fct.trim(P.idx, P.weight, P.count)
    # Y may differ bitwise between runs (shared-memory atomic order, reading R20), so p may
    # differ by an ulp: same rows up to ambiguous ones, weights equal to fp32-ulp level
    common, ih, idd = np.intersect1d(hi.numpy(), di.numpy(), return_indices=True)
    assert len(common) >= 0.99 * max(hc, dc)
    np.testing.assert_allclose(hw.numpy()[ih], dw.numpy()[idd], rtol=1e-5)
    u = fctgen.uniforms(5, 0, n)
    phat = np.minimum(1.0, cfg.m * P.p.cpu().numpy().astype(np.float64))
    assert all(abs(u[i] - phat[i]) <= 1e-5 * phat[i] for i in np.setxor1d(hi.numpy(), di.numpy()))


@pytest.mark.parametrize("c", [4, 5])
@pytest.mark.parametrize("direct", ["0", "1"])
def test_sketch_direct_aux_matches_too(fct, c, direct, monkeypatch):
    """K1 with the aux read through L2 (DIRECT, opt-in) and with the staged default."""
    monkeypatch.setenv("FCT_SKETCH_DIRECT", direct)
    cfg = fctgen.CONFIGS[c]
    inp = fctgen.make_inputs(cfg, n=9 * cfg.s + 5)
    Yo, Mb = oracle.sketch(inp.A, inp.signs, inp.cauchy, inp.hash, cfg.s, cfg.r1)
    assert_sketch_close(sketch_gpu(fct, inp), Yo, Mb)


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_sketch_generic_path_matches_too(fct, c, monkeypatch):
    """The generic (any s, d, lda) kernel stays parity-green: forced with FCT_SKETCH_GENERIC=1."""
    monkeypatch.setenv("FCT_SKETCH_GENERIC", "1")
    cfg = fctgen.CONFIGS[c]
    inp = fctgen.make_inputs(cfg, n=5 * cfg.s + 3)
    Yo, Mb = oracle.sketch(inp.A, inp.signs, inp.cauchy, inp.hash, cfg.s, cfg.r1)
    assert_sketch_close(sketch_gpu(fct, inp), Yo, Mb)


@pytest.mark.parametrize("c", [2, 4, 5])
def test_rownorm_simt_path_matches_too(fct, c, monkeypatch):
    """The SIMT row-norm kernel (fallback for unaligned / d > 128) stays parity-green."""
    monkeypatch.setenv("FCT_ROWNORM_SIMT", "1")
    cfg = fctgen.CONFIGS[c]
    inp = fctgen.make_inputs(cfg, n=2 * cfg.s)
    Rinv = _rinv_for(inp)
    B = fctgen.matrix(cfg.kind, cfg.seed, max(cfg.n, 5000), cfg.d, 0, 5000 + 7)
    lam_o, _ = oracle.rownorm(B, Rinv, inp.pi2)
    lam, _ = fct.l1_rownorm(dev(B), dev(Rinv), dev(inp.pi2))
    lam = lam.cpu().numpy().astype(np.float64)
    assert (np.abs(lam - lam_o) <= LAM_TOL * lam_o).all()


@pytest.mark.parametrize("env", ["FCT_ROWNORM_WS1", "FCT_ROWNORM_EG2", "FCT_ROWNORM_NOKEEP", "FCT_ROWNORM_STATIC", "FCT_ROWNORM_VAR=3",
                                 "FCT_ROWNORM_SS", "FCT_ROWNORM_SS FCT_ROWNORM_EG2", None])
@pytest.mark.parametrize("c", [2, 4, 5])
def test_rownorm_tc_variants(fct, c, env, monkeypatch):
    """Each tcgen05 row-norm variant (ws2 with 3 or 2 epilogue groups, the older ws) is parity-green,
    including special rows: zero, tiny (norm underflows in fp32), huge, and a row with exact ties."""
    for e in (env or "").split():
        k, _, v = e.partition("=")
        monkeypatch.setenv(k, v or "1")
    cfg = fctgen.CONFIGS[c]
    inp = fctgen.make_inputs(cfg, n=2 * cfg.s)
    Rinv = _rinv_for(inp)
    B = fctgen.matrix(cfg.kind, cfg.seed, max(cfg.n, 9000), cfg.d, 0, 9000 + 77)
    B[0] = 0.0
    B[1] *= np.float32(1e-20)
    B[2] *= np.float32(1e15)
    B[3] = 1.0
    B[4, ::3] = np.float32(3e-39)                   # subnormal entries (exact fp64 conversion path)
    lam_o, _ = oracle.rownorm(B, Rinv, inp.pi2)
    lam, _ = fct.l1_rownorm(dev(B), dev(Rinv), dev(inp.pi2))
    lam = lam.cpu().numpy().astype(np.float64)
    assert lam[0] == 0.0
    assert (np.abs(lam - lam_o) <= LAM_TOL * lam_o).all()


@pytest.mark.parametrize("c", [1, 3, 4, 5])
def test_sketch_hot_buckets(fct, c):
    """Adversarial hashes that put most H~-rows of every block into a handful of buckets: the shared-memory
    scatter contends constantly and every update must still land exactly once."""
    cfg = fctgen.CONFIGS[c]
    inp = fctgen.make_inputs(cfg, n=7 * cfg.s + 19)
    Yo, Mb = oracle.sketch(inp.A, inp.signs, inp.cauchy, inp.hash, cfg.s, cfg.r1)
    assert_sketch_close(sketch_gpu(fct, inp), Yo, Mb)
    hot = inp.hash.copy()
    hot[::2] %= 8                      # half of all H~-rows in 8 hot buckets
    hot[1::4] = 11 % cfg.r1            # a quarter in one bucket
    inp.hash = hot
    Yo2, Mb2 = oracle.sketch(inp.A, inp.signs, inp.cauchy, inp.hash, cfg.s, cfg.r1)
    assert_sketch_close(sketch_gpu(fct, inp), Yo2, Mb2)


# ---------------------------------------------------------------- NEXT-1: exact l1 row norms (tcgen05)
@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_rownorm_exact_configs(fct, c):
    """lambda_i = ||(A R^-1)_i||_1 on the tensor cores vs the fp64 oracle, with R^-1 from the oracle's own
    conditioning of the config's sketch.  Tolerance (derived from the arithmetic): 2^-14 times
    the magnitude sum_j sum_l |A_il||R^-1_lj| plus 2^-17 relative (fp32 sum over j).  Both the stacked
    (d <= 64) and the four-pass (d = 100) forms are covered; zero, tiny and huge rows included."""
    cfg = fctgen.CONFIGS[c]
    inp = fctgen.make_inputs(cfg, n=2 * cfg.s)
    Rinv = _rinv_for(inp)
    B = fctgen.matrix(cfg.kind, cfg.seed, max(cfg.n, 9000), cfg.d, 0, 9000 + 45)
    B[0] = 0.0
    B[1] *= np.float32(1e-20)
    B[2] *= np.float32(1e15)
    lam_o, tot_o, bnd = oracle.rownorm_exact(B, Rinv, with_bound=True)
    lam, tot = fct.l1_rownorm_exact(dev(B), dev(Rinv))
    lam = lam.cpu().numpy().astype(np.float64)
    err = np.abs(lam - lam_o)
    assert lam[0] == 0.0
    assert (err <= 2.0 ** -14 * bnd + 2.0 ** -17 * lam_o).all(), f"max err/bound {np.max(err / np.maximum(bnd, 1e-300)):.3e}"
    np.testing.assert_allclose(float(tot.item()), lam.sum(), rtol=1e-12)
    # the pure 1e-5 relative bar (north_star's lambda bar): fp32 accumulation cannot be certified to it, so the
    # fraction of rows above it is measured and bounded (reading R28); the worst relative error too
    rel = err / np.maximum(lam_o, 1e-300)
    fail = float(np.mean(rel[3:] > 1e-5))
    import json, os
    if os.path.isdir("gpurun_out"):
        with open("gpurun_out/rownorm_exact_rel.jsonl", "a") as f:
            f.write(json.dumps({"config": c, "rows": int(len(rel) - 3), "frac_over_1e-5": fail,
                                "max_rel": float(rel[3:].max()), "median_rel": float(np.median(rel[3:]))}) + "\n")
    assert fail <= EXACT_FAIL_FRAC[c], (fail, float(rel[3:].max()))
    assert rel[3:].max() <= EXACT_MAX_REL


def test_rownorm_exact_identity_and_errors(fct):
    rng = np.random.default_rng(4)
    A = rng.standard_normal((1000, 16)).astype(np.float32)
    lam, _ = fct.l1_rownorm_exact(dev(A), dev(np.eye(16)))
    np.testing.assert_allclose(lam.cpu().numpy(), np.abs(A.astype(np.float64)).sum(1), rtol=2e-6)
    # d % 4 != 0 and the SIMT form (also forced for d = 16) agree with the oracle too
    rng2 = np.random.default_rng(5)
    for dd, force in ((10, False), (16, True)):
        Rinv = np.triu(rng2.standard_normal((dd, dd))) + 2 * np.eye(dd)
        B = A[:, :dd].copy()
        lam_o, _, bnd = oracle.rownorm_exact(B, Rinv, with_bound=True)
        import os
        if force:
            os.environ["FCT_ROWNORM_SIMT"] = "1"
        try:
            lam, _ = fct.l1_rownorm_exact(dev(B), dev(Rinv))
        finally:
            os.environ.pop("FCT_ROWNORM_SIMT", None)
        err = np.abs(lam.cpu().numpy().astype(np.float64) - lam_o)
        assert (err <= 2.0 ** -14 * bnd + 2.0 ** -17 * lam_o).all()


# ---------------------------------------------------------------- NEXT-4: multinomial sampling (bit-exact)
@pytest.mark.parametrize("n,m,row_base", [(1, 5, 0), (2047, 100, 0), (2049, 1000, 9), (300001, 4096, 123456),
                                          (1 << 22, 65536, 1 << 30)])
def test_sample_multinomial_bit_exact(fct, n, m, row_base):
    rng = np.random.default_rng(n + m)
    p = np.abs(rng.standard_cauchy(n)).astype(np.float32)
    p[1::7] = 0.0
    if n > 3:
        p[2] = -1.0                     # negative / NaN entries count as zero probability on both sides
        p[3] = np.nan
    p[0] = max(p[0], 1e-3)
    idx, w, tot = fct.l1_sample_multinomial(dev(p), m, seed=21, row_base=row_base)
    oi, ow, oT, oF = oracle.sample_multinomial(p, m, seed=21, row_base=row_base)
    assert int(tot.item()) == oT
    np.testing.assert_array_equal(idx.cpu().numpy(), oi)
    np.testing.assert_array_equal(w.cpu().numpy(), ow)


def test_sample_multinomial_no_mass(fct):
    idx, w, tot = fct.l1_sample_multinomial(dev(np.zeros(100, np.float32)), 7, seed=1)
    assert int(tot.item()) == 0 and (idx.cpu().numpy() == -1).all() and (w.cpu().numpy() == 0).all()
