"""GPU parity for NEXT-2 (coreset l1 regression, FastCauchyRegression steps 6-8).

  gather   Z = D X bit-exact against oracle.lad.coreset_rows (one fp64 product per entry on both sides)
  solve    objective f(x_gpu) (evaluated by the oracle in fp64) within 1e-8 relative of the LP optimum
           (oracle.lad, HiGHS dual simplex); the GPU's own f and gap reported in info agree with it.
           Tolerance from the stopping rule: the interior-point method stops at relative gap <= tol = 1e-10,
           the LP's feasibility tolerances are 1e-10, so 1e-8 leaves two orders of margin.  x is compared
           loosely (1e-5 relative to max(1, |x|)): the l1 optimum is unique for data in general position but
           the objective is flat along the optimal face to first order.
"""
import numpy as np
import pytest

import fctgen
import oracle
from oracle import lad as OL

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

F_TOL = 1e-8


@pytest.fixture(scope="module")
def fct():
    import paper_1207_4684_b200 as m
    from paper_1207_4684_b200 import build
    build.build()
    m.load()
    return m


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def planted(m, p, seed, outlier=0.05, scale_rows=True):
    """cfg-2-style planted l1 regression rows X = [A, -b] (fp32), b = A x* + noise with Cauchy outliers."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, p))
    if scale_rows:
        A *= rng.uniform(0.2, 5.0, (m, 1))
    b = A @ rng.standard_normal(p) + 0.1 * rng.standard_normal(m)
    out = rng.random(m) < outlier
    b[out] += 100 * rng.standard_cauchy(int(out.sum()))
    return np.concatenate([A, -b[:, None]], axis=1).astype(np.float32)


def solve_and_check(fct, Z_np, m_dev=None, tol=1e-10):
    Z = dev(Z_np)
    x, info = fct.l1_lad_solve(Z, m_dev, max_iter=200, tol=tol)
    x, info = x.cpu().numpy(), info.cpu().numpy()
    mm = int(info[6])
    xo, fo = OL.lad(Z_np[:mm])
    fg = OL.objective(Z_np[:mm], x)
    assert info[5] == 0, f"status {info[5]} after {info[3]} iterations, gap {info[2]:.3e}"
    assert fg <= fo * (1 + F_TOL) + 1e-300, f"f_gpu {fg!r} vs LP {fo!r}"
    assert fg >= fo * (1 - 1e-9)                    # cannot beat the optimum
    assert info[0] == pytest.approx(fg, rel=1e-12)  # the kernel's own objective at its x
    return x, xo, info


@pytest.mark.parametrize("m,p,seed", [(2000, 5, 0), (777, 1, 1), (4099, 15, 2), (3000, 63, 3), (2500, 99, 4),
                                      (1500, 127, 5), (40, 3, 6)])
def test_lad_matches_lp(fct, m, p, seed):
    Z = planted(m, p, seed).astype(np.float64)
    x, xo, info = solve_and_check(fct, Z)
    np.testing.assert_allclose(x, xo, rtol=0, atol=1e-5 * max(1.0, np.abs(xo).max()))


def test_lad_weighted_median(fct):
    """q = 2, Z_i = w_i [1, -b_i]: the weighted median (the p = 1 closed form)."""
    rng = np.random.default_rng(7)
    b = rng.standard_cauchy(1001)
    w = rng.uniform(1, 50, 1001)
    Z = np.stack([w, -w * b], axis=1)
    x, xo, info = solve_and_check(fct, Z)
    assert x[0] == pytest.approx(xo[0], rel=1e-7, abs=1e-9)


def test_lad_exact_fit_and_empty(fct):
    rng = np.random.default_rng(8)
    A = rng.standard_normal((500, 7))
    xs = rng.standard_normal(7)
    Z = np.concatenate([A, -(A @ xs)[:, None]], axis=1)
    x, info = fct.l1_lad_solve(dev(Z), None, max_iter=200)
    x, info = x.cpu().numpy(), info.cpu().numpy()
    assert info[5] == 0
    np.testing.assert_allclose(x, xs, rtol=0, atol=1e-7)
    # m = 0 rows: nothing to fit, converged, f = 0
    m0 = torch.zeros(1, dtype=torch.int64, device="cuda")
    x, info = fct.l1_lad_solve(dev(Z), m0)
    info = info.cpu().numpy()
    assert info[5] == 0 and info[0] == 0.0 and info[6] == 0


def test_lad_rank_deficient_and_wide_weights(fct):
    """A duplicated column (rank-deficient coreset: collapsed Cholesky pivots, non-unique x) and Horvitz-Thompson
    weights spanning 1 .. 1e6: the objective still reaches the LP optimum."""
    rng = np.random.default_rng(11)
    X = planted(3000, 6, 12).astype(np.float64)
    Z = np.concatenate([X[:, :3], X[:, :1], X[:, 3:]], axis=1)       # column 0 repeated
    Z *= np.exp(rng.uniform(0, np.log(1e6), (Z.shape[0], 1)))       # row weights 1 .. 1e6
    Zd = dev(Z)
    x, info = fct.l1_lad_solve(Zd, None, max_iter=200)
    x, info = x.cpu().numpy(), info.cpu().numpy()
    _, fo = OL.lad(Z)
    fg = OL.objective(Z, x)
    assert info[5] == 0 and info[7] >= 1       # converged, a pivot collapsed
    assert fo * (1 - 1e-9) <= fg <= fo * (1 + F_TOL)


def test_lad_count_prefix_and_clamp(fct):
    """m on the device selects a prefix of the capacity rows; m > capacity is clamped."""
    Z = planted(3000, 8, 9).astype(np.float64)
    m = torch.tensor([1234], dtype=torch.int64, device="cuda")
    _, _, info = solve_and_check(fct, Z, m)
    assert info[6] == 1234
    m = torch.tensor([10 ** 9], dtype=torch.int64, device="cuda")
    _, _, info = solve_and_check(fct, Z, m)
    assert info[6] == 3000


def test_gather_bit_exact_and_out_of_range(fct):
    rng = np.random.default_rng(10)
    n, q = 5000, 17
    X = rng.standard_normal((n, q)).astype(np.float32)
    row_base = 100000
    idx = np.sort(rng.choice(n, 700, replace=False)).astype(np.int64) + row_base
    w = 1.0 / rng.uniform(1e-4, 1.0, 700)
    cnt = torch.tensor([650], dtype=torch.int64, device="cuda")
    Z = fct.l1_coreset_gather(dev(X), dev(idx), dev(w), cnt, row_base=row_base).cpu().numpy()
    np.testing.assert_array_equal(Z[:650], OL.coreset_rows(X, idx[:650], w[:650], row_base))
    # an index outside the shard gives a NaN row (loud), the others are untouched
    bad = idx.copy()
    bad[3] = row_base + n
    Z = fct.l1_coreset_gather(dev(X), dev(bad), dev(w), None, row_base=row_base).cpu().numpy()
    assert np.isnan(Z[3]).all() and np.isfinite(np.delete(Z, 3, axis=0)).all()
    x, info = fct.l1_lad_solve(dev(Z), None)
    assert info.cpu().numpy()[5] == 2


def test_errors(fct):
    Z = torch.zeros((10, 129), dtype=torch.float64, device="cuda")
    with pytest.raises(fct.FctError):
        fct.l1_lad_solve(Z)
    with pytest.raises(fct.FctError):
        fct.l1_lad_solve(torch.zeros((10, 1), dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("sampler", ["bernoulli", "multinomial"])
def test_coreset_regression_after_pipeline(fct, sampler):
    """cfg 2 (planted l1 regression, last column -b): the full path -> sample -> gather -> solve, against the
    oracle's gather + LP on the same idx / weight."""
    cfg = fctgen.CONFIGS[2]
    n = 256 * cfg.s
    inp = fctgen.make_inputs(cfg, n=n)
    P = fct.Pipeline(n, cfg.d, cfg.s, cfg.r1, cfg.k, cfg.m, seed=3)
    Xd = dev(inp.A)
    P.run(Xd, dev(inp.signs), dev(inp.cauchy), dev(inp.hash), dev(inp.pi2))
    if sampler == "bernoulli":
        idx, w, cnt = P.idx, P.weight, P.count
    else:
        idx, w, _ = fct.l1_sample_multinomial(P.p, cfg.m, seed=3)
        cnt = torch.tensor([cfg.m], dtype=torch.int64, device="cuda")
    x, info = fct.l1_coreset_regression(Xd, idx, w, cnt)
    c = int(cnt.item())
    x, info = x.cpu().numpy(), info.cpu().numpy()
    assert info[5] == 0 and info[6] == c
    xo, fo, Zo = OL.coreset_regression(inp.A, idx.cpu().numpy()[:c], w.cpu().numpy()[:c])
    fg = OL.objective(Zo, x)
    assert fo * (1 - 1e-9) <= fg <= fo * (1 + F_TOL)
    # the coreset solution is a good solution of the full problem (Thm P:L2955-2980): compare with the full
    # LAD optimum on all n rows (oracle LP)
    xf, ff = OL.lad(inp.A.astype(np.float64))
    f_hat = OL.objective(inp.A.astype(np.float64), x)
    assert f_hat <= 1.05 * ff
