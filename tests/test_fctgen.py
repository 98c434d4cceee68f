"""Input generators: determinism, shard-regenerability, distributions (no method arithmetic)."""
import os

import numpy as np
import pytest
from scipy import stats

import fctgen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
G = 0x9E3779B97F4A7C15
MASK = (1 << 64) - 1


def _golden_splitmix():
    vals = []
    with open(os.path.join(GOLDEN, "splitmix64_state0.txt")) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                vals.append(int(line, 16))
    return vals


def test_mix64_matches_splitmix64_reference():
    want = _golden_splitmix()
    got = [fctgen.mix64((k * G) & MASK) for k in range(1, len(want) + 1)]
    assert got == want


def test_rng_definition_and_oracle_copy_agree():
    # rng_u64(seed, stream, i) = mix64(mix64(seed + G(stream+1)) + G(i+1))
    for seed, stream, i in [(0, 0, 0), (1, 9, 12345), (5, 6, 2**40 + 7), (2**63 + 11, 3, 99)]:
        key = fctgen.mix64((seed + G * (stream + 1)) & MASK)
        want = fctgen.mix64((key + G * (i + 1)) & MASK)
        assert fctgen.rng_u64(seed, stream, i) == want
        assert oracle.rng_u64(seed, stream, i) == want      # the oracle's own copy


def test_block_equals_scalar_and_slices_regenerate():
    blk = fctgen.rng_block(7, 9, 1000, 64)
    assert [int(x) for x in blk[:5]] == [fctgen.rng_u64(7, 9, 1000 + t) for t in range(5)]
    full = fctgen.make_inputs(fctgen.CONFIGS[1], n=4096, s=64, r1=64)
    half = fctgen.make_inputs(fctgen.CONFIGS[1], n=2048, row0=2048, s=64, r1=64)
    np.testing.assert_array_equal(full.A[2048:], half.A)
    np.testing.assert_array_equal(full.signs[2048:], half.signs)
    np.testing.assert_array_equal(full.cauchy[4096:], half.cauchy)
    np.testing.assert_array_equal(full.hash[4096:], half.hash)


def test_value_distributions():
    c = fctgen.cauchy(3, fctgen.ST_CAUCHY, 0, 20000).astype(np.float64)
    assert stats.kstest(c, "cauchy").pvalue > 1e-3
    h = fctgen.hashes(3, 0, 64000, 64)
    assert h.min() == 0 and h.max() == 63
    assert stats.chisquare(np.bincount(h, minlength=64)).pvalue > 1e-3
    sg = fctgen.signs(3, 0, 20000)
    assert set(np.unique(sg)) == {-1, 1} and abs(sg.mean()) < 0.05
    z = fctgen.normals(3, 1, 0, 20000)
    assert stats.kstest(z, "norm").pvalue > 1e-3
    u = fctgen.uniforms(3, 0, 20000)
    assert u.min() >= 0 and u.max() < 1 and stats.kstest(u, "uniform").pvalue > 1e-3


@pytest.mark.parametrize("kind", [1, 2, 3, 4, 5])
def test_matrix_kinds(kind):
    cfg = fctgen.CONFIGS[kind]
    d = min(cfg.d, 16)
    A = fctgen.matrix(kind, cfg.seed, 1 << 20, d, 0, 4096)
    assert A.shape == (4096, d) and np.isfinite(A).all()
    if kind == 4:
        big = (np.abs(A).max(axis=1) > 100).mean()
        assert 0.003 < big < 0.02
    if kind in (2, 5):
        # last column is -b with b = F x* + e: the residual -(A[:, -1]) - F x* is the noise
        xs = fctgen.normals(cfg.seed, fctgen.ST_XSTAR, 0, d - 1)
        e = -A[:, -1].astype(np.float64) - A[:, :-1].astype(np.float64) @ xs
        assert np.median(np.abs(e)) < (0.2 if kind == 2 else 2.0)
