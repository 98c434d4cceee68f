"""GPU parity for NEXT-3, the FCT2 sketch (Sec. 3.2), through the C ABI (fct2_sketch) against oracle.fct2.

Tolerance (DESIGN.md NEXT-3): entrywise |Y - Y_o| <= 1e-5 * Mbound, Mbound = kappa |C| |H~| |A|, the same form as
FCT1's north_star bound.  The GPU forms Z = H~ A in fp32 (log2 t butterfly stages, each rounding relative to the
magnitude bound) and accumulates C Z in fp32 partials of 256 terms folded into fp64, so the error stays orders of
magnitude inside it.
"""
import numpy as np
import pytest

import fctgen
from oracle import fct2 as F

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fct():
    import paper_1207_4684_b200 as m
    from paper_1207_4684_b200 import build
    build.build()
    m.load()
    return m


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def run(fct, A, inp):
    Y = fct.fct2_sketch(dev(A), dev(inp.signs_t), dev(inp.sel), dev(inp.C), inp.t, inp.s, inp.r1)
    return Y.cpu().numpy().astype(np.float64)


def check(Yg, Yo, Mb, tol=1e-5):
    err = np.abs(Yg - Yo)
    assert (err <= tol * Mb + 1e-30).all(), (err / np.maximum(Mb, 1e-300)).max()


@pytest.fixture(params=["tc", "simt"])
def path(request, monkeypatch):
    """The tcgen05 3xTF32 contraction (default) and the SIMT one (FCT2_SIMT=1)."""
    if request.param == "simt":
        monkeypatch.setenv("FCT2_SIMT", "1")
    return request.param


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_fct2_config_shapes(fct, c, path):
    """Each BASELINE config's matrix family and d with the paper's FCT2 parameters (s, t, r1) = params(d),
    3 blocks plus a ragged tail."""
    cfg = fctgen.CONFIGS[c]
    s, t, r1 = F.params(cfg.d)
    n = 3 * t + 37
    A = fctgen.matrix(cfg.kind, cfg.seed, max(cfg.n, n), cfg.d, 0, n)
    inp = fctgen.fct2_inputs(cfg.seed, n, t, s, r1)
    Yo, Mb = F.sketch(A, inp.signs_t, inp.sel, inp.C, t, s, r1)
    check(run(fct, A, inp), Yo, Mb)


@pytest.mark.parametrize("n,d,t,s,r1", [(1, 1, 1, 1, 1), (5, 3, 8, 8, 4), (100, 7, 64, 1, 9), (64, 2, 64, 64, 3),
                                        (1000, 65, 256, 17, 130), (2049, 9, 2048, 100, 70), (40000, 4, 32768, 50, 8)])
def test_fct2_edges(fct, n, d, t, s, r1, path):
    """n < t (one partial block), t = 1, s = t (orthogonal G), s = 1, d > 64 (two output tiles), t = 32768."""
    rng = np.random.default_rng(n + d + t)
    A = rng.standard_normal((n, d)).astype(np.float32)
    inp = fctgen.fct2_inputs(7, n, t, s, r1)
    Yo, Mb = F.sketch(A, inp.signs_t, inp.sel, inp.C, t, s, r1)
    check(run(fct, A, inp), Yo, Mb)


def test_fct2_strided_and_padded_C(fct, path):
    """lda > d and ldc > nb s (C with padding columns that must be ignored)."""
    rng = np.random.default_rng(3)
    n, d, t, s, r1 = 3000, 6, 512, 40, 33
    Afull = rng.standard_normal((n, 10)).astype(np.float32)
    inp = fctgen.fct2_inputs(2, n, t, s, r1)
    Cpad = np.full((r1, inp.C.shape[1] + 5), 1e30, np.float32)
    Cpad[:, :inp.C.shape[1]] = inp.C
    Yo, Mb = F.sketch(Afull[:, :d], inp.signs_t, inp.sel, inp.C, t, s, r1)
    Ad = dev(Afull)[:, :d]
    Y = fct.fct2_sketch(Ad, dev(inp.signs_t), dev(inp.sel), dev(Cpad)[:, :inp.C.shape[1]], t, s, r1)
    check(Y.cpu().numpy().astype(np.float64), Yo, Mb)


def test_fct2_errors(fct):
    A = torch.zeros((10, 2), dtype=torch.float32, device="cuda")
    sg = torch.ones(12, dtype=torch.int8, device="cuda")
    sel = torch.arange(4, dtype=torch.int32, device="cuda")
    C = torch.zeros((3, 8), dtype=torch.float32, device="cuda")
    with pytest.raises(fct.FctError, match="power of two"):
        fct.fct2_sketch(A, sg, sel, C, 12, 4, 3)                 # t not a power of two
    with pytest.raises(fct.FctError):
        fct.fct2_sketch(A, sg, sel, C, 8, 9, 3)                  # s > t
    with pytest.raises(fct.FctError, match="ldc"):
        fct.fct2_sketch(A, sg, sel, C[:, :7].contiguous(), 8, 4, 3)   # ldc = 7 < nb s = 2 * 4
