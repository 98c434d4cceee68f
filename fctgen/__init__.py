"""fctgen -- seeded synthetic inputs for the FCT1 hot path (shared by tests, bench and oracle checks).

Holds none of the method's arithmetic: it only draws A, the sign diagonal D, the Cauchy
diagonal C, the bucket indices of B, Pi2 and explicit sampling uniforms, each as a pure
function of (seed, stream, index).
The five named configurations mirror BASELINE.json ``configs``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libfctgen.so")
_lib = None

ST_A, ST_ROWMOD, ST_XSTAR, ST_NOISE, ST_SIGN, ST_CAUCHY, ST_HASH, ST_PI2, ST_SAMPLE = range(1, 10)


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-o", _SO, src, "-lm"])
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        u64, i64, i32, vp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
        lib.fg_mix64.restype = u64
        lib.fg_mix64.argtypes = [u64]
        lib.fg_rng_u64.restype = u64
        lib.fg_rng_u64.argtypes = [u64, u64, u64]
        lib.fg_rng_block.argtypes = [u64, u64, i64, i64, vp]
        lib.fg_signs.argtypes = [u64, i64, i64, vp]
        lib.fg_cauchy.argtypes = [u64, u64, i64, i64, vp]
        lib.fg_hash.restype = ctypes.c_int
        lib.fg_hash.argtypes = [u64, i64, i64, i32, vp]
        lib.fg_uniforms.argtypes = [u64, i64, i64, vp]
        lib.fg_normals.argtypes = [u64, u64, i64, i64, vp]
        lib.fg_matrix.restype = ctypes.c_int
        lib.fg_matrix.argtypes = [ctypes.c_int, u64, i64, i64, i64, i64, vp, i64]
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def mix64(z: int) -> int:
    return int(_L().fg_mix64(z & 0xFFFFFFFFFFFFFFFF))


def rng_u64(seed: int, stream: int, i: int) -> int:
    return int(_L().fg_rng_u64(seed, stream, i))


def rng_block(seed: int, stream: int, i0: int, count: int) -> np.ndarray:
    out = np.empty(count, np.uint64)
    _L().fg_rng_block(seed, stream, i0, count, _p(out))
    return out


def signs(seed: int, row0: int, count: int, out: np.ndarray | None = None) -> np.ndarray:
    out = np.empty(count, np.int8) if out is None else out
    _L().fg_signs(seed, row0, count, _p(out))
    return out


def cauchy(seed: int, stream: int, idx0: int, count: int, out: np.ndarray | None = None) -> np.ndarray:
    out = np.empty(count, np.float32) if out is None else out
    _L().fg_cauchy(seed, stream, idx0, count, _p(out))
    return out


def hashes(seed: int, idx0: int, count: int, r1: int, out: np.ndarray | None = None) -> np.ndarray:
    out = np.empty(count, np.int32) if out is None else out
    if _L().fg_hash(seed, idx0, count, r1, _p(out)) != 0:
        raise ValueError("r1 must be a power of two")
    return out


def uniforms(seed: int, row0: int, count: int) -> np.ndarray:
    out = np.empty(count, np.float64)
    _L().fg_uniforms(seed, row0, count, _p(out))
    return out


def normals(seed: int, stream: int, j0: int, count: int) -> np.ndarray:
    out = np.empty(count, np.float64)
    _L().fg_normals(seed, stream, j0, count, _p(out))
    return out


def matrix(kind: int, seed: int, n: int, d: int, row0: int = 0, nrows: int | None = None,
           out: np.ndarray | None = None) -> np.ndarray:
    nrows = n - row0 if nrows is None else nrows
    if out is None:
        out = np.empty((nrows, d), np.float32)
    assert out.dtype == np.float32 and out.flags.c_contiguous and out.shape[1] >= d
    if _L().fg_matrix(kind, seed, n, d, row0, nrows, _p(out), out.shape[1]) != 0:
        raise ValueError("bad matrix arguments")
    return out


@dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration."""
    idx: int
    n: int
    d: int
    s: int
    r1: int
    k: int
    m: int
    kind: int
    seed: int

    @property
    def n_pad(self) -> int:
        return -(-self.n // self.s) * self.s


CONFIGS = {
    1: Config(1, 1 << 14, 8, 64, 64, 16, 256, 1, 1),
    2: Config(2, 1 << 20, 16, 256, 256, 20, 4096, 2, 2),
    3: Config(3, 1 << 24, 32, 1024, 1024, 24, 16384, 3, 3),
    4: Config(4, 1 << 26, 64, 1024, 4096, 27, 65536, 4, 4),
    5: Config(5, 1 << 28, 100, 2048, 8192, 29, 1 << 18, 5, 5),
}


@dataclass
class Inputs:
    """Host-side inputs of one (possibly row-sliced) problem instance."""
    A: np.ndarray          # (rows, d) fp32
    signs: np.ndarray      # (rows_pad,) int8   (padded rows get +1; they multiply zero rows)
    cauchy: np.ndarray     # (2*rows_pad,) fp32, indexed by H~-row
    hash: np.ndarray       # (2*rows_pad,) int32, indexed by H~-row
    pi2: np.ndarray        # (d, k) fp32
    s: int
    r1: int
    k: int
    m: int
    seed: int
    row0: int


def make_inputs(cfg: Config, n: int | None = None, row0: int = 0, s: int | None = None,
                r1: int | None = None, k: int | None = None, d: int | None = None,
                seed: int | None = None, kind: int | None = None) -> Inputs:
    """Generate a row slice [row0, row0+n) of configuration ``cfg`` (overrides for tests).

    The aux arrays are generated for the s-aligned padded row range, indexed by the
    GLOBAL H~-row 2*row0 + t, so shards regenerate exactly the slice of the full problem.
    """
    s = cfg.s if s is None else s
    r1 = cfg.r1 if r1 is None else r1
    k = cfg.k if k is None else k
    d = cfg.d if d is None else d
    seed = cfg.seed if seed is None else seed
    kind = cfg.kind if kind is None else kind
    n = cfg.n - row0 if n is None else n
    n_total = max(cfg.n, row0 + n)
    assert row0 % s == 0
    n_pad = -(-n // s) * s
    A = matrix(kind, seed, n_total, d, row0, n)
    sg = np.ones(n_pad, np.int8)
    signs(seed, row0, n, sg[:n])
    c = cauchy(seed, ST_CAUCHY, 2 * row0, 2 * n_pad)
    h = hashes(seed, 2 * row0, 2 * n_pad, r1)
    pi2 = cauchy(seed, ST_PI2, 0, d * k).reshape(d, k)
    return Inputs(A, sg, c, h, pi2, s, r1, k, cfg.m, seed, row0)


# ---------------------------------------------------------------- NEXT-3: FCT2 inputs (Sec. 3.2)
ST_FCT2_SIGN, ST_FCT2_SEL, ST_FCT2_C = 10, 11, 12


@dataclass
class Fct2Inputs:
    signs_t: np.ndarray   # int8[t], the Rademacher D_t of the SRHT G (same G in every block)
    sel: np.ndarray       # int32[s], ascending distinct rows of H_t kept by R
    C: np.ndarray         # float32[r1, nb * s], i.i.d. standard Cauchy
    t: int
    s: int
    r1: int


def fct2_inputs(seed: int, n: int, t: int, s: int, r1: int) -> Fct2Inputs:
    """Seeded FCT2 randomness: D_t signs (top bit of the draw), R = the s smallest of t random keys (uniform
    s-subset), C Cauchy on its own stream indexed row-major r * (nb s) + j."""
    sg = np.where((rng_block(seed, ST_FCT2_SIGN, 0, t) >> np.uint64(63)) == 0, 1, -1).astype(np.int8)
    keys = rng_block(seed, ST_FCT2_SEL, 0, t)
    sel = np.sort(np.argsort(keys, kind="stable")[:s]).astype(np.int32)
    nb = -(-n // t)
    C = cauchy(seed, ST_FCT2_C, 0, r1 * nb * s).reshape(r1, nb * s)
    return Fct2Inputs(sg, sel, C, t, s, r1)
