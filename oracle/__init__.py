"""oracle -- TEST INFRASTRUCTURE ONLY: the plain fp64 CPU oracle of the FCT1 hot path.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may
import this package.  It shares no code with paper_1207_4684_b200 (the CUDA path).

  sketch(...)     O1  Y = 4 B C H~ D A   (C, explicit Hadamard)      -> oracle.c
  dense_sketch    O1-dense: materialised B, C, H~, D (numpy, tiny n)             -> dense.py
  condition(Y)    O2  Householder QR of Y = Pi1 A, diag(R) > 0, R^-1
  rownorm(...)    O3  lambda_i = median_j |(A R^-1 Pi2)_ij|   P:L2921-2938        -> oracle.c
  rownorm_exact   NEXT-1  lambda_i = ||(A R^-1)_i||_1 (exact row norms) -> oracle.c
  probs(...)          p_i = lambda_i / sum lambda   (t_i of P:L2028-2033)
  sample(...)     O4  Bernoulli l1 sampling   P:L1258-1268                        -> oracle.c
  sample_multinomial  NEXT-4  m i.i.d. draws from an exact fixed-point CDF          -> oracle.c
  lad.coreset_regression  NEXT-2  x_hat = argmin ||D(Ax - b)||_1 (LP)  -> lad.py
  fct2.sketch     NEXT-3  Pi1 A = (8/r1) sqrt(pi t/2s) C H~ A, SRHT blocks (Sec. 3.2)  -> fct2.py
Parity-unpinned items are listed in DESIGN.md ("Oracle pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, src, "-lm"])
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, i32, vp, u64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_uint64
        lib.or_rng_u64.restype = u64
        lib.or_rng_u64.argtypes = [u64, u64, u64]
        lib.or_num_threads.restype = ctypes.c_int
        lib.or_sketch.restype = ctypes.c_int
        lib.or_sketch.argtypes = [vp, i64, i64, i64, vp, vp, vp, i32, i32, i64, i64, vp, vp]
        lib.or_rownorm.restype = ctypes.c_int
        lib.or_rownorm.argtypes = [vp, i64, i64, i64, vp, vp, i32, vp, vp, vp]
        lib.or_rownorm_exact.restype = ctypes.c_int
        lib.or_rownorm_exact.argtypes = [vp, i64, i64, i64, vp, vp, vp, vp]
        lib.or_sample_multinomial.restype = u64
        lib.or_sample_multinomial.argtypes = [vp, i64, i64, u64, i64, vp, vp, vp]
        lib.or_sample.restype = i64
        lib.or_sample.argtypes = [vp, vp, i64, i64, i64, u64, vp, vp, i64]
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def num_threads() -> int:
    return int(_L().or_num_threads())


def rng_u64(seed: int, stream: int, i: int) -> int:
    return int(_L().or_rng_u64(seed, stream, i))


def sketch(A: np.ndarray, signs: np.ndarray, cauchy: np.ndarray, hash_rows: np.ndarray, s: int, r1: int,
           blocks: tuple[int, int] | None = None, with_bound: bool = True):
    """O1: (Y, Mbound) in fp64, Y = 4 B C H~ D A (Sec. 3.1)."""
    A = np.ascontiguousarray(A, np.float32)
    n, d = A.shape
    n_pad = -(-n // s) * s
    assert signs.shape[0] >= n and cauchy.shape[0] >= 2 * n_pad and hash_rows.shape[0] >= 2 * n_pad
    signs = np.ascontiguousarray(signs, np.int8)
    cauchy = np.ascontiguousarray(cauchy, np.float32)
    hash_rows = np.ascontiguousarray(hash_rows, np.int32)
    Y = np.zeros((r1, d), np.float64)
    M = np.zeros((r1, d), np.float64) if with_bound else None
    b0, b1 = (0, -1) if blocks is None else blocks
    rc = _L().or_sketch(_p(A), n, d, d, _p(signs), _p(cauchy), _p(hash_rows), s, r1, b0, b1, _p(Y), _p(M))
    if rc != 0:
        raise ValueError(f"or_sketch failed ({rc})")
    return (Y, M) if with_bound else Y


def condition(Y: np.ndarray, Pi2: np.ndarray | None = None):
    """O2: R with Y = QR (Householder, LAPACK geqrf via numpy), diag(R) > 0, Rinv, M = Rinv Pi2.

    FastL1Basis: "construct Pi1 A and an R such that Pi1 A = QR";
    diag(R) > 0 makes R unique (reading R19).  Returns (R, Rinv, M or None).
    """
    Y = np.asarray(Y, np.float64)
    R = np.linalg.qr(Y, mode="r")
    sgn = np.where(np.diag(R) < 0, -1.0, 1.0)
    R = sgn[:, None] * R
    d = R.shape[0]
    Rinv = np.linalg.solve(R, np.eye(d))          # upper-triangular inverse
    Rinv = np.triu(Rinv)
    M = None if Pi2 is None else Rinv @ np.asarray(Pi2, np.float64)
    return R, Rinv, M


def rownorm(A: np.ndarray, Rinv: np.ndarray, Pi2: np.ndarray, with_bound: bool = False):
    """O3: lambda (fp64), sum lambda, [bound] -- P:L2921-2938, M = Rinv Pi2 formed first."""
    A = np.ascontiguousarray(A, np.float32)
    n, d = A.shape
    Rinv = np.ascontiguousarray(Rinv, np.float64)
    Pi2 = np.ascontiguousarray(Pi2, np.float32)
    k = Pi2.shape[1]
    lam = np.empty(n, np.float64)
    tot = np.zeros(1, np.float64)
    bnd = np.empty(n, np.float64) if with_bound else None
    rc = _L().or_rownorm(_p(A), n, d, d, _p(Rinv), _p(Pi2), k, _p(lam), _p(tot), _p(bnd))
    if rc != 0:
        raise ValueError("or_rownorm failed")
    return (lam, float(tot[0]), bnd) if with_bound else (lam, float(tot[0]))


def rownorm_exact(A: np.ndarray, Rinv: np.ndarray, with_bound: bool = False):
    """NEXT-1: exact l1 row norms lambda_i = ||(A R^-1)_i||_1 (fp64), sum, [bound_i = sum_j sum_l |A_il||Rinv_lj|]
    -- the row norms the paper's Sec. 6.2 experiments compute exactly."""
    A = np.ascontiguousarray(A, np.float32)
    n, d = A.shape
    Rinv = np.ascontiguousarray(Rinv, np.float64)
    lam = np.empty(n, np.float64)
    tot = np.zeros(1, np.float64)
    bnd = np.empty(n, np.float64) if with_bound else None
    rc = _L().or_rownorm_exact(_p(A), n, d, d, _p(Rinv), _p(lam), _p(tot), _p(bnd))
    if rc != 0:
        raise ValueError("or_rownorm_exact failed")
    return (lam, float(tot[0]), bnd) if with_bound else (lam, float(tot[0]))


def probs(lam: np.ndarray, total: float) -> np.ndarray:
    """p_i = lambda_i / sum_j lambda_j in fp64 (t_i of P:L2028-2033, reading R12)."""
    if not total > 0:
        raise ValueError("sum of lambda must be positive")
    return np.asarray(lam, np.float64) / total


def sample(p32: np.ndarray, m: int, seed: int = 0, row_base: int = 0, u: np.ndarray | None = None,
           capacity: int | None = None):
    """O4: Bernoulli l1 sampling from fp32 probabilities. Returns (idx, weight, count)."""
    p32 = np.ascontiguousarray(p32, np.float32)
    n = p32.shape[0]
    cap = n if capacity is None else capacity
    idx = np.empty(max(cap, 1), np.int64)
    w = np.empty(max(cap, 1), np.float64)
    if u is not None:
        u = np.ascontiguousarray(u, np.float64)
        assert u.shape[0] == n
    cnt = int(_L().or_sample(_p(p32), _p(u), n, row_base, m, seed, _p(idx), _p(w), cap))
    k = min(cnt, cap)
    return idx[:k].copy(), w[:k].copy(), cnt


def sample_multinomial(p32: np.ndarray, m: int, seed: int = 0, row_base: int = 0):
    """NEXT-4: m i.i.d. draws proportional to fp32 p from an exact fixed-point CDF (bit-exact integer
    arithmetic; see oracle.c). Returns (idx[m], weight[m], T, F)."""
    p32 = np.ascontiguousarray(p32, np.float32)
    n = p32.shape[0]
    idx = np.empty(max(m, 1), np.int64)
    w = np.empty(max(m, 1), np.float64)
    F = np.zeros(1, np.int32)
    T = int(_L().or_sample_multinomial(_p(p32), n, m, seed, row_base, _p(idx), _p(w), _p(F)))
    if T == 0:
        raise ValueError("no positive probability")
    return idx[:m].copy(), w[:m].copy(), T, int(F[0])
