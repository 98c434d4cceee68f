"""Thin Python binding of libfct.so (include/fct.h) for torch CUDA tensors.

Argument marshalling only: every step of the path runs in the CUDA kernels behind the C ABI.
Functions keep the C names.  All work is enqueued on torch's current CUDA stream.
"""
from __future__ import annotations

import torch

from . import _lib

_WS: dict[tuple, torch.Tensor] = {}


def _lib_():
    return _lib.load()


def _stream():
    return ctypes_ptr(torch.cuda.current_stream().cuda_stream)


def ctypes_ptr(x: int):
    import ctypes
    return ctypes.c_void_p(x)


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes_ptr(t.data_ptr())


def _need(t: torch.Tensor, dtype, name: str, dev=True):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if dev and not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def workspace(nbytes: int, tag: str = "default", device=None) -> torch.Tensor:
    """A cached device byte buffer of at least nbytes, re-used across calls with the same tag, device and
    current stream (calls enqueued on different streams never share scratch memory)."""
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    key = (tag, device.index, torch.cuda.current_stream(device).cuda_stream)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf


def fct_sketch(A, signs, cauchy_diag, hash_rows, s: int, r1: int, Y=None, accumulate: bool = False,
               ws: torch.Tensor | None = None):
    """Y = [Y +] 4 B C H~ D A  (Sec. 3.1).  A: (n, d) fp32 CUDA (row stride = lda)."""
    L = _lib_()
    _need(signs, torch.int8, "signs")
    _need(cauchy_diag, torch.float32, "cauchy_diag")
    _need(hash_rows, torch.int32, "hash_rows")
    if A.dtype != torch.float32 or not A.is_cuda or A.dim() != 2 or A.stride(1) != 1:
        raise ValueError("A must be a 2-D fp32 CUDA tensor with unit column stride")
    n, d = A.shape
    lda = A.stride(0)
    n_pad = -(-n // s) * s
    if signs.numel() < n or cauchy_diag.numel() < 2 * n_pad or hash_rows.numel() < 2 * n_pad:
        raise ValueError("aux arrays too short (signs[n], cauchy/hash[2n'])")
    if Y is None:
        Y = torch.empty((r1, d), dtype=torch.float32, device=A.device)
        accumulate = False
    _need(Y, torch.float32, "Y")
    nb = L.fct_sketch_workspace_bytes(n, d, s, r1)
    ws = workspace(nb, "sketch") if ws is None else ws
    _lib.check(L.fct_sketch(_ptr(A), n, d, lda, _ptr(signs), _ptr(cauchy_diag), _ptr(hash_rows), s, r1, _ptr(Y),
                            int(bool(accumulate)), _ptr(ws), ws.numel(), _stream()))
    return Y


def fct_condition(Y, check: bool = True):
    """(R, Rinv, info) with Y = QR, diag(R) > 0 (CholeskyQR2, fp64; shifted CholeskyQR3 fallback on the device,
    info = -1).  check=True syncs and raises when even the fallback failed (info > 0)."""
    L = _lib_()
    _need(Y, torch.float32, "Y")
    r1, d = Y.shape
    R = torch.empty((d, d), dtype=torch.float64, device=Y.device)
    Rinv = torch.empty_like(R)
    info = torch.zeros(1, dtype=torch.int32, device=Y.device)
    nb = L.fct_condition_workspace_bytes(r1, d)
    ws = workspace(nb, "condition")
    _lib.check(L.fct_condition(_ptr(Y), r1, d, _ptr(R), _ptr(Rinv), _ptr(info), _ptr(ws), ws.numel(), _stream()))
    if check:
        v = int(info.item())
        if v > 0:
            raise _lib.FctError(-5, f"Cholesky pivot {v} not positive even with the shifted fallback (non-finite Y)")
    return R, Rinv, info


def l1_rownorm(A, Rinv, Pi2, lam=None, lambda_sum=None):
    """lambda_i = median_j |(A Rinv Pi2)_ij| (fp32); lambda_sum (fp64 device scalar) += sum lambda."""
    L = _lib_()
    if A.dtype != torch.float32 or not A.is_cuda or A.dim() != 2 or A.stride(1) != 1:
        raise ValueError("A must be a 2-D fp32 CUDA tensor with unit column stride")
    _need(Rinv, torch.float64, "Rinv")
    _need(Pi2, torch.float32, "Pi2")
    n, d = A.shape
    k = Pi2.shape[1]
    lam = torch.empty(n, dtype=torch.float32, device=A.device) if lam is None else lam
    if lambda_sum is None:
        lambda_sum = torch.zeros(1, dtype=torch.float64, device=A.device)
    nb = L.l1_rownorm_workspace_bytes(n, d, k)
    ws = workspace(nb, "rownorm")
    _lib.check(L.l1_rownorm(_ptr(A), n, d, A.stride(0), _ptr(Rinv), _ptr(Pi2), k, _ptr(lam), _ptr(lambda_sum),
                            _ptr(ws), ws.numel(), _stream()))
    return lam, lambda_sum


def l1_rownorm_exact(A, Rinv, lam=None, lambda_sum=None):
    """NEXT-1: exact l1 row norms lambda_i = ||(A Rinv)_i||_1 (fp32) and their fp64 sum."""
    L = _lib_()
    if A.dtype != torch.float32 or not A.is_cuda or A.dim() != 2 or A.stride(1) != 1:
        raise ValueError("A must be a 2-D fp32 CUDA tensor with unit column stride")
    _need(Rinv, torch.float64, "Rinv")
    n, d = A.shape
    lam = torch.empty(n, dtype=torch.float32, device=A.device) if lam is None else lam
    lambda_sum = torch.zeros(1, dtype=torch.float64, device=A.device) if lambda_sum is None else lambda_sum
    nb = L.l1_rownorm_exact_workspace_bytes(n, d)
    ws = workspace(nb, "rownorm_exact")
    _lib.check(L.l1_rownorm_exact(_ptr(A), n, d, A.stride(0), _ptr(Rinv), _ptr(lam), _ptr(lambda_sum), _ptr(ws),
                                  ws.numel(), _stream()))
    return lam, lambda_sum


def l1_probs(lam, lambda_total, p=None):
    L = _lib_()
    _need(lam, torch.float32, "lambda")
    _need(lambda_total, torch.float64, "lambda_total")
    p = torch.empty_like(lam) if p is None else p
    _lib.check(L.l1_probs(_ptr(lam), lam.numel(), _ptr(lambda_total), _ptr(p), _stream()))
    return p


def l1_rownorm_probs(A, Rinv, Pi2):
    """(lambda, p, total) on one device."""
    L = _lib_()
    n, d = A.shape
    k = Pi2.shape[1]
    lam = torch.empty(n, dtype=torch.float32, device=A.device)
    p = torch.empty_like(lam)
    tot = torch.zeros(1, dtype=torch.float64, device=A.device)
    _need(Rinv, torch.float64, "Rinv")
    _need(Pi2, torch.float32, "Pi2")
    nb = L.l1_rownorm_workspace_bytes(n, d, k)
    ws = workspace(nb, "rownorm")
    _lib.check(L.l1_rownorm_probs(_ptr(A), n, d, A.stride(0), _ptr(Rinv), _ptr(Pi2), k, _ptr(lam), _ptr(p),
                                  _ptr(tot), _ptr(ws), ws.numel(), _stream()))
    return lam, p, tot


def _sample(p, m, seed, row_base, capacity, u):
    L = _lib_()
    _need(p, torch.float32, "p")
    n = p.numel()
    cap = 2 * m + 64 if capacity is None else capacity
    idx = torch.empty(max(cap, 1), dtype=torch.int64, device=p.device)
    w = torch.empty(max(cap, 1), dtype=torch.float64, device=p.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=p.device)
    nb = L.l1_sample_workspace_bytes(n)
    ws = workspace(nb, "sample")
    if u is None:
        rc = L.l1_sample(_ptr(p), n, row_base, m, seed & 0xFFFFFFFFFFFFFFFF, _ptr(idx), _ptr(w), cap, _ptr(cnt),
                         _ptr(ws), ws.numel(), _stream())
    else:
        _need(u, torch.float64, "u")
        rc = L.l1_sample_u(_ptr(p), _ptr(u), n, row_base, m, _ptr(idx), _ptr(w), cap, _ptr(cnt), _ptr(ws),
                           ws.numel(), _stream())
    _lib.check(rc)
    return idx, w, cnt


def l1_sample(p, m: int, seed: int, row_base: int = 0, capacity: int | None = None):
    """Bernoulli l1 sampling. Returns (idx[capacity], weight[capacity], count[1]) device tensors."""
    return _sample(p, m, seed, row_base, capacity, None)


def l1_sample_u(p, u, m: int, row_base: int = 0, capacity: int | None = None):
    return _sample(p, m, 0, row_base, capacity, u)


def l1_probs_sample(lam, lambda_total, m: int, seed: int, row_base: int = 0, capacity: int | None = None):
    """Fused probabilities + Bernoulli sampling (one pass over lambda).
    Returns (p, idx[capacity], weight[capacity], count[1]) device tensors."""
    L = _lib_()
    _need(lam, torch.float32, "lambda")
    _need(lambda_total, torch.float64, "lambda_total")
    n = lam.numel()
    cap = 2 * m + 64 if capacity is None else capacity
    p = torch.empty_like(lam)
    idx = torch.empty(max(cap, 1), dtype=torch.int64, device=lam.device)
    w = torch.empty(max(cap, 1), dtype=torch.float64, device=lam.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=lam.device)
    nb = L.l1_probs_sample_workspace_bytes(n)
    ws = workspace(nb, "probs_sample")
    _lib.check(L.l1_probs_sample(_ptr(lam), n, _ptr(lambda_total), row_base, m, seed & 0xFFFFFFFFFFFFFFFF, _ptr(p),
                                 _ptr(idx), _ptr(w), cap, _ptr(cnt), _ptr(ws), ws.numel(), _stream()))
    return p, idx, w, cnt


def l1_sample_multinomial(p, m: int, seed: int, row_base: int = 0):
    """NEXT-4: exactly m i.i.d. draws proportional to p (exact fixed-point CDF).
    Returns (idx[m] int64, weight[m] fp64, total[1] uint64-as-int64) device tensors."""
    L = _lib_()
    _need(p, torch.float32, "p")
    n = p.numel()
    idx = torch.empty(m, dtype=torch.int64, device=p.device)
    w = torch.empty(m, dtype=torch.float64, device=p.device)
    tot = torch.zeros(1, dtype=torch.int64, device=p.device)
    nb = L.l1_sample_multinomial_workspace_bytes(n)
    ws = workspace(nb, "multinomial")
    _lib.check(L.l1_sample_multinomial(_ptr(p), n, m, seed & 0xFFFFFFFFFFFFFFFF, row_base, _ptr(idx), _ptr(w),
                                       _ptr(tot), _ptr(ws), ws.numel(), _stream()))
    return idx, w, tot


def l1_coreset_gather(X, idx=None, weight=None, count=None, row_base: int = 0, capacity: int | None = None,
                      Z=None):
    """NEXT-2: Z = D X over the sampled rows (fp64), Z_j = weight_j * X[idx_j - row_base].
    X: (n, q) fp32 CUDA, last column -b.  Returns Z (capacity, q) fp64."""
    L = _lib_()
    if X.dim() != 2 or X.dtype != torch.float32 or not X.is_cuda or X.stride(1) != 1:
        raise ValueError("X must be a CUDA fp32 (n, q) tensor with unit column stride")
    n, q = X.shape
    if idx is not None:
        _need(idx, torch.int64, "idx")
    if weight is not None:
        _need(weight, torch.float64, "weight")
    if count is not None:
        _need(count, torch.int64, "count")
    if capacity is None:
        capacity = idx.numel() if idx is not None else n
    if Z is None:
        Z = torch.empty((capacity, q), dtype=torch.float64, device=X.device)
    _lib.check(L.l1_coreset_gather(_ptr(X), n, q, X.stride(0), _ptr(idx), _ptr(weight), _ptr(count), row_base,
                                   capacity, _ptr(Z), Z.stride(0), _stream()))
    return Z


def l1_lad_solve(Z, m=None, max_iter: int = 100, tol: float = 1e-10):
    """NEXT-2: x = argmin_x sum_{j<m} |Z_j . [x; 1]| (interior point, fp64, on the device).
    Z: (capacity, q) fp64 CUDA; m: device int64 scalar tensor (rows used) or None (all rows).
    Returns (x (q-1,) fp64, info (8,) fp64) device tensors (see include/fct.h)."""
    L = _lib_()
    _need(Z, torch.float64, "Z")
    cap, q = Z.shape
    if m is not None:
        _need(m, torch.int64, "m")
    x = torch.empty(q - 1, dtype=torch.float64, device=Z.device)
    info = torch.empty(8, dtype=torch.float64, device=Z.device)
    nb = L.l1_lad_workspace_bytes(cap, q)
    ws = workspace(nb, "lad", Z.device)
    _lib.check(L.l1_lad_solve(_ptr(Z), _ptr(m), cap, q, Z.stride(0), max_iter, tol, _ptr(x), _ptr(info), _ptr(ws),
                              ws.numel(), _stream()))
    return x, info


def l1_coreset_regression(X, idx, weight, count, row_base: int = 0, max_iter: int = 100, tol: float = 1e-10):
    """FastCauchyRegression steps 6-8 on one device: gather D X and solve min ||D(Ax - b)||_1.
    Returns (x_hat, info)."""
    Z = l1_coreset_gather(X, idx, weight, count, row_base)
    return l1_lad_solve(Z, count, max_iter, tol)


def fct2_sketch(A, signs_t, sel, C, t: int, s: int, r1: int, Y=None):
    """NEXT-3: Y = (8/r1) sqrt(pi t/2s) C H~ A, the FCT2 sketch (Sec. 3.2) with SRHT blocks of t rows.
    A: (n, d) fp32 CUDA (row stride lda); signs_t int8[t]; sel int32[s]; C: (r1, >= nb*s) fp32 CUDA."""
    L = _lib_()
    if A.dim() != 2 or A.dtype != torch.float32 or not A.is_cuda or A.stride(1) != 1:
        raise ValueError("A must be a CUDA fp32 (n, d) tensor with unit column stride")
    _need(signs_t, torch.int8, "signs_t")
    _need(sel, torch.int32, "sel")
    if C.dim() != 2 or C.dtype != torch.float32 or not C.is_cuda or C.stride(1) != 1:
        raise ValueError("C must be a CUDA fp32 (r1, nb*s) tensor with unit column stride")
    n, d = A.shape
    if Y is None:
        Y = torch.empty((r1, d), dtype=torch.float32, device=A.device)
    nb = L.fct2_workspace_bytes(n, d, t, s, r1)
    ws = workspace(nb, "fct2", A.device)
    _lib.check(L.fct2_sketch(_ptr(A), n, d, A.stride(0), _ptr(signs_t), _ptr(sel), _ptr(C), C.stride(0), t, s, r1,
                             _ptr(Y), _ptr(ws), ws.numel(), _stream()))
    return Y


def trim(idx, w, cnt):
    """Host copies of the first min(count, capacity) samples."""
    c = int(cnt.item())
    k = min(c, idx.numel())
    return idx[:k].cpu(), w[:k].cpu(), c


class Pipeline:
    """Pre-allocated single-device hot path: sketch -> condition -> row-norm -> probs -> sample.

    Buffers are allocated once, so `run()` only enqueues kernels (CUDA-graph capturable)."""

    def __init__(self, n: int, d: int, s: int, r1: int, k: int, m: int, seed: int, device=None,
                 capacity: int | None = None):
        self.L = _lib_()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.n, self.d, self.s, self.r1, self.k, self.m, self.seed = n, d, s, r1, k, m, seed
        self.capacity = 2 * m + 64 if capacity is None else capacity
        f32, f64 = torch.float32, torch.float64
        self.Y = torch.empty((r1, d), dtype=f32, device=dev)
        self.R = torch.empty((d, d), dtype=f64, device=dev)
        self.Rinv = torch.empty((d, d), dtype=f64, device=dev)
        self.lam = torch.empty(n, dtype=f32, device=dev)
        self.p = torch.empty(n, dtype=f32, device=dev)
        self.idx = torch.empty(self.capacity, dtype=torch.int64, device=dev)
        self.weight = torch.empty(self.capacity, dtype=f64, device=dev)
        self.count = torch.zeros(1, dtype=torch.int64, device=dev)
        self.info = torch.zeros(1, dtype=torch.int32, device=dev)
        nb = self.L.fct_pipeline_workspace_bytes(n, d, s, r1, k)
        self.ws = torch.empty(nb, dtype=torch.uint8, device=dev)

    def run(self, A, signs, cauchy_diag, hash_rows, Pi2):
        _lib.check(self.L.fct_pipeline(_ptr(A), self.n, self.d, A.stride(0), _ptr(signs), _ptr(cauchy_diag),
                                       _ptr(hash_rows), self.s, self.r1, _ptr(Pi2), self.k, self.m,
                                       self.seed & 0xFFFFFFFFFFFFFFFF, _ptr(self.Y), _ptr(self.R), _ptr(self.Rinv),
                                       _ptr(self.lam), _ptr(self.p), _ptr(self.idx), _ptr(self.weight),
                                       self.capacity, _ptr(self.count), _ptr(self.info), _ptr(self.ws),
                                       self.ws.numel(), _stream()))
        return self


class HostPipeline:
    """End-to-end entry point: inputs in (pinned) HOST memory, result (idx, weight, count) on the host.
    Wraps fct_pipeline_host; device buffers for A and the aux arrays are allocated once."""

    def __init__(self, n: int, d: int, s: int, r1: int, k: int, m: int, seed: int, device=None,
                 capacity: int | None = None):
        self.L = _lib_()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.n, self.d, self.s, self.r1, self.k, self.m, self.seed = n, d, s, r1, k, m, seed
        self.capacity = 2 * m + 64 if capacity is None else capacity
        self.dev_A = torch.empty((n, d), dtype=torch.float32, device=dev)
        self.dev_aux = torch.empty(self.L.fct_pipeline_aux_bytes(n, d, s, k), dtype=torch.uint8, device=dev)
        self.ws = torch.empty(self.L.fct_pipeline_host_workspace_bytes(n, d, s, r1, k, self.capacity),
                              dtype=torch.uint8, device=dev)
        self.idx = torch.empty(self.capacity, dtype=torch.int64).pin_memory()
        self.weight = torch.empty(self.capacity, dtype=torch.float64).pin_memory()
        self.count = torch.zeros(1, dtype=torch.int64)

    def run(self, A_host, signs_host, cauchy_host, hash_host, Pi2_host):
        for t, nm in ((A_host, "A"), (signs_host, "signs"), (cauchy_host, "cauchy"), (hash_host, "hash"),
                      (Pi2_host, "Pi2")):
            if t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{nm} must be a contiguous HOST tensor")
        _lib.check(self.L.fct_pipeline_host(_ptr(A_host), self.n, self.d, self.d, _ptr(signs_host),
                                            _ptr(cauchy_host), _ptr(hash_host), self.s, self.r1, _ptr(Pi2_host),
                                            self.k, self.m, self.seed & 0xFFFFFFFFFFFFFFFF, _ptr(self.idx),
                                            _ptr(self.weight), self.capacity, _ptr(self.count), _ptr(self.dev_A),
                                            _ptr(self.dev_aux), _ptr(self.ws), self.ws.numel(), _stream()))
        c = int(self.count[0])
        k = min(c, self.capacity)
        return self.idx[:k], self.weight[:k], c
