"""Multi-GPU row sharding of the hot path over torch.distributed.

Pi1 A = sum_g Pi1_g A_g for contiguous s-aligned row shards (H~, C, D are (block-)diagonal and the
columns of B partition across row blocks, Sec. 3.1), so:
    each rank sketches its slice  ->  ONE sum-allreduce of the r1 x d partial sketches (C1)
    -> every rank conditions the identical reduced Y (no broadcast needed)
    -> row-norms of the local rows -> sum-allreduce of the fp64 local sums (C3)
    -> probabilities and Bernoulli sampling keyed by the GLOBAL row index (row_base).
This mirrors the paper's map/reduce two-pass structure.

The compute steps are injected (`ops`), so the same plumbing runs on the CUDA path (`cuda_ops`,
NCCL) and -- in tests only -- on CPU stand-ins with the gloo backend.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    row0: int       # first global row of this rank (multiple of s)
    rows: int       # rows owned by this rank (may be 0 for tiny problems)


def shard_rows(n: int, s: int, rank: int, world: int) -> Shard:
    """Contiguous s-aligned row shards: block b goes to rank floor(b * world / nblocks)."""
    nb = -(-n // s)
    b0 = (rank * nb) // world
    b1 = ((rank + 1) * nb) // world
    row0 = b0 * s
    rows = max(0, min(n, b1 * s) - row0)
    return Shard(rank, world, row0, rows)


@dataclass
class Ops:
    """Per-rank compute steps (all tensors on the rank's device)."""
    sketch: Callable      # (A, signs, cauchy, hash, s, r1) -> Y (r1, d)
    condition: Callable   # (Y) -> (R, Rinv)
    rownorm: Callable     # (A, Rinv, Pi2) -> (lambda, local_sum[1] fp64)
    probs: Callable       # (lambda, total[1]) -> p
    sample: Callable      # (p, m, seed, row_base) -> (idx, weight, count[1])
    probs_sample: Callable | None = None   # fused: (lambda, total[1], m, seed, row_base) -> (p, idx, weight, count)
    coreset_gather: Callable | None = None  # NEXT-2: (X, idx, weight, k, row_base) -> Z (k, q) fp64 = rows of D X
    lad_solve: Callable | None = None       # NEXT-2: (Z) -> (x, info)


def cuda_ops(estimator: str = "median") -> Ops:
    """The CUDA compute steps.  estimator = "median" (the Cauchy median estimate of P:L2921-2938, a8) or
    "exact" (NEXT-1: the exact l1 row norms of U = A R^-1 that the paper's Sec. 6.2 uses)."""
    from . import api
    if estimator not in ("median", "exact"):
        raise ValueError(f"estimator must be 'median' or 'exact', not {estimator!r}")

    def _cond(Y):
        R, Rinv, info = api.fct_condition(Y, check=False)
        return R, Rinv, info

    def _rown(A, Rinv, Pi2):
        if estimator == "exact":
            return api.l1_rownorm_exact(A, Rinv)
        return api.l1_rownorm(A, Rinv, Pi2)

    return Ops(sketch=lambda A, sg, c, h, s, r1: api.fct_sketch(A, sg, c, h, s, r1),
               condition=_cond, rownorm=_rown,
               probs=lambda lam, tot: api.l1_probs(lam, tot),
               sample=lambda p, m, seed, row_base: api.l1_sample(p, m, seed, row_base=row_base),
               probs_sample=lambda lam, tot, m, seed, row_base: api.l1_probs_sample(lam, tot, m, seed,
                                                                                    row_base=row_base),
               coreset_gather=lambda X, idx, w, k, row_base: api.l1_coreset_gather(X, idx[:k], w[:k], None,
                                                                                   row_base=row_base, capacity=k),
               lad_solve=lambda Z: api.l1_lad_solve(Z))


@dataclass
class StepResult:
    Y: torch.Tensor
    R: torch.Tensor
    Rinv: torch.Tensor
    lam: torch.Tensor
    p: torch.Tensor
    total: torch.Tensor
    idx: torch.Tensor
    weight: torch.Tensor
    count: torch.Tensor
    extra: tuple = ()


def run_step(ops: Ops, shard: Shard, A, signs, cauchy, hash_rows, Pi2, s: int, r1: int, m: int, seed: int,
             group=None, events: dict | None = None) -> StepResult:
    """One pass of the whole hot path on this rank's shard; collectives only at C1 and C3."""
    ev = events or {}
    mark = (lambda k: ev[k].record()) if ev else (lambda k: None)
    mark("start")
    Y = ops.sketch(A, signs, cauchy, hash_rows, s, r1)
    mark("sketch")
    if shard.world > 1:
        dist.all_reduce(Y, op=dist.ReduceOp.SUM, group=group)          # C1: r1 x d partial sketches
    mark("allreduce_Y")
    cond = ops.condition(Y)
    R, Rinv = cond[0], cond[1]
    mark("condition")
    lam, total = ops.rownorm(A, Rinv, Pi2)
    mark("rownorm")
    if shard.world > 1:
        dist.all_reduce(total, op=dist.ReduceOp.SUM, group=group)      # C3: one fp64 scalar
    mark("allreduce_sum")
    if ops.probs_sample is not None:
        p, idx, w, cnt = ops.probs_sample(lam, total, m, seed, shard.row0)
    else:
        p = ops.probs(lam, total)
        idx, w, cnt = ops.sample(p, m, seed, shard.row0)
    mark("sample")
    return StepResult(Y, R, Rinv, lam, p, total, idx, w, cnt, tuple(cond[2:]))


def gather_samples(res: StepResult, group=None):
    """All ranks' (idx, weight) concatenated in rank order = ascending global rows (every rank gets it)."""
    world = dist.get_world_size(group)
    dev = res.idx.device
    k = min(int(res.count.item()), res.idx.numel())
    meta = torch.tensor([k, int(res.count.item())], dtype=torch.int64, device=dev)
    metas = [torch.zeros_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta, group=group)
    mx = max(1, max(int(m[0].item()) for m in metas))
    idx = torch.full((mx,), -1, dtype=torch.int64, device=dev)
    w = torch.zeros((mx,), dtype=torch.float64, device=dev)
    idx[:k] = res.idx[:k]
    w[:k] = res.weight[:k]
    gi = [torch.empty_like(idx) for _ in range(world)]
    gw = [torch.empty_like(w) for _ in range(world)]
    dist.all_gather(gi, idx, group=group)
    dist.all_gather(gw, w, group=group)
    out_i = [gi[r][:int(metas[r][0].item())] for r in range(world)]
    out_w = [gw[r][:int(metas[r][0].item())] for r in range(world)]
    return torch.cat(out_i), torch.cat(out_w), int(sum(int(m[1].item()) for m in metas))


def coreset_regression(ops: Ops, shard: Shard, X, res: StepResult, group=None):
    """NEXT-2 across ranks (FastCauchyRegression steps 6-8): every rank forms the rows of D X
    for its own samples (X = [A, -b] is its row shard, row_base = shard.row0), ONE all-gather of the
    k_r x q fp64 blocks assembles the coreset in rank order (= ascending global rows), and every rank solves
    the identical small problem (no broadcast).  Returns (x_hat, info, Z)."""
    k = min(int(res.count.item()), res.idx.numel())
    Z = ops.coreset_gather(X, res.idx, res.weight, k, shard.row0)
    if shard.world > 1:
        world = dist.get_world_size(group)
        meta = torch.tensor([k], dtype=torch.int64, device=Z.device)
        metas = [torch.zeros_like(meta) for _ in range(world)]
        dist.all_gather(metas, meta, group=group)
        ks = [int(t.item()) for t in metas]
        mx = max(1, max(ks))
        pad = torch.zeros((mx, Z.shape[1]), dtype=Z.dtype, device=Z.device)
        pad[:k] = Z
        outs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(outs, pad, group=group)
        Z = torch.cat([o[:kr] for o, kr in zip(outs, ks)]).contiguous()
    x, info = ops.lad_solve(Z)
    return x, info, Z
