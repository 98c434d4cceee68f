"""Multi-rank plumbing of paper_1207_4684_b200.dist on CPU (gloo, world_size 2 and 3).

The per-rank compute is the oracle (test-only stand-in for the CUDA ops), so this checks the
sharding, the two collectives (sum of partial sketches, sum of lambda totals), the global-row keying
of the sampler and the gather -- against the single-process oracle pipeline on the full problem.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import fctgen
import oracle
from oracle import lad as OL
from paper_1207_4684_b200.dist import Ops, coreset_regression, run_step, gather_samples, shard_rows


def test_shard_rows_cover_and_align():
    for n, s, world in [(1000, 64, 2), (1 << 20, 256, 8), (5, 4, 3), (64 * 7 + 3, 64, 4)]:
        shards = [shard_rows(n, s, r, world) for r in range(world)]
        assert shards[0].row0 == 0
        tot = 0
        for a, b in zip(shards, shards[1:]):
            assert a.row0 + a.rows == b.row0 or b.rows == 0
        for sh in shards:
            assert sh.row0 % s == 0
            tot += sh.rows
        assert tot == n


def oracle_ops():
    def sketch(A, sg, c, h, s, r1):
        Y, _ = oracle.sketch(A.numpy(), sg.numpy(), c.numpy(), h.numpy(), s, r1)
        return torch.from_numpy(Y)

    def condition(Y):
        R, Rinv, _ = oracle.condition(Y.numpy())
        return torch.from_numpy(R), torch.from_numpy(Rinv)

    def rownorm(A, Rinv, Pi2):
        lam, tot = oracle.rownorm(A.numpy(), Rinv.numpy(), Pi2.numpy())
        return torch.from_numpy(lam), torch.tensor([tot], dtype=torch.float64)

    def probs(lam, tot):
        return (lam / tot).to(torch.float32)

    def sample(p, m, seed, row_base):
        idx, w, cnt = oracle.sample(p.numpy(), m, seed=seed, row_base=row_base)
        return torch.from_numpy(idx), torch.from_numpy(w), torch.tensor([cnt], dtype=torch.int64)

    def coreset_gather(X, idx, w, k, row_base):
        return torch.from_numpy(OL.coreset_rows(X.numpy(), idx[:k].numpy(), w[:k].numpy(), row_base))

    def lad_solve(Z):
        x, f = OL.lad(Z.numpy())
        return torch.from_numpy(x), torch.tensor([f])

    return Ops(sketch, condition, rownorm, probs, sample, coreset_gather=coreset_gather, lad_solve=lad_solve)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = fctgen.CONFIGS[2]
        sh = shard_rows(n, cfg.s, rank, world)
        inp = fctgen.make_inputs(cfg, n=sh.rows, row0=sh.row0)
        t = torch.from_numpy
        res = run_step(oracle_ops(), sh, t(inp.A), t(inp.signs), t(inp.cauchy), t(inp.hash), t(inp.pi2),
                       cfg.s, cfg.r1, cfg.m, seed=3)
        gi, gw, gc = gather_samples(res)
        lam_all = [torch.zeros(shard_rows(n, cfg.s, r, world).rows, dtype=torch.float64) for r in range(world)]
        # variable-size gather via padding
        L = max(x.numel() for x in lam_all)
        pad = torch.zeros(L, dtype=torch.float64)
        pad[:res.lam.numel()] = res.lam
        outs = [torch.zeros(L, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(outs, pad)
        lam = torch.cat([o[:x.numel()] for o, x in zip(outs, lam_all)])
        xh, info, Z = coreset_regression(oracle_ops(), sh, t(inp.A), res)
        if rank == 0:
            q.put((res.Y.numpy(), lam.numpy(), float(res.total.item()), gi.numpy(), gw.numpy(), gc, Z.numpy(),
                   xh.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_dist_pipeline_equals_single_process(world):
    cfg = fctgen.CONFIGS[2]
    n = 12 * cfg.s + 17
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    t0 = time.time()
    got = None
    while got is None and time.time() - t0 < 240:
        try:
            got = q.get(timeout=2)
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    assert got is not None and all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    Y, lam, tot, gi, gw, gc, Z, xh = got
    # single-process oracle pipeline on the full problem
    inp = fctgen.make_inputs(cfg, n=n)
    Y1, _ = oracle.sketch(inp.A, inp.signs, inp.cauchy, inp.hash, cfg.s, cfg.r1)
    np.testing.assert_allclose(Y, Y1, rtol=1e-12, atol=1e-12 * np.abs(Y1).max())
    _, Rinv, _ = oracle.condition(Y1)
    lam1, tot1 = oracle.rownorm(inp.A, Rinv, inp.pi2)
    np.testing.assert_allclose(lam, lam1, rtol=1e-9)
    np.testing.assert_allclose(tot, tot1, rtol=1e-12)
    p1 = (lam1 / tot1).astype(np.float32)
    i1, w1, c1 = oracle.sample(p1, cfg.m, seed=3)
    # the sharded sampler keys uniforms by GLOBAL row: same decisions as one process
    assert gc == c1
    common = np.intersect1d(gi, i1)
    assert len(common) >= c1 - 2            # at most an ulp-level p difference may flip a decision
    assert (np.diff(gi) > 0).all()
    # NEXT-2: the all-gathered coreset is exactly D X over the gathered samples, in ascending global rows,
    # and its solution is the single-process one
    np.testing.assert_array_equal(Z, OL.coreset_rows(inp.A, gi, gw))
    x1, f1 = OL.lad(Z)
    np.testing.assert_array_equal(xh, x1)


def _bench_worker(rank, world, port, n, q):
    """bench.py's own timed region (run_timed: warm-up, barrier + sync on both sides, K steps, MAX over ranks)
    driving dist.run_step end to end on a gloo process group, with the oracle stand-in ops."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = fctgen.CONFIGS[1]
        sh = shard_rows(n, cfg.s, rank, world)
        inp = fctgen.make_inputs(cfg, n=sh.rows, row0=sh.row0)
        t = torch.from_numpy
        ops = oracle_ops()
        calls = []

        def step(events):
            calls.append(events)
            return run_step(ops, sh, t(inp.A), t(inp.signs), t(inp.cauchy), t(inp.hash), t(inp.pi2), cfg.s, cfg.r1,
                            cfg.m, seed=cfg.seed)

        res, ms_max, evs = bench.run_timed(step, K=2, W=3, world=world, names=[], cuda=False)
        mine = torch.tensor([ms_max], dtype=torch.float64)
        allv = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allv, mine)
        gi, gw, gc = gather_samples(res)
        q.put((rank, len(calls), [float(v.item()) for v in allv], gi.numpy(), gw.numpy(), gc))
    finally:
        dist.destroy_process_group()


def test_bench_timed_region_on_gloo():
    """W + K steps per rank, every rank reports the same (maximum) time, and the samples of the timed run equal the
    single-process oracle pipeline's (the same code path bench.py runs under torchrun with NCCL)."""
    world, n = 2, 4 * 1024 + 37
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_bench_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in ps:
        p.start()
    outs = [q.get(timeout=600) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ncalls, times, gi, gw, gc in outs:
        assert ncalls == 3 + 2
        assert len(set(times)) == 1 and times[0] > 0          # max over ranks, identical on every rank
    # single process reference
    cfg = fctgen.CONFIGS[1]
    inp = fctgen.make_inputs(cfg, n=n)
    Y, _ = oracle.sketch(inp.A, inp.signs, inp.cauchy, inp.hash, cfg.s, cfg.r1)
    _, Rinv, _ = oracle.condition(Y)
    lam, tot = oracle.rownorm(inp.A, Rinv, inp.pi2)
    p = oracle.probs(lam, tot).astype(np.float32)
    oi, ow, oc = oracle.sample(p, cfg.m, seed=cfg.seed)
    _, _, _, gi, gw, gc = outs[0]
    assert gc == oc
    np.testing.assert_array_equal(gi, oi)
    np.testing.assert_array_equal(gw, ow)
