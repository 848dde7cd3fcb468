"""Expert-parallel exchange and per-shard scheduling on CPU with gloo,
world_size 2.  The MoE layer computed expert-parallel
must equal the single-process layer; each rank's cache trace over its owned
experts must equal the oracle fed with that rank's access subsequence."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_26730_b200 import ep


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _weights(M, d, ff, seed=0):
    rng = np.random.default_rng(seed)
    return [(rng.standard_normal((ff, d)) / d ** 0.5, rng.standard_normal((ff, d)) / d ** 0.5,
             rng.standard_normal((d, ff)) / ff ** 0.5) for _ in range(M)]


def _swiglu(x, w):
    g, u = x @ w[0].T, x @ w[1].T
    return (g / (1 + np.exp(-g)) * u) @ w[2].T


def _reference(xs, sels, wts, W):
    out = []
    for x, sel, w in zip(xs, sels, wts):
        o = x.copy()
        for t in range(x.shape[0]):
            for r in range(sel.shape[1]):
                o[t] += w[t, r] * _swiglu(x[t:t + 1], W[sel[t, r]])[0]
        out.append(o)
    return out


def _worker(rank, world, port, q, M, d, ff, B, k):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W = _weights(M, d, ff)
        rng = np.random.default_rng(100 + rank)
        x = rng.standard_normal((B, d))
        sel = np.stack([rng.choice(M, k, replace=False) for _ in range(B)])
        wts = rng.random((B, k))
        ex = ep.EPExchange(M)
        got, plan = ex.dispatch(torch.tensor(x), sel)
        # every received row belongs to an expert this rank owns
        mine = set(ep.owned_experts(rank, M, world))
        assert set(int(e) for e in plan.recv_experts) <= mine
        y = torch.zeros_like(got)
        for e, rows in ep.local_groups(plan.recv_experts):
            y[rows] = torch.tensor(_swiglu(got[rows].numpy(), W[e]))
        out = ex.combine(y, plan, torch.tensor(wts), residual=torch.tensor(x))
        q.put((rank, x, sel, wts, out.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B,k", [(5, 2), (1, 2), (16, 4)])
def test_ep_dispatch_combine_matches_single_process(B, k):
    world, M, d, ff = 2, 8, 32, 48
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, M, d, ff, B, k))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    W = _weights(M, d, ff)
    want = _reference([r[1] for r in res], [r[2] for r in res], [r[3] for r in res], W)
    for (rank, *_rest, got), w in zip(res, want):
        np.testing.assert_allclose(got, w, rtol=1e-12, atol=1e-12)


def test_owner_partition_and_budget():
    assert [ep.owner(e, 8, 8) for e in range(8)] == list(range(8))
    assert [ep.owner(e, 8, 2) for e in range(8)] == [0] * 4 + [1] * 4
    assert ep.owned_experts(1, 64, 4) == list(range(16, 32))
    assert ep.shard_budget(102, 8, 2, 32) == 51


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_peer_pool_placement(G):
    """E3 placement: the pools partition every layer's experts (each expert's
    home copy exactly once) and, for G > 1, no pool sits on its owner's GPU."""
    L, M = 56, 8
    seen = []
    for r in range(G):
        ids = ep.peer_pool_ids(r, L, M, G)
        assert all(ep.owner(i % M, M, G) == r for i in ids)
        assert ids == sorted(ids)
        if G > 1:
            assert ep.home_pool_rank(r, G) != r
        seen += ids
    assert sorted(seen) == list(range(L * M))
    assert sorted(ep.home_pool_rank(r, G) for r in range(G)) == list(range(G))


def test_per_shard_cache_traces_match_oracle():
    """E2: each rank's ExpertCache sees only its owned experts; replaying the
    same access stream through the oracle per shard gives the same trace."""
    import paper_2510_26730_b200 as ef
    from oracle import decisions as D
    M, G, L = 8, 2, 4
    rng = np.random.default_rng(7)
    stream = [(l, int(e)) for _ in range(6) for l in range(L) for e in rng.choice(M, 2, replace=False)]
    for rank in range(G):
        mine = [(l, e) for l, e in stream if ep.owner(e, M, G) == rank]
        prod = ef.ExpertCache(3 * ef.MB, ef.MB, record_events=True)
        orc = D.ExpertCache(3 * ef.MB, ef.MB, record_events=True)
        for now, (l, e) in enumerate(mine):
            if not prod.access(ef.ExpertId(l, e), now):
                prod.admit(ef.ExpertId(l, e), ef.TIER_HIGH, now)
            if not orc.access((l, e), now):
                orc.admit((l, e), D.HIGH, now)
        assert [(n, k, x.layer, x.expert) for n, k, x in prod.events] == \
            [(n, k, x[0], x[1]) for n, k, x in orc.events]
