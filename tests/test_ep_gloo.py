"""Expert parallelism on CPU with gloo, world sizes 2 and 4 (SURVEY §8e
E1/E2/E4).  Each process is one rank of an expert-parallel decode: it routes
its own tokens, all-gathers the routing blocks, runs the experts it owns for
every rank's tokens, returns the outputs by all-to-all and combines them in
rank order — the data flow of engine.cu ep_step_on, with the layer
arithmetic taken from the fp64 oracle (there is no GPU here).  Checked:

* every rank's outputs equal the single-process oracle layer stack;
* every rank's scheduler — the product's C++ stepper fed through the
  product's shard view (ef_ep_shard_view) — makes exactly the decisions of the
  per-shard oracle (oracle/ep_shard.py: the reference loop per shard)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2510_26730_b200 as ef
from paper_2510_26730_b200 import ep


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


SHAPE = dict(L=4, M=8, k=2, d=64, ff=96)


def _ep_decode(rank, world, B, steps, seed):
    """One rank's expert-parallel decode over `steps` tokens (fp64 oracle
    arithmetic, gloo exchange).  Returns (inputs, outputs, global routing log)."""
    from oracle import numerics as N
    L, M, k, d, ff = (SHAPE[x] for x in ("L", "M", "k", "d", "ff"))
    w = N.ModelWeights(L=L, M=M, d=d, ff=ff, dtype="f32", seed=seed)
    own = ep.owned_experts(rank, M, world)
    h_in, h_out, log = [], [], []
    for t in range(steps):
        h = N.input_hidden(seed + 100 * rank, t, B, d).astype(np.float64)
        h_in.append(h.copy())
        for l in range(L):
            x = N.rmsnorm(h)
            # all router rows l..L-1 (the pre-gate rows a horizon may ask for)
            lg = np.stack([N.router_logits(x, w.router(l + j)) for j in range(L - l)]
                          ).astype(np.float32)
            sel = N.topk_select(lg[0], k)
            wts = N.route_weights(lg[0], sel, "mixtral")
            # dispatch: every rank's (x, logits, sel) to every rank
            xe = N.cast(x.astype(np.float32), "f32").astype(np.float64)  # expert input T(x)
            blk = [torch.tensor(xe), torch.tensor(lg), torch.tensor(sel)]
            gx, glg, gsel = [], [], []
            for src, dst in zip(blk, (gx, glg, gsel)):
                out = [torch.empty_like(src) for _ in range(world)]
                dist.all_gather(out, src)
                dst.extend(o.numpy() for o in out)
            X = np.concatenate(gx)              # [G*B, d]
            LG = np.concatenate(glg, axis=1)    # [R, G*B, M]
            SEL = np.concatenate(gsel)          # [G*B, k]
            log.append((LG, SEL.astype(np.int32), 0))
            # owner: my experts for every rank's tokens, y in global slot order
            y = np.zeros((world * B * k, d))
            for f in range(world * B * k):
                e = int(SEL[f // k, f % k])
                if e in own:
                    w1, w3, w2 = w.expert(l, e)
                    y[f] = N.swiglu(X[f // k:f // k + 1], w1, w3, w2, "f32")[0]
            # combine: all-to-all (chunk g = rank g's slots), rank-order sum
            recv = torch.empty(world * B * k * d, dtype=torch.float64)
            dist.all_to_all_single(recv, torch.tensor(y.reshape(-1)))
            recv = recv.numpy().reshape(world, B * k, d)
            moe = np.zeros((B, d))
            for tt in range(B):
                for r in range(k):
                    o = ep.owner(int(sel[tt, r]), M, world)
                    moe[tt] += wts[tt, r] * recv[o, tt * k + r]
            h = h + moe
        h_out.append(h)
    return h_in, h_out, log


def _worker(rank, world, port, q, B, steps, seed):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h_in, h_out, log = _ep_decode(rank, world, B, steps, seed)
        q.put((rank, h_in, h_out, log))
    finally:
        dist.destroy_process_group()


def _run(world, B, steps, seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, B, steps, seed))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _product_shard_decisions(log, rank, world, policy, budget, steps, link_bw, layer_ns):
    """The product's C++ stepper over the product's shard view of the log."""
    L, M, k = SHAPE["L"], SHAPE["M"], SHAPE["k"]
    E_s = 3 * SHAPE["d"] * SHAPE["ff"] * 4
    model = ep.shard_model(ef.ModelSpec(L, M, k, E_s, 8, 64), world)
    cur = {"t": 0}

    def pregate(layer, h):
        return ep.shard_view(log[cur["t"] * L + layer][0][h], log[cur["t"] * L + layer][1], M, k,
                             world, rank)[0]

    sim = ef.Simulator(model, ef.HardwareSpec(link_bw, budget * E_s, layer_ns / 1e9), policy,
                       ef.Seed(0), emit_events=True, pregate=pregate)
    for t in range(steps):
        gates, actual, groups = [], [], []
        for l in range(L):
            g, grp, a = ep.shard_view(log[t * L + l][0][0], log[t * L + l][1], M, k, world, rank)
            gates.append(ef.GateDistribution(g))
            groups.append(grp)
            actual.append(a)
        GB = log[t * L][1].shape[0]
        tr = ef.ActivationTrace(ef.TokenBatch((-(t + 1),)), tuple(gates), tuple(actual),
                                tuple(groups), tuple([1] * GB))
        cur["t"] = t
        sim.run_token(tr)
    return sim


@pytest.mark.parametrize("world", [2, 4])
def test_ep_decode_matches_single_process_and_shard_oracle(world):
    from oracle import numerics as N
    from oracle import replay as R
    from oracle.ep_shard import replay_shard
    from oracle.sim import Policy
    B, steps, seed = 2, 3, 5
    res = _run(world, B, steps, seed)
    L, M, k, d, ff = (SHAPE[x] for x in ("L", "M", "k", "d", "ff"))
    w = N.ModelWeights(L=L, M=M, d=d, ff=ff, dtype="f32", seed=seed)
    # (1) outputs: the layer stack of the single-process oracle, per rank
    for rank, h_in, h_out, log in res:
        for t in range(steps):
            h = h_in[t]
            for l in range(L):
                lg, sel, _ = log[t * L + l]
                h = N.moe_layer(h, w, l, k, "mixtral", logits_override=lg[0][rank * B:(rank + 1) * B],
                                sel_override=sel[rank * B:(rank + 1) * B])["h_next"]
            np.testing.assert_allclose(h_out[t], h, rtol=1e-12, atol=1e-12)
    # every rank saw the same global routing
    for r in res[1:]:
        for a, b in zip(r[3], res[0][3]):
            assert np.array_equal(a[1], b[1]) and np.array_equal(a[0], b[0])
    # (2) per-shard decisions: product stepper on the product's shard view ==
    # the reference loop per shard (oracle)
    log = res[0][3]
    budget = ep.shard_budget(int(0.4 * L * M), M, world, L)
    link_bw, layer_ns = 2_000_000_000, 150_000
    pol = ef.PolicyConfig("a", "adaptive", predictor="pregate")
    opol = Policy("a", "adaptive", predictor="pregate")
    E_s = 3 * d * ff * 4
    for rank in range(world):
        sim = _product_shard_decisions(log, rank, world, pol, budget, steps, link_bw, layer_ns)
        orc = replay_shard(log, L=L, M=M, k=k, G=world, rank=rank, expert_bytes=E_s,
                           link_bw=link_bw, budget_experts=budget, layer_ns=layer_ns, policy=opol,
                           tokens_per_step=[(-(t + 1),) for t in range(steps)])
        got = R.product_metrics_dict(sim.metrics(), sim.cache_events())
        assert R.diff_dicts(got, R.oracle_metrics_dict(orc)) == [], rank
        assert orc.metrics.hits + orc.metrics.misses > 0


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_shard_view_matches_oracle(G):
    """ef_ep_shard_view (the C++ the engine uses) against oracle/ep_shard.py:
    restricted fp64 gates bit-exact, groups and unions identical."""
    from oracle import ep_shard as O
    rng = np.random.default_rng(G)
    M, k, GB = 8, 2, 6
    for _ in range(20):
        lg = rng.standard_normal((GB, M)).astype(np.float32)
        sel = np.stack([rng.choice(M, k, replace=False) for _ in range(GB)]).astype(np.int32)
        for rank in range(G):
            g1, grp1, a1 = ep.shard_view(lg, sel, M, k, G, rank)
            g2, grp2, a2 = O.shard_view(lg, sel, M, G, rank)
            assert np.array_equal(g1, g2) and grp1 == grp2 and a1 == a2


def test_owner_partition_and_budget():
    assert [ep.owner(e, 8, 8) for e in range(8)] == list(range(8))
    assert [ep.owner(e, 8, 2) for e in range(8)] == [0] * 4 + [1] * 4
    assert ep.owned_experts(1, 64, 4) == list(range(16, 32))
    assert ep.shard_budget(102, 8, 2, 32) == 51
    m = ep.shard_model(ef.ModelSpec(56, 8, 2, 604 * ef.MB, 8, 32000), 8)
    assert (m.experts_per_layer, m.top_k) == (1, 1)
    with pytest.raises(ValueError):
        ep.shard_model(ef.ModelSpec(4, 6, 2, ef.MB, 8, 64), 4)


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
