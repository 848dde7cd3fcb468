"""Expert-parallel decode on the B200 (engine.cu ep_step_on):

* G = 1 (local transport): the EP step's kernels — routing-block pack,
  owner permutation over the gathered blocks, the decode GEMV pair on the
  gathered rows with y in global slot order, the home combine — against the
  fp64 oracle, decisions bit-exact with the shard oracle;
* G = 2 as two processes on one GPU exchanging through gloo
  (ep.TorchCollective; NCCL refuses two ranks on one device): every rank's
  decisions equal the per-shard oracle of the reference loop, every rank's
  outputs the oracle layer stack over its own tokens."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2510_26730_b200 as ef  # noqa: E402
from paper_2510_26730_b200 import ep  # noqa: E402
from paper_2510_26730_b200.runtime import MoEConfig, MoEEngine, PRESETS, synthetic_hidden  # noqa: E402

POL = ef.PolicyConfig("a", "adaptive", predictor="pregate")
LINK, LAYER_S = 2 * ef.GB, 2e-4


def _opol():
    from oracle.sim import Policy
    return Policy("a", "adaptive", predictor="pregate")


def _run_rank(cfg, rank, world, B, steps, seed, budget, collective=None):
    eng = MoEEngine(cfg, budget_experts=budget, policy=POL, link_bw=LINK, layer_time_s=LAYER_S,
                    max_batch=B, seed=seed, record_routing=True, emit_events=True,
                    ep_rank=rank, ep_world=world, ep_collective=collective)
    dev = torch.device("cuda", 0)
    h_in, h_out = [], []
    for t in range(steps):
        h = synthetic_hidden(cfg, seed + 100 * rank, t, B, dev)
        h_in.append(h.cpu().numpy())
        eng.step(h)
        torch.cuda.synchronize()
        h_out.append(h.cpu().numpy())
    log = eng.routing_log()
    return eng, h_in, h_out, log


def _check(cfg, rank, world, B, steps, seed, budget, eng_metrics, cache_events, h_in, h_out, log,
           tol):
    from oracle import numerics as N
    from oracle import replay as R
    from oracle.ep_shard import replay_shard
    L = cfg.num_layers
    assert len(log) == steps * L and log[0][1].shape == (world * B, cfg.top_k)
    orc = replay_shard(log, L=L, M=cfg.num_experts, k=cfg.top_k, G=world, rank=rank,
                       expert_bytes=cfg.expert_bytes, link_bw=LINK, budget_experts=budget,
                       layer_ns=round(LAYER_S * 1e9), policy=_opol(),
                       tokens_per_step=[(-(t + 1),) for t in range(steps)])
    got = R.product_metrics_dict(eng_metrics, cache_events)
    assert R.diff_dicts(got, R.oracle_metrics_dict(orc)) == [], rank
    w = N.ModelWeights(L=L, M=cfg.num_experts, d=cfg.d_model, ff=cfg.d_ff, dtype=cfg.dtype,
                       seed=seed, shared_ff=cfg.shared_ff, shared_gate=cfg.shared_gate, cache=True)
    mine = slice(rank * B, (rank + 1) * B)
    for t in range(steps):
        h = np.asarray(h_in[t], np.float64)
        for l in range(L):
            lg, sel, _ = log[t * L + l]
            h = N.moe_layer(h, w, l, cfg.top_k, cfg.route_mode, logits_override=lg[0][mine],
                            sel_override=sel[mine])["h_next"]
        err = R.rel_err(h_out[t], h)
        assert err < tol, (rank, t, err)


@pytest.mark.parametrize("shape", ["tiny", "qwen"])
def test_ep_single_rank_matches_oracle(shape):
    if shape == "tiny":
        cfg, budget, B, tol = PRESETS["tiny"], 12, 3, 1e-5
    else:
        cfg = MoEConfig("qwen-2l", 2, 60, 4, 2048, 1408, route_mode="softmax_topk",
                        shared_ff=5632, shared_gate=True)
        budget, B, tol = 48, 2, 2e-2
    eng, h_in, h_out, log = _run_rank(cfg, 0, 1, B, 3, 7, budget)
    _check(cfg, 0, 1, B, 3, 7, budget, eng.metrics(), eng.cache_events(), h_in, h_out, log, tol)
    st = eng.stats()
    assert st["copies"] > 0 and st["ffn_launches"] > 0
    with pytest.raises(ValueError):
        eng.step(synthetic_hidden(cfg, 1, 0, B - 1, torch.device("cuda", 0)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, cfg, B, steps, seed, budget):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        coll = ep.TorchCollective()
        eng, h_in, h_out, log = _run_rank(cfg, rank, world, B, steps, seed, budget, coll)
        q.put((rank, eng.metrics(), eng.cache_events(), h_in, h_out, log, eng.stats(), coll.calls))
        eng.close()
    except BaseException as exc:  # surface the failure in the parent
        q.put((rank, repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape", ["tiny", "mixtral-2l"])
def test_ep_two_ranks_one_gpu(shape):
    import torch.multiprocessing as mp
    if shape == "tiny":
        cfg, B, tol = PRESETS["tiny"], 2, 1e-5
    else:  # the Mixtral expert shape (Mixtral-8x22B runs the same path at d=6144)
        cfg, B, tol = MoEConfig("mixtral-2l", 2, 8, 2, 4096, 14336), 1, 2e-2
    world, steps, seed = 2, 3, 9
    budget = ep.shard_budget(int(0.4 * cfg.total_experts), cfg.num_experts, world,
                             cfg.num_layers)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, cfg, B, steps, seed, budget))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert len(r) > 2, r
    res.sort(key=lambda r: r[0])
    for p in procs:
        assert p.exitcode == 0
    for rank, metrics, events, h_in, h_out, log, stats, calls in res:
        _check(cfg, rank, world, B, steps, seed, budget, metrics, events, h_in, h_out, log, tol)
        assert calls == 2 * steps * cfg.num_layers  # one all-gather + one all-to-all per layer
    # both ranks saw the same global routing
    for a, b in zip(res[0][5], res[1][5]):
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[0], b[0])
