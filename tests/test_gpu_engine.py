"""End-to-end parity of MoEEngine.step() on the B200 against the oracle:

* decisions (routing selection given the GPU's fp32 logits, predicted sets,
  step sizes, cache hit/miss/admit/evict trace, SimEvents, SimMetrics) are
  bit-exact with the OracleStepper restatement of the reference scheduler;
* layer outputs match the float64 oracle within rel 1e-5 (fp32) / 2e-2 (bf16);
* the physical slab holds exactly the bytes of the expert each slot maps to.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2510_26730_b200 as ef  # noqa: E402
from paper_2510_26730_b200.runtime import PRESETS, MoEConfig, MoEEngine, synthetic_hidden  # noqa: E402
from oracle import numerics as N  # noqa: E402
from oracle import replay as R  # noqa: E402
from oracle.sim import Policy  # noqa: E402

DEV = torch.device("cuda", 0)


def oracle_policy(p: ef.PolicyConfig) -> Policy:
    return Policy(p.name, p.strategy, p.predictor, p.interval, p.cache_aware_routing, p.cold_start,
                  p.cum_threshold, p.stall_threshold, p.overfetch_threshold, p.min_step,
                  p.max_step, p.recent_window, p.noise.decay_rate, p.prediction_cache_capacity)


def run_and_check(cfg: MoEConfig, policy, *, B=2, steps=3, budget, link_bw, layer_s, seed=11,
                  bias=0.0, tol=None, check_numerics=True, token_ids=None, forest=None,
                  table=None, timing=False):
    eng = MoEEngine(cfg, budget_experts=budget, policy=policy, link_bw=link_bw,
                    layer_time_s=layer_s, max_batch=B, seed=seed, routing_bias=bias,
                    record_routing=True, emit_events=True, forest=forest, table=table,
                    timing=timing)
    h_in, h_out, toks = [], [], []
    for t in range(steps):
        h = synthetic_hidden(cfg, seed, t, B, DEV)
        h_in.append(h.cpu().numpy())
        tk = token_ids[t] if token_ids else None
        eng.step(h, tk)
        toks.append(tuple(tk) if tk else (-(t + 1),))
        h_out.append(h.cpu().numpy())
    torch.cuda.synchronize()
    log = eng.routing_log()
    xs = eng.routing_x()
    assert len(log) == len(xs) == steps * cfg.num_layers
    w = N.ModelWeights(L=cfg.num_layers, M=cfg.num_experts, d=cfg.d_model, ff=cfg.d_ff,
                       dtype=cfg.dtype, seed=seed, shared_ff=cfg.shared_ff,
                       shared_gate=cfg.shared_gate, cache=True)
    check_router_rows(log, xs, w, cfg.num_layers)
    feats = None
    ofo = None
    if forest is not None:
        from oracle import forest as F
        ofo = F.Forest.from_json(ef.model_to_json(forest))
        tv = np.asarray(table.vectors)

        def feats(tokens, step, target, hist):
            return F.features(tv, cfg.num_layers, cfg.num_experts, tokens, step, target, hist)
    st, mask_bad, sel_bad = _replay(log, cfg, budget, link_bw, layer_s, policy, toks, bias, ofo,
                                    feats, [m for _, m in xs])
    assert not mask_bad, mask_bad[:3]
    assert not sel_bad, sel_bad[:3]
    got = R.product_metrics_dict(eng.metrics(), eng.cache_events())
    want = R.oracle_metrics_dict(st)
    assert R.diff_dicts(got, want) == []
    if check_numerics:
        check_layer_numerics(h_in, h_out, log, xs, w, cfg, tol)
    return eng, log


# Router rows: the GPU's logits against the fp64 product of the GPU's own x_l
# with W_r^(l+h), for the layer's row and every pre-gate row.  Both dtypes
# accumulate in fp32 over identical inputs, so the bound is fp32 rounding.
ROUTER_ROW_TOL = 1e-5


def check_router_rows(log, xs, w, L):
    errs = R.router_row_errors(log, xs, w, L)
    assert errs, "no router rows checked"
    worst = max(errs, key=lambda e: e[3])
    assert worst[3] < ROUTER_ROW_TOL, ("router row mismatch (entry, h, token, rel)", worst)
    return len(errs)


def check_layer_numerics(h_in, h_out, log, xs, w, cfg, tol=None):
    """Every layer's router input x_l (GPU, incl. a combine folded into the
    router kernel) and every step output against the fp64 oracle: rel 1e-5
    (fp32) / 2e-2 (bf16), the north star's tolerances."""
    tol = tol or (1e-5 if cfg.dtype == "f32" else 2e-2)
    for t in range(len(h_in)):
        x_errs = []
        ref = R.forward_step(h_in[t], log, t, w, cfg.num_layers, cfg.top_k, cfg.route_mode,
                             xs=xs, x_errs=x_errs)
        for (_s, layer, e) in x_errs:
            assert e < tol, ("layer input x", t, layer, e)
        err = R.rel_err(h_out[t], ref)
        assert err < tol, (t, err)


def _replay(log, cfg, budget, link_bw, layer_s, policy, toks, bias, forest, feats,
            mask_tokens):
    from oracle.sim import OracleStepper
    traces = R.token_traces(log, cfg.num_layers, toks, bias)
    L, M = cfg.num_layers, cfg.num_experts
    cur = {"t": 0}
    holder = {}

    def pregate_fn(tt, layer, h):
        cache = holder["st"].cache
        i = cur["t"] * L + layer
        lg = log[i][0]
        mask = N.routing_mask([(layer + h, e) in cache for e in range(M)], M, cfg.top_k, budget,
                              L, mask_tokens[i], lg[h]) if bias else 0
        return N.batch_gate(lg[h], bias, mask)

    st = OracleStepper(num_layers=L, experts_per_layer=cfg.num_experts, top_k=cfg.top_k,
                       expert_size_bytes=cfg.expert_bytes, link_bw=link_bw,
                       device_memory_bytes=budget * cfg.expert_bytes,
                       layer_compute_ns=round(layer_s * 1e9), policy=oracle_policy(policy),
                       emit_events=True, forest=forest, features_fn=feats,
                       pregate_fn=pregate_fn)
    holder["st"] = st
    mask_bad, sel_bad = [], []

    def hook(layer, resident):
        i = cur["t"] * L + layer
        logits, sel, mask = log[i]
        want = N.routing_mask([(layer, e) in resident for e in range(M)], M, cfg.top_k, budget, L,
                              mask_tokens[i], logits[0]) if bias else 0
        if mask != want:
            mask_bad.append((cur["t"], layer))
        res = N.mask_bits(want, M)
        if not np.array_equal(N.topk_select(logits[0], cfg.top_k, bias, res if bias else None), sel):
            sel_bad.append((cur["t"], layer))
    st.pre_layer_hook = hook
    for t, tt in enumerate(traces):
        cur["t"] = t
        st.run_token(tt)
    return st, mask_bad, sel_bad


POLICIES = [
    ef.PolicyConfig("static", "static"),
    ef.PolicyConfig("static_pre", "static", cold_start="preload"),
    ef.PolicyConfig("reactive", "reactive"),
    ef.PolicyConfig("reactive_pg_car", "reactive", predictor="pregate", cache_aware_routing=True),
    ef.PolicyConfig("fixed2", "fixed_interval", predictor="pregate", interval=2),
    ef.PolicyConfig("adaptive", "adaptive", predictor="pregate"),
    ef.PolicyConfig("adaptive_w", "adaptive", predictor="pregate", recent_window=2,
                    stall_threshold=1, overfetch_threshold=1, cold_start="preload"),
]


@pytest.mark.parametrize("policy", POLICIES, ids=lambda p: p.name)
def test_tiny_f32_engine_parity(policy):
    run_and_check(PRESETS["tiny"], policy, B=3, steps=3, budget=16, link_bw=4 * ef.GB,
                  layer_s=0.0002)


@pytest.mark.parametrize("bias", [0.0, 1e4])
def test_tiny_bf16_batch32_engine_parity(bias):
    """B = 32 (the general route kernel and counting sort); with the
    residency bias the mask is topped up by router votes on the device."""
    run_and_check(PRESETS["tiny-bf16"], ef.PolicyConfig("a", "adaptive", predictor="pregate"),
                  B=32, steps=3, budget=12, link_bw=ef.GB, layer_s=0.0003, bias=bias)


def test_qwen_shape_batch32_topup_parity():
    """Qwen expert shape at B = 32 with the residency bias: the top-up by
    router votes (kernels.cu topup_mask) is bit-exact with the oracle's rule,
    including the pre-gate rows' masks on the host (engine.cu scored_mask)."""
    cfg = MoEConfig("qwen-3l", 3, 60, 4, 2048, 1408, route_mode="softmax_topk", shared_ff=5632,
                    shared_gate=True)
    run_and_check(cfg, ef.PolicyConfig("a", "adaptive", predictor="pregate"), B=32, steps=3,
                  budget=72, link_bw=50 * ef.GB, layer_s=5e-5, bias=1e4)


def test_cache_aware_bias_engine_parity():
    rates = {}
    for bias in (0.0, 1.0, 1e4):
        eng, log = run_and_check(PRESETS["tiny"],
                                 ef.PolicyConfig("a", "adaptive", predictor="pregate"), B=2,
                                 steps=6, budget=12, link_bw=2 * ef.GB, layer_s=0.0002, bias=bias)
        rates[bias] = eng.metrics().hit_rate
        del eng
    # routing toward resident experts can only raise the hit rate on the same inputs
    assert rates[1e4] >= rates[0.0], rates


def test_qwen_shape_shared_gated_expert():
    cfg = MoEConfig("qwen-3l", 3, 60, 4, 2048, 1408, route_mode="softmax_topk", shared_ff=5632,
                    shared_gate=True)
    run_and_check(cfg, ef.PolicyConfig("a", "adaptive", predictor="pregate"), B=8, steps=2,
                  budget=70, link_bw=50 * ef.GB, layer_s=5e-5)


def test_deepseek_shape_shared_experts():
    cfg = MoEConfig("ds-3l", 3, 64, 6, 2048, 1408, route_mode="softmax_topk", shared_ff=2816)
    run_and_check(cfg, ef.PolicyConfig("r", "reactive", predictor="pregate"), B=4, steps=2,
                  budget=60, link_bw=50 * ef.GB, layer_s=5e-5)


def test_forest_predictor_in_engine():
    import goldens as G
    case = G.load("forest.json")[0]
    forest = ef.model_from_json(case["forest"])
    model = ef.ModelSpec(**case["model"])
    table = ef.build_embedding_table(model, ef.Seed(case["table_seed"]))
    cfg = MoEConfig("forest6", 6, 8, 2, 256, 256, dtype="f32", embed_dim=8, vocab_size=64)
    run_and_check(cfg, ef.PolicyConfig("f", "adaptive", predictor="forest"), B=2, steps=3,
                  budget=20, link_bw=2 * ef.GB, layer_s=1e-4, forest=forest, table=table,
                  token_ids=[(1, 2), (3, 4), (1, 2)])


def _slot_matches(eng, cfg, layer, expert, seed):
    import ctypes as C
    from paper_2510_26730_b200 import _lib as L
    s = eng.slot_of(layer, expert)
    if s < 0:
        return None
    es = cfg.elem_bytes
    n = cfg.d_model * cfg.d_ff
    key = N.stream_key(seed, layer, expert, 0)
    ref = torch.empty(n, dtype=torch.bfloat16 if es == 2 else torch.float32, device=DEV)
    L.check(L.lib.ef_fill_uniform(C.c_void_p(torch.cuda.current_stream().cuda_stream),
                                  C.c_void_p(ref.data_ptr()), 1 if es == 2 else 0, n, key,
                                  float(N.fan_scale(cfg.d_model)), 0))
    torch.cuda.synchronize()
    got = eng.slab_view(s)[: n * es]
    return bool(torch.equal(got, ref.view(torch.uint8)))


def test_mixtral_full_size_decisions_and_slab_contents():
    """Full Mixtral-8x7B shape at a 40% budget (102 of 256 experts): the
    decision trace is bit-exact, outputs are finite, and every resident
    slot holds the right expert's W1 bytes."""
    cfg = PRESETS["mixtral-8x7b"]
    eng, log = run_and_check(cfg, ef.PolicyConfig("a", "adaptive", predictor="pregate"), B=1,
                             steps=2, budget=102, link_bw=55 * ef.GB, layer_s=1e-4, seed=3,
                             check_numerics=False)
    checked = 0
    for layer in range(0, cfg.num_layers, 5):
        for e in range(cfg.num_experts):
            ok = _slot_matches(eng, cfg, layer, e, 3)
            if ok is not None:
                assert ok, (layer, e)
                checked += 1
    assert checked > 0


def test_step_host_matches_device_step():
    """MoEEngine.step_host (pinned host buffers, zero-copy I/O) produces the
    same bytes as step() on a device tensor, over several tokens, for two
    engines driven in lockstep with identical inputs."""
    cfg = PRESETS["tiny"]
    pol = ef.PolicyConfig("a", "adaptive", predictor="pregate")
    kw = dict(budget_experts=16, policy=pol, link_bw=4 * ef.GB, layer_time_s=0.0002, max_batch=3,
              seed=5, routing_bias=1.0)
    e_dev, e_host = MoEEngine(cfg, **kw), MoEEngine(cfg, **kw)
    for t in range(4):
        h = synthetic_hidden(cfg, 5, t, 3, DEV)
        hin = h.cpu().pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        e_dev.step(h)
        e_host.step_host(hin, hout)
        torch.cuda.synchronize()
        assert torch.equal(hout, h.cpu()), t
        # in place (h_out aliases h_in)
        h2 = synthetic_hidden(cfg, 5, 100 + t, 3, DEV)
        hin2 = h2.cpu().pin_memory()
        e_dev.step(h2)
        e_host.step_host(hin2)
        torch.cuda.synchronize()
        assert torch.equal(hin2, h2.cpu()), t
    with pytest.raises(ValueError):
        e_host.step_host(torch.zeros(3, cfg.d_model))  # not pinned


@pytest.mark.parametrize("shape,bias", [("tiny", 0.0), ("tiny", 1e4), ("qwen", 0.0),
                                        ("qwen", 1e4), ("deepseek", 0.0)])
def test_prefill_then_decode_parity(shape, bias):
    """Prefill (tcgen05/TMA grouped GEMM path) of T tokens as one scheduler
    step, then decode steps from the same cache: every decision bit-exact
    with the oracle replay (with the residency bias too: prefill masks are
    residents-only, mask_tokens = 0), every router row within fp32 rounding
    of x_l . W_r^T, every layer input and output within the bf16 tolerance."""
    if shape == "tiny":
        cfg, T, B, budget = PRESETS["tiny-bf16"], 96, 2, 12
    elif shape == "qwen":
        cfg = MoEConfig("qwen-2l", 2, 60, 4, 2048, 1408, dtype="bf16", route_mode="softmax_topk",
                        shared_ff=5632, shared_gate=True)
        T, B, budget = 160, 4, 80
    else:  # DeepSeek-V2-Lite expert shape: 64 experts top-6, two ungated shared experts
        cfg = MoEConfig("ds-2l", 2, 64, 6, 2048, 1408, dtype="bf16", route_mode="softmax_topk",
                        shared_ff=2816)
        T, B, budget = 256, 2, 100
    pol = ef.PolicyConfig("a", "adaptive", predictor="pregate")
    link_bw, layer_s, seed = 4 * ef.GB, 2e-4, 3
    eng = MoEEngine(cfg, budget_experts=budget, policy=pol, link_bw=link_bw, layer_time_s=layer_s,
                    max_batch=B, seed=seed, record_routing=True, emit_events=True, max_prefill=T,
                    routing_bias=bias)
    hs_in, hs_out, toks = [], [], []
    h = synthetic_hidden(cfg, seed, 0, T, DEV)
    hs_in.append(h.cpu().numpy())
    eng.prefill(h, list(range(T)))
    torch.cuda.synchronize()
    hs_out.append(h.cpu().numpy())
    toks.append(tuple(range(T)))
    for t in range(1, 3):
        h = synthetic_hidden(cfg, seed, t, B, DEV)
        hs_in.append(h.cpu().numpy())
        eng.step(h, [1000 + t])
        torch.cuda.synchronize()
        hs_out.append(h.cpu().numpy())
        toks.append((1000 + t,))
    log = eng.routing_log()
    xs = eng.routing_x()
    L = cfg.num_layers
    assert len(log) == len(xs) == 3 * L
    assert log[0][1].shape == (T, cfg.top_k)
    assert [m for _, m in xs] == [0] * L + [B] * (2 * L)
    st, mask_bad, sel_bad = _replay(log, cfg, budget, link_bw, layer_s, pol, toks, bias, None, None,
                                    [m for _, m in xs])
    assert not mask_bad and not sel_bad, (mask_bad[:3], sel_bad[:3])
    got = R.product_metrics_dict(eng.metrics(), eng.cache_events())
    assert R.diff_dicts(got, R.oracle_metrics_dict(st)) == []
    w = N.ModelWeights(L=L, M=cfg.num_experts, d=cfg.d_model, ff=cfg.d_ff, dtype=cfg.dtype,
                       seed=seed, shared_ff=cfg.shared_ff, shared_gate=cfg.shared_gate, cache=True)
    check_router_rows(log, xs, w, L)
    check_layer_numerics(hs_in, hs_out, log, xs, w, cfg)
    assert eng.stats()["steps"] == 2


@pytest.mark.parametrize("shape", ["mixtral", "qwen", "deepseek"])
def test_b1_headline_path_numerics(shape):
    """The batch-1 decode path the headline runs — router_route_row_kernel
    (one CTA per router row, the previous layer's combine + rmsnorm folded
    in), device-side slot resolution, the fused gate/up + down GEMVs — at the
    real expert shapes with L = 2 and the residency-first bias of the bench:
    every router row (incl. pre-gate rows) within fp32 rounding, every layer
    input x_l and every step output within the bf16 tolerance, decisions
    bit-exact."""
    if shape == "mixtral":
        cfg, budget = MoEConfig("mixtral-2l", 2, 8, 2, 4096, 14336), 6
    elif shape == "qwen":
        cfg = MoEConfig("qwen-2l", 2, 60, 4, 2048, 1408, route_mode="softmax_topk",
                        shared_ff=5632, shared_gate=True)
        budget = 48
    else:
        cfg = MoEConfig("ds-2l", 2, 64, 6, 2048, 1408, route_mode="softmax_topk", shared_ff=2816)
        budget = 51
    eng, _ = run_and_check(cfg, ef.PolicyConfig("a", "adaptive", predictor="pregate"), B=1,
                           steps=3, budget=budget, link_bw=50 * ef.GB, layer_s=1e-4, seed=4,
                           bias=1e4, timing=True)
    assert eng.stats()["fast_layers"] > 0  # the device-resolved (headline) path ran


@pytest.mark.parametrize("shape,mega,B", [("qwen", "1", 1), ("qwen", "1", 8), ("qwen", "0", 1),
                                          ("deepseek", "1", 4), ("mixtral", "2", 1),
                                          ("tiny", "2", 8)])
def test_layer_kernel_parity(monkeypatch, shape, mega, B):
    """The persistent one-launch-per-layer decode kernel (decode_layer.cuh:
    previous combine + rmsnorm, router rows, the route computed by every
    worker from the logits, shared + routed expert units on mma.sync) against
    the oracle: decisions bit-exact, router rows and layer inputs within fp32
    rounding, outputs within the bf16 tolerance.  EF_MEGA=2 forces it on
    shapes without a shared expert, EF_MEGA=0 runs the classic pipeline; the
    engine reports which one ran."""
    monkeypatch.setenv("EF_MEGA", mega)
    if shape == "mixtral":
        cfg, budget = MoEConfig("mixtral-2l", 2, 8, 2, 4096, 14336), 6
    elif shape == "qwen":
        cfg = MoEConfig("qwen-3l", 3, 60, 4, 2048, 1408, route_mode="softmax_topk",
                        shared_ff=5632, shared_gate=True)
        budget = 72
    elif shape == "deepseek":
        cfg = MoEConfig("ds-2l", 2, 64, 6, 2048, 1408, route_mode="softmax_topk", shared_ff=2816)
        budget = 51
    else:
        cfg, budget = PRESETS["tiny-bf16"], 12
    eng, _ = run_and_check(cfg, ef.PolicyConfig("a", "adaptive", predictor="pregate"), B=B,
                           steps=3, budget=budget, link_bw=50 * ef.GB, layer_s=1e-4, seed=5,
                           bias=1e4, timing=True)
    ran = eng.stats()["layer_kernel_steps"]
    assert (ran > 0) == (mega != "0"), ran


@pytest.mark.parametrize("fuse,pdl", [("0", "1"), ("1", "1"), ("3", "1"), ("11", "0"), ("27", "0"),
                                      ("19", "1")])
def test_pipeline_variants_parity(monkeypatch, fuse, pdl):
    """Every EF_FUSE / EF_PDL combination of the decode pipeline (separate or
    fused router+route, gate, combine-in-router, device-side slot resolution,
    programmatic dependent launch) gives the oracle's decisions and outputs."""
    monkeypatch.setenv("EF_FUSE", fuse)
    monkeypatch.setenv("EF_PDL", pdl)
    run_and_check(PRESETS["tiny"], ef.PolicyConfig("a", "adaptive", predictor="pregate"), B=2,
                  steps=3, budget=12, link_bw=2 * ef.GB, layer_s=0.0002, bias=1e4)


def test_shared_host_store_attach():
    """Two engines on one node sharing one pinned host expert store (POSIX
    shared memory): the second attaches to the store the first filled and
    decodes identically (the replica path of bench.py --gpus N)."""
    import os
    cfg = PRESETS["tiny-bf16"]
    pol = ef.PolicyConfig("a", "adaptive", predictor="pregate")
    kw = dict(budget_experts=12, policy=pol, link_bw=2 * ef.GB, layer_time_s=2e-4, max_batch=2,
              seed=9, routing_bias=1e4)
    name = f"/ef_test_store_{os.getpid()}"
    a = MoEEngine(cfg, host_store_shm=name, **kw)
    b = MoEEngine(cfg, host_store_shm=name, host_store_attach=True, **kw)
    for t in range(4):
        h1 = synthetic_hidden(cfg, 9, t, 2, DEV)
        h2 = h1.clone()
        a.step(h1)
        b.step(h2)
        torch.cuda.synchronize()
        assert torch.equal(h1, h2), t
    assert a.stats()["copies"] == b.stats()["copies"] > 0


def test_activation_log_round_trip():
    """GPU decode -> activation-log lines in the reference's wire format ->
    parse_activation_log gives back the engine's samples (the input of the
    reference's offline forest training)."""
    cfg = MoEConfig("forest6", 6, 8, 2, 256, 256, dtype="f32", embed_dim=8, vocab_size=64)
    eng = MoEEngine(cfg, budget_experts=20, policy=ef.PolicyConfig("a", "adaptive",
                                                                   predictor="pregate"),
                    link_bw=2 * ef.GB, layer_time_s=1e-4, max_batch=2, seed=4)
    for t in range(4):
        eng.step(synthetic_hidden(cfg, 4, t, 2, DEV), [3 * t, 3 * t + 1])
    torch.cuda.synchronize()
    lines = eng.activation_log()
    samples = eng.metrics().samples
    assert lines and len(lines) == len(samples)
    parsed = ef.parse_activation_log(lines, cfg.model_spec())
    key = lambda x: (tuple(x.token_ids), x.layer_idx, tuple(x.predicted_experts),  # noqa: E731
                     tuple(x.actual_experts), x.step_size)
    assert [key(x) for x in parsed] == [key(x) for x in samples]
    assert all(s.token_ids in ((3 * t, 3 * t + 1) for t in range(4)) for s in parsed)


def test_compare_engines_report():
    """compare-style reporting for real decode: the reactive baseline and the
    adaptive policy over the same hidden-state sequences, in the reference's
    comparison-table schema (header and paired reductions)."""
    cfg = PRESETS["tiny"]
    pols = [ef.PolicyConfig("reactive", "reactive"),
            ef.PolicyConfig("adaptive", "adaptive", predictor="pregate")]
    work = [[synthetic_hidden(cfg, 20 + w, t, 2, DEV) for t in range(3)] for w in range(2)]
    res = ef.compare_engines(cfg, pols, work, budget_experts=12, link_bw=2 * ef.GB,
                             layer_time_s=2e-4, seed=3)
    lines = res.to_csv().strip().split("\n")
    assert lines[0] == ("workload,policy,waiting_ns,cache_miss_ns,total_ns,final_step,"
                        "hit_rate,miss_rate,reduction_pct")
    assert len(lines) == 1 + 2 * 2
    for w in range(2):
        base = res.reduction_pct[(w, "reactive")]
        assert base is None or base == 0.0
        assert (w, "adaptive") in res.device_ms


@pytest.mark.gpu
def test_peer_hbm_tier_changes_latency_not_decisions(monkeypatch):
    """Peer-HBM miss tier: swap-ins of experts with a home copy
    in the peer pool are served by cudaMemcpyPeerAsync instead of the host
    copy.  The tier changes only where the bytes come from: outputs, the cache
    event trace and every scheduler counter equal the host-only engine's.  On
    a one-GPU box the pool sits on the engine's own device (test-only mode: a
    same-device copy runs on SMs, so the shape must leave SMs free)."""
    monkeypatch.setenv("EF_PEER_SAME_DEVICE", "1")
    cfg = PRESETS["tiny-bf16"]
    pol = ef.PolicyConfig("a", "adaptive", predictor="pregate")
    kw = dict(budget_experts=12, policy=pol, link_bw=2 * ef.GB, layer_time_s=2e-4, max_batch=2,
              seed=5, emit_events=True)
    n_pool = cfg.num_layers * cfg.num_experts // 2
    a = MoEEngine(cfg, **kw)
    b = MoEEngine(cfg, peer_pool_experts=n_pool, **kw)
    for t in range(6):
        h1 = synthetic_hidden(cfg, 5, t, 2, DEV)
        h2 = h1.clone()
        a.step(h1)
        b.step(h2)
        torch.cuda.synchronize()
        assert torch.equal(h1, h2), t
    assert a.cache_events() == b.cache_events()
    import dataclasses
    ma, mb = (dataclasses.replace(m.metrics(), bandwidth_estimate=0.0) for m in (a, b))
    assert ma == mb
    sa, sb = a.stats(), b.stats()
    assert sa["peer_copies"] == 0 and sa["copies"] == sb["copies"]
    assert 0 < sb["peer_copies"] < sb["copies"]
    assert sb["peer_bytes"] == sb["peer_copies"] * cfg.expert_bytes
    # expert-parallel placement: the home copies of rank 0's experts at G=2
    from paper_2510_26730_b200 import ep
    ids = ep.peer_pool_ids(0, cfg.num_layers, cfg.num_experts, 2)
    c = MoEEngine(cfg, peer_pool_experts=len(ids), peer_pool_ids=ids, **kw)
    for t in range(6):
        h1 = synthetic_hidden(cfg, 5, t, 2, DEV)
        c.step(h1)
    torch.cuda.synchronize()
    assert c.cache_events() == a.cache_events()
    assert 0 < c.stats()["peer_copies"] < c.stats()["copies"]
    with pytest.raises(ValueError):
        MoEEngine(cfg, peer_pool_experts=2, peer_pool_ids=[3, 3], **kw)
    monkeypatch.delenv("EF_PEER_SAME_DEVICE")
    with pytest.raises(ValueError):
        MoEEngine(cfg, peer_pool_experts=n_pool, **kw)
    with pytest.raises(ValueError):
        MoEEngine(cfg, peer_pool_experts=-1, **kw)


_IPC_CHILD = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2510_26730_b200 as ef
from paper_2510_26730_b200.runtime import PRESETS, MoEEngine, synthetic_hidden
cfg = PRESETS["tiny-bf16"]
kw = dict(budget_experts=12, policy=ef.PolicyConfig("a", "adaptive", predictor="pregate"),
          link_bw=2 * ef.GB, layer_time_s=2e-4, max_batch=2, seed=5)
n, handle, lh = int(sys.argv[3]), bytes.fromhex(sys.argv[2]), int(sys.argv[4])
a = MoEEngine(cfg, **kw)
b = MoEEngine(cfg, peer_pool_experts=n, peer_ipc_handle=handle, peer_ipc_layout_hash=lh, **kw)
for t in range(6):
    h1 = synthetic_hidden(cfg, 5, t, 2, torch.device("cuda", 0))
    h2 = h1.clone()
    a.step(h1)
    b.step(h2)
    torch.cuda.synchronize()
    assert torch.equal(h1, h2), t
assert a.cache_events() == b.cache_events()
sb = b.stats()
assert 0 < sb["peer_copies"] < sb["copies"], sb
try:  # another id order than the exporter's: refused, never silently wrong bytes
    MoEEngine(cfg, peer_pool_experts=n, peer_pool_ids=list(range(n))[::-1], peer_ipc_handle=handle,
              peer_ipc_layout_hash=lh, **kw)
    raise SystemExit("layout mismatch not detected")
except ValueError:
    pass
print("ipc ok", int(sb["peer_copies"]), int(sb["copies"]))
"""


@pytest.mark.gpu
def test_peer_pool_ipc_across_processes(monkeypatch):
    """One process per GPU: this process fills an export-only peer pool (no
    same-device override needed: its own misses never read it) and exports
    its CUDA IPC handle and layout hash; an engine in another process opens
    it (``peer_ipc_handle``) and serves its misses from it, decoding exactly
    like a host-only engine; an opener with another id order is refused.  On
    a one-GPU box the opener shares the device (test-only same-device mode)."""
    import os
    import subprocess
    import sys
    cfg = PRESETS["tiny-bf16"]
    n_pool = cfg.num_layers * cfg.num_experts // 2
    owner = MoEEngine(cfg, budget_experts=12, policy=ef.PolicyConfig("a", "adaptive",
                                                                     predictor="pregate"),
                      link_bw=2 * ef.GB, layer_time_s=2e-4, max_batch=2, seed=5,
                      peer_pool_experts=n_pool, peer_pool_export=True)
    handle, lh = owner.peer_pool_handle()
    assert len(handle) == 64
    for t in range(2):  # the exporter's own decode never reads its pool
        owner.step(synthetic_hidden(cfg, 5, t, 2, DEV))
    torch.cuda.synchronize()
    assert owner.stats()["peer_copies"] == 0
    monkeypatch.setenv("EF_PEER_SAME_DEVICE", "1")  # inherited by the child process
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _IPC_CHILD, root, handle.hex(), str(n_pool), str(lh)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ipc ok" in r.stdout, r.stdout + r.stderr
    owner.close()


def test_reset_equals_fresh_engine():
    """MoEEngine.reset(policy, bias) — the bench's grid / baselines reuse one
    engine — behaves exactly like a new engine: same outputs, cache event
    trace and scheduler metrics on the same inputs."""
    cfg = PRESETS["tiny-bf16"]
    kw = dict(budget_experts=12, link_bw=2 * ef.GB, layer_time_s=2e-4, max_batch=2, seed=6,
              emit_events=True)
    a = MoEEngine(cfg, policy=ef.PolicyConfig("r", "reactive"), routing_bias=0.0, **kw)
    for t in range(3):
        a.step(synthetic_hidden(cfg, 6, 50 + t, 2, DEV))
    pol = ef.PolicyConfig("a", "adaptive", predictor="pregate")
    a.reset(pol, 1e4)
    b = MoEEngine(cfg, policy=pol, routing_bias=1e4, **kw)
    for t in range(5):
        h1 = synthetic_hidden(cfg, 6, t, 2, DEV)
        h2 = h1.clone()
        a.step(h1)
        b.step(h2)
        torch.cuda.synchronize()
        assert torch.equal(h1, h2), t
    assert a.cache_events() == b.cache_events()
    assert a.metrics() == b.metrics()
    with pytest.raises(ValueError):
        a.reset(ef.PolicyConfig("a", "adaptive", predictor="pregate", cum_threshold=0.5))


def test_physical_bandwidth_estimate_and_feedback():
    """A13: the copy engine's measured transfer rates feed an EWMA next to the
    logical one; with bandwidth_feedback the adaptive controller re-bases S
    on it.  Off (default) keeps the reference's decisions."""
    cfg = PRESETS["tiny-bf16"]
    kw = dict(budget_experts=12, policy=ef.PolicyConfig("a", "adaptive", predictor="pregate"),
              link_bw=2 * ef.GB, layer_time_s=2e-4, max_batch=2, seed=8)
    a = MoEEngine(cfg, **kw)
    b = MoEEngine(cfg, bandwidth_feedback=True, **kw)
    for t in range(6):
        a.step(synthetic_hidden(cfg, 8, t, 2, DEV))
        b.step(synthetic_hidden(cfg, 8, t, 2, DEV))
    torch.cuda.synchronize()
    sa, sb = a.stats(), b.stats()
    assert sa["bw_physical_transfers"] > 0 and sb["bw_physical_transfers"] > 0
    # 1.5 MB blobs over PCIe: well above 1 GB/s, below the 64 GB/s link
    assert 1e9 < sa["bw_physical_Bps"] < 80e9, sa["bw_physical_Bps"]
    assert abs(a.metrics().bandwidth_estimate - 2 * ef.GB) < 0.01 * ef.GB  # logical clock's EWMA
