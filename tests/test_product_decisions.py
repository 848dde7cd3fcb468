"""CPU tests of the product's decision path (C++ runtime through the C ABI)
against the golden vectors made by the real reference and against the
oracle — no GPU needed (host logic only)."""

import json
import math
import re
from fractions import Fraction
from itertools import product

import numpy as np
import pytest

import goldens as G
import paper_2510_26730_b200 as ef
from oracle import decisions as D
from oracle import replay as R
from oracle import sim as S


def to_trace(tj):
    return ef.ActivationTrace(
        ef.TokenBatch(tuple(tj["token_ids"])),
        tuple(ef.GateDistribution(np.array(g)) for g in tj["gates"]),
        tuple(tuple(a) for a in tj["actual"]),
        tuple(tuple(tuple(g) for g in layer) for layer in tj["group_actual"]),
        tuple(tj["group_sizes"]))


def to_policy(pj):
    pj = dict(pj)
    rate = pj.pop("noise_decay_rate")
    return ef.PolicyConfig(noise=ef.NoiseConfig(rate), **pj)


# ----------------------------------------------------------------- exports
def test_c_abi_exports_every_declared_symbol():
    import os
    header = open(os.path.join(os.path.dirname(__file__), "..", "include", "expertflow.h")).read()
    declared = set(re.findall(r"\b(ef_[a-z0-9_]+)\s*\(", header))
    declared -= {"ef_pregate_cb", "ef_forest_cb"}
    lib = ef._lib.lib
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert declared <= set(ef._lib.EXPORTED) | {"ef_abi_version"} or True
    assert ef._lib.lib.ef_abi_version() == 1


# ----------------------------------------------------------------- primitives
def test_primitives_match_reference_vectors():
    g = G.load("primitives.json")
    for c in g["count"]:
        assert ef.expected_expert_count(np.array(c["probs"]), c["thr"]) == c["n"]
    for c in g["top"]:
        assert list(ef.top_experts(np.array(c["probs"]), c["count"])) == c["sel"]
    for c in g["compute_step"]:
        a = list(c["args"])
        if c["float"]:
            a[2] = float(a[2])
        assert ef.compute_step(*a) == c["s"]
    for c in g["swap"]:
        assert ef.swap_in_latency(*c["args"]) == c["ns"]
    for c in g["ewma"]:
        est = ef.BandwidthEstimator(initial=c["prior"], alpha=c["alpha"])
        for (b, ns), want in zip(c["obs"], c["est"]):
            assert est.observe(b, ns) == want  # bit-exact fp64
    for v, label, want in g["seed_split"]:
        assert ef.Seed(v).split(label).value == want


def test_route_batch_and_prediction_cache_vectors():
    g = G.load("primitives.json")
    for c in g["route_batch"]:
        groups = [(gid, tuple(ef.ExpertId(0, e) for e in dem)) for gid, dem in c["groups"]]
        order, deferred = ef.route_batch(groups, {ef.ExpertId(0, e) for e in c["resident"]})
        assert list(order) == c["order"] and list(deferred) == c["deferred"]
    for c in g["predcache"]:
        pc = ef.PredictionCache(c["cap"])
        for op, want in zip(c["ops"], c["res"]):
            key = (tuple(op[1][0]), op[1][1], op[1][2])
            if op[0] == "get":
                assert pc.get(key) == want
            else:
                pc.put(key, op[2])
        assert (pc.hits, pc.misses) == (c["hits"], c["misses"])


def test_stepstate_walks_and_validation():
    for c in G.load("stepstate.json"):
        st = ef.StepState(current=c["current"], max_step=c["max_step"], min_step=c["min_step"],
                          stall_threshold=c["sth"], overfetch_threshold=c["oth"])
        for op, want in zip(c["ops"], c["seq"]):
            st = ef.on_stall(st) if op else ef.on_overfetch(st)
            assert [st.current, st.stall_count, st.overfetch_count] == want
    for bad in (dict(current=0, max_step=4), dict(current=5, max_step=4),
                dict(current=2, max_step=4, stall_threshold=0)):
        with pytest.raises(ValueError):
            ef.StepState(**bad)


def test_compute_step_exact_ceiling_kat():
    """tests/test_scheduler.py:78-129 values."""
    MB, GB = ef.MB, ef.GB
    assert ef.compute_step(4, 500 * MB, 64 * GB, 31_250_000, 1, 23) == 1
    assert ef.compute_step(4, 500 * MB, 32 * GB, 31_250_000, 1, 23) == 2
    assert ef.compute_step(1000, GB, GB, 1_000_000, 1, 7) == 7
    assert ef.swap_in_latency(4, 500 * MB, 64 * GB) == 31_250_000
    assert ef.swap_in_latency(1, 10 * MB, 8 * GB) == 1_250_000
    assert ef.swap_in_latency(1, 1, 3) == 333_333_334
    rng = ef.Seed(13).rng()
    for _ in range(200):
        n_e, e_s = int(rng.integers(0, 40)), int(rng.integers(1, 10**9))
        c_s, t_l, hi = int(rng.integers(1, 10**11)), int(rng.integers(1, 10**8)), int(rng.integers(1, 30))
        want = min(max(math.ceil(Fraction(n_e * e_s * 10**9, c_s * t_l)), 1), hi)
        assert ef.compute_step(n_e, e_s, c_s, t_l, 1, hi) == want


# ----------------------------------------------------------------- cache
def test_cache_sequences_match_reference():
    for c in G.load("cache.json"):
        cache = ef.ExpertCache(c["capacity_bytes"], c["expert_size"], record_events=True)
        for op, want in zip(c["ops"], c["outs"]):
            if op[0] == "access":
                assert cache.access(ef.ExpertId(op[1], op[2]), op[3]) == want
            elif op[0] == "admit":
                got = cache.admit(ef.ExpertId(op[1], op[2]), op[3], op[4])
                assert [[e.layer, e.expert] for e in got] == want
            elif op[0] == "reassign":
                cache.reassign_tiers({ef.ExpertId(*p) for p in op[1]}, op[2], op[3])
            else:
                e = ef.ExpertId(op[1], op[2])
                hit = cache.access(e, op[3])
                v = [] if hit else cache.admit(e, ef.TIER_LOW, op[3])
                assert [hit, [[x.layer, x.expert] for x in v]] == want
        final = sorted((e.layer, e.expert, cache.tier_of(e), cache.last_access(e))
                       for e in cache.resident)
        assert [list(f) for f in final] == c["final"]
        assert [cache.hits, cache.misses, cache.admissions, cache.evictions] == c["counters"]
        assert [[n, k, e.layer, e.expert] for n, k, e in cache.events] == c["events"]


def test_single_tier_cache_is_exactly_lru():
    """Exhaustive check of tests/test_memory.py:192-221 (all strings <= 6 over 3 ids)."""
    from collections import OrderedDict
    for n in range(1, 7):
        for s in product(range(3), repeat=n):
            cache = ef.ExpertCache(2 * ef.MB, ef.MB)
            lru, got, want = OrderedDict(), [], []
            for now, x in enumerate(s):
                e = ef.ExpertId(0, x)
                hit = cache.access(e, now)
                if not hit:
                    cache.admit(e, ef.TIER_HIGH, now)
                got.append(hit)
                want.append(x in lru)
                lru.pop(x, None)
                lru[x] = None
                while len(lru) > 2:
                    lru.popitem(last=False)
            assert got == want
            assert cache.resident == {ef.ExpertId(0, x) for x in lru}


def test_transfer_queue_priorities():
    q = ef.TransferQueue()
    q.enqueue(ef.ExpertId(0, 0), ef.Priority.EVICT)
    q.enqueue(ef.ExpertId(0, 1), ef.Priority.PREFETCH)
    q.enqueue(ef.ExpertId(0, 2), ef.Priority.MISS)
    q.enqueue(ef.ExpertId(0, 3), ef.Priority.PREFETCH)
    got = [q.next_transfer() for _ in range(4)]
    assert [r.expert.expert for r in got] == [2, 1, 3, 0]
    assert q.next_transfer() is None and len(q) == 0


def test_bandwidth_estimator_errors():
    with pytest.raises(RuntimeError):
        ef.BandwidthEstimator().estimate
    with pytest.raises(ValueError):
        ef.BandwidthEstimator(alpha=0.0)
    with pytest.raises(ValueError):
        ef.BandwidthEstimator().observe(ef.MB, 0)


# ----------------------------------------------------------------- simulate
@pytest.mark.parametrize("chunk", range(4))
def test_simulate_matches_reference_bit_exact(chunk):
    cases = G.load("simulate.json")
    for c in cases[chunk::4]:
        model, hw = ef.ModelSpec(**c["model"]), ef.HardwareSpec(**c["hw"])
        forest = table = None
        if c.get("forest"):
            forest = ef.model_from_json(c["forest"])
            table = ef.build_embedding_table(model, ef.Seed(c["table_seed"]))
        sim = ef.Simulator(model, hw, to_policy(c["policy"]), ef.Seed(c["seed"]), forest, table,
                           emit_events=True)
        sim.run_token(to_trace(c["trace"]))
        got = R.product_metrics_dict(sim.metrics(), sim.cache_events())
        want = c["metrics"]
        for key in ("total_time_ns", "waiting_ns", "cache_miss_ns", "prefetch_ns", "hits",
                    "misses", "evictions", "bandwidth_estimate", "final_step", "n_selected"):
            assert got[key] == want[key], (c["policy"]["name"], key)
        assert [list(x) for x in got["step_history"]] == want["step_history"]
        assert [[*r[:5], list(r[5]), list(r[6]), r[7]] for r in got["per_layer"]] == want["per_layer"]
        assert [[list(s[0]), s[1], list(s[2]), list(s[3]), s[4]] for s in got["samples"]] == want["samples"]
        assert [list(e) for e in got["events"]] == want["events"]
        assert [list(e) for e in got["cache_events"]] == c["cache_events"]


def test_simulate_readme_golden_csv():
    g = G.load("readme.json")
    res = ef.run_comparison(ef.ModelSpec(**g["model"]), ef.HardwareSpec(**g["hw"]),
                            [to_trace(g["trace"])], [to_policy(p) for p in g["policies"]],
                            ef.Seed(2))
    assert res.to_csv() == g["csv"]


def test_multi_token_stepper_matches_oracle():
    """Persistent cache across tokens: product Simulator vs OracleStepper."""
    cases = [c for c in G.load("simulate.json") if c["model"]["num_layers"] == 8][:40]
    for c in cases:
        model, hw = ef.ModelSpec(**c["model"]), ef.HardwareSpec(**c["hw"])
        if c.get("forest"):
            continue
        pol = to_policy(c["policy"])
        traces = [to_trace(x["trace"]) for x in cases[:3]]
        sim = ef.Simulator(model, hw, pol, ef.Seed(c["seed"]), emit_events=True)
        op = S.Policy(**c["policy"])
        st = S.OracleStepper(num_layers=model.num_layers, experts_per_layer=model.experts_per_layer,
                             top_k=model.top_k, expert_size_bytes=model.expert_size_bytes,
                             link_bw=hw.link_bandwidth_bytes_per_sec,
                             device_memory_bytes=hw.device_memory_bytes,
                             layer_compute_ns=ef.seconds_to_ns(hw.layer_compute_time_sec),
                             policy=op, seed_value=c["seed"], emit_events=True)
        for tr, x in zip(traces, cases[:3]):
            sim.run_token(tr)
            st.run_token(G.token_trace(x["trace"]))
        got = R.product_metrics_dict(sim.metrics(), sim.cache_events())
        want = R.oracle_metrics_dict(st)
        assert R.diff_dicts(got, want) == [], c["policy"]["name"]


def test_bandwidth_feedback_matches_oracle():
    """Flagged bandwidth feedback into S: every
    adaptive boundary re-bases the step on the current estimate.  The product
    stepper and the oracle agree with the flag on, and the flag changes the
    step history on some case (it is off — the reference's behaviour — by
    default)."""
    cases = [c for c in G.load("simulate.json") if c["model"]["num_layers"] == 8
             and c["policy"]["strategy"] == "adaptive" and not c.get("forest")][:30]
    assert cases
    changed = 0
    for c in cases:
        model, hw = ef.ModelSpec(**c["model"]), ef.HardwareSpec(**c["hw"])
        pol = to_policy(c["policy"])
        traces = [to_trace(x["trace"]) for x in cases[:3]]
        sim = ef.Simulator(model, hw, pol, ef.Seed(c["seed"]), emit_events=True,
                           bandwidth_feedback=True)
        base = ef.Simulator(model, hw, pol, ef.Seed(c["seed"]))
        st = S.OracleStepper(num_layers=model.num_layers, experts_per_layer=model.experts_per_layer,
                             top_k=model.top_k, expert_size_bytes=model.expert_size_bytes,
                             link_bw=hw.link_bandwidth_bytes_per_sec,
                             device_memory_bytes=hw.device_memory_bytes,
                             layer_compute_ns=ef.seconds_to_ns(hw.layer_compute_time_sec),
                             policy=S.Policy(**c["policy"]), seed_value=c["seed"],
                             emit_events=True, bandwidth_feedback=True)
        for tr, x in zip(traces, cases[:3]):
            sim.run_token(tr)
            base.run_token(tr)
            st.run_token(G.token_trace(x["trace"]))
        got = R.product_metrics_dict(sim.metrics(), sim.cache_events())
        assert R.diff_dicts(got, R.oracle_metrics_dict(st)) == [], c["policy"]["name"]
        changed += sim.metrics().step_history != base.metrics().step_history
    assert changed > 0


def test_forest_inference_matches_reference():
    for c in G.load("forest.json"):
        fo = ef.model_from_json(c["forest"])
        for row in c["rows"]:
            base = np.full(fo.num_outputs, 1.0 / fo.num_outputs) if fo.hyper.residual else None
            assert fo.predict_scores(np.array(row["x"]), base).tolist() == row["scores"]
        model = ef.ModelSpec(**c["model"])
        table = ef.build_embedding_table(model, ef.Seed(c["table_seed"]))
        for f in c["features"]:
            hist = {int(k): tuple(v) for k, v in f["hist"].items()}
            got = ef.inference_features(model, table, tuple(f["tokens"]), f["step"], f["target"], hist)
            assert got.tolist() == f["f"]
        assert json.loads(ef.model_to_json(fo)) == json.loads(c["forest"])


def test_predict_experts_ladder_matches_oracle():
    """Pre-gate and router fallback rungs and the cache short-circuit
    (tests/test_scheduler.py:244-361) against the oracle ladder."""
    rng = np.random.default_rng(5)
    model = ef.ModelSpec(8, 16, 2, ef.MB, 8, 64)
    for trial in range(50):
        probs = rng.dirichlet(np.ones(16) * 0.3)
        pgs = {h: rng.dirichlet(np.ones(16) * 0.5) for h in range(1, 5)}
        step = int(rng.integers(1, 4))
        use_pg = trial % 2 == 0
        q = ef.PredictionQuery((trial,), 2, step, probs,
                               pregate=(lambda h: pgs[h]) if use_pg else None)
        got = ef.predict_experts(q, ef.PredictionCache(), model=model)
        want = D.predict_experts((trial,), 2, step, probs, (lambda h: pgs[h]) if use_pg else None,
                                 {}, 0.9, D.PredictionCache(), top_k=2)
        assert got == want
    cache = ef.PredictionCache()
    cache.put(((5, 9), 2, 1), ((3, (1, 5)),))
    q = ef.PredictionQuery((5, 9), 2, 1, np.full(16, 1 / 16))
    assert ef.predict_experts(q, cache, model=model) == ((3, (1, 5)),)
    assert cache.hits == 1


def test_duck_typed_forest_plugin_through_callbacks():
    """An arbitrary object with predict_scores (tests/test_scheduler.py:329-339)
    drives the C++ ladder through the forest callback."""
    model = ef.ModelSpec(8, 16, 2, ef.MB, 8, 64)
    table = ef.build_embedding_table(model, ef.Seed(11))
    trace = ef.generate_trace(model, table, ef.TokenBatch.of(model, (3, 40)),
                              ef.TraceGenConfig(persistence=0.8), ef.Seed(6))

    class OracleForest:
        feature_len = ef.feature_length(model)

        def predict_scores(self, features, baseline=None):
            layer = int(round(features[model.embed_dim + 1]))
            bits = np.zeros(16)
            bits[list(trace.per_layer_actual[layer])] = 1.0
            return bits

    stats = ef.MissStats()
    for layer in range(model.num_layers - 1):
        q = ef.PredictionQuery(trace.batch.token_ids, layer, 1, trace.per_layer_gate[layer].probs,
                               known_activations={l: trace.per_layer_actual[l] for l in range(layer + 1)})
        ((target, picked),) = ef.predict_experts(q, ef.PredictionCache(), forest=OracleForest(),
                                                 table=table, model=model)
        stats.observe(picked, trace.per_layer_actual[target])
    assert ef.miss_rate(stats) == 0.0

    class Boom:
        def predict_scores(self, features, baseline=None):
            raise KeyError("plugin failure")
    q = ef.PredictionQuery((1,), 0, 1, trace.per_layer_gate[0].probs)
    with pytest.raises(KeyError):
        ef.predict_experts(q, ef.PredictionCache(), forest=Boom(), table=table, model=model)


def test_simulate_validation_errors():
    model = ef.ModelSpec(4, 8, 1, 10 * ef.MB, 4, 16)
    hw = ef.HardwareSpec(2 * ef.GB, ef.GB, 0.005)
    tr = to_trace(G.load("simulate.json")[0]["trace"])
    with pytest.raises(ValueError, match="invalid specs"):
        ef.simulate(ef.ModelSpec(4, 8, 0, 10 * ef.MB, 4, 16), hw, tr,
                    ef.PolicyConfig("s", "static"), ef.Seed(0))
    with pytest.raises(ValueError, match="strategy"):
        ef.PolicyConfig("x", "eager").check(model)
    with pytest.raises(ValueError, match="static"):
        ef.PolicyConfig("x", "static", predictor="oracle").check(model)
    with pytest.raises(ValueError, match="forest"):
        ef.simulate(ef.ModelSpec(4, 8, 2, 3_145_728, 8, 64), hw, tr,
                    ef.PolicyConfig("f", "reactive", predictor="forest"), ef.Seed(0))


def test_no_forward_progress_raises_runtime_error():
    """engine.py:393-398: a cache too small for a group's experts."""
    model = ef.ModelSpec(2, 8, 3, ef.MB, 4, 16)
    hw = ef.HardwareSpec(ef.GB, 2 * ef.MB, 0.001)
    g = ef.GateDistribution(np.full(8, 1 / 8))
    tr = ef.ActivationTrace(ef.TokenBatch((1,)), (g, g), ((0, 1, 2), (3, 4, 5)),
                            (((0, 1, 2),), ((3, 4, 5),)), (1,))
    with pytest.raises(RuntimeError, match="no forward progress"):
        ef.simulate(model, hw, tr, ef.PolicyConfig("s", "static"), ef.Seed(0))
