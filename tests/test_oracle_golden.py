"""Pin the CPU oracle (oracle/) to golden vectors produced by the real
reference (tests/golden/make_golden.py) and to the README CSV
(/root/reference/pkg/README.md:84-88)."""

import math

import numpy as np
import pytest

import goldens as G
from oracle import decisions as D
from oracle import forest as F
from oracle import sim as S


def test_primitives_count_and_top():
    g = G.load("primitives.json")
    for c in g["count"]:
        assert D.expected_expert_count(c["probs"], c["thr"]) == c["n"]
    for c in g["top"]:
        assert list(D.top_experts(c["probs"], c["count"])) == c["sel"]


def test_primitives_compute_step_and_swap():
    g = G.load("primitives.json")
    for c in g["compute_step"]:
        a = c["args"]
        if c["float"]:
            a = [a[0], a[1], float(a[2])] + a[3:]
        assert D.compute_step(*a) == c["s"]
    for c in g["swap"]:
        assert D.swap_in_latency(*c["args"]) == c["ns"]


def test_primitives_ewma_bit_exact():
    for c in G.load("primitives.json")["ewma"]:
        est = D.BandwidthEstimator(initial=c["prior"], alpha=c["alpha"])
        for (b, ns), want in zip(c["obs"], c["est"]):
            assert est.observe(b, ns) == want


def test_primitives_predcache_route_batch_seed():
    g = G.load("primitives.json")
    for c in g["predcache"]:
        pc = D.PredictionCache(c["cap"])
        for op, want in zip(c["ops"], c["res"]):
            key = (tuple(op[1][0]), op[1][1], op[1][2])
            if op[0] == "get":
                assert pc.get(key) == want
            else:
                pc.put(key, op[2])
        assert (pc.hits, pc.misses) == (c["hits"], c["misses"])
    for c in g["route_batch"]:
        groups = [(gid, tuple((0, e) for e in dem)) for gid, dem in c["groups"]]
        order, deferred = D.route_batch(groups, {(0, e) for e in c["resident"]})
        assert list(order) == c["order"] and list(deferred) == c["deferred"]
    for v, label, want in g["seed_split"]:
        assert D.seed_split(v, label) == want


def test_stepstate_walks():
    for c in G.load("stepstate.json"):
        st = D.StepState(c["current"], c["max_step"], c["min_step"], c["sth"], c["oth"])
        for op, want in zip(c["ops"], c["seq"]):
            st.stall() if op else st.overfetch()
            assert [st.current, st.stall_count, st.overfetch_count] == want


def test_cache_op_sequences_and_event_log():
    for c in G.load("cache.json"):
        cache = D.ExpertCache(c["capacity_bytes"], c["expert_size"], record_events=True)
        for op, want in zip(c["ops"], c["outs"]):
            if op[0] == "access":
                assert cache.access((op[1], op[2]), op[3]) == want
            elif op[0] == "admit":
                assert [list(v) for v in cache.admit((op[1], op[2]), op[3], op[4])] == want
            elif op[0] == "reassign":
                cache.reassign_tiers({tuple(p) for p in op[1]}, op[2], op[3])
            else:
                hit = cache.access((op[1], op[2]), op[3])
                v = [] if hit else cache.admit((op[1], op[2]), D.LOW, op[3])
                assert [hit, [list(x) for x in v]] == want
        final = sorted((e[0], e[1], cache.tier[e], cache.last[e]) for e in cache.tier)
        assert [list(f) for f in final] == c["final"]
        assert [cache.hits, cache.misses, cache.admissions, cache.evictions] == c["counters"]
        assert [[n, k, e[0], e[1]] for n, k, e in cache.events] == c["events"]


def _forest_and_features(case):
    if case.get("forest") is None:
        return None, None
    fo = F.Forest.from_json(case["forest"])
    m = case["model"]
    table = F.embedding_table(m["vocab_size"], m["embed_dim"], case["table_seed"])
    L, M = m["num_layers"], m["experts_per_layer"]

    def feats(tokens, step, target, hist):
        return F.features(table, L, M, tokens, step, target, hist)
    return fo, feats


def run_oracle_case(case):
    m, hw = case["model"], case["hw"]
    fo, feats = _forest_and_features(case)
    return S.simulate(
        trace=G.token_trace(case["trace"]), num_layers=m["num_layers"],
        experts_per_layer=m["experts_per_layer"], top_k=m["top_k"],
        expert_size_bytes=m["expert_size_bytes"], link_bw=hw["link_bandwidth_bytes_per_sec"],
        device_memory_bytes=hw["device_memory_bytes"],
        layer_compute_ns=G.seconds_to_ns(hw["layer_compute_time_sec"]),
        policy=G.oracle_policy(case["policy"]), seed_value=case["seed"], emit_events=True,
        forest=fo, features_fn=feats)


def metrics_as_golden(m: S.Metrics):
    return {
        "policy": m.policy, "total_time_ns": m.total_time_ns, "compute_ns": m.compute_ns,
        "waiting_ns": m.waiting_ns, "cache_miss_ns": m.cache_miss_ns, "prefetch_ns": m.prefetch_ns,
        "cold_start_ns": m.cold_start_ns, "hits": m.hits, "misses": m.misses,
        "admissions": m.admissions, "evictions": m.evictions, "stall_events": m.stall_events,
        "overfetch_events": m.overfetch_events,
        "prediction_cache_hits": m.prediction_cache_hits,
        "prediction_cache_misses": m.prediction_cache_misses,
        "bandwidth_estimate": m.bandwidth_estimate, "final_step": m.final_step,
        "n_selected": m.n_selected, "n_total": m.n_total, "hit_rate": m.hit_rate,
        "miss_rate": m.miss_rate, "step_history": [list(x) for x in m.step_history],
        "per_layer": [[r[0], r[1], r[2], r[3], r[4], list(r[5]), list(r[6]), r[7]] for r in m.per_layer],
        "samples": [[list(s[0]), s[1], list(s[2]), list(s[3]), s[4]] for s in m.samples],
        "events": None if m.events is None else [list(e) for e in m.events],
    }


@pytest.mark.parametrize("chunk", range(8))
def test_oracle_simulate_matches_reference(chunk):
    cases = G.load("simulate.json")
    for case in cases[chunk::8]:
        m = run_oracle_case(case)
        got = metrics_as_golden(m)
        want = case["metrics"]
        for key in want:
            assert got[key] == want[key], (case["policy"]["name"], key)


def test_oracle_cache_events_match_reference():
    for case in G.load("simulate.json")[::5]:
        m, hw = case["model"], case["hw"]
        fo, feats = _forest_and_features(case)
        st = S.OracleStepper(
            num_layers=m["num_layers"], experts_per_layer=m["experts_per_layer"],
            top_k=m["top_k"], expert_size_bytes=m["expert_size_bytes"],
            link_bw=hw["link_bandwidth_bytes_per_sec"],
            device_memory_bytes=hw["device_memory_bytes"],
            layer_compute_ns=G.seconds_to_ns(hw["layer_compute_time_sec"]),
            policy=G.oracle_policy(case["policy"]), seed_value=case["seed"], emit_events=True,
            forest=fo, features_fn=feats)
        st.run_token(G.token_trace(case["trace"]))
        assert [[n, k, e[0], e[1]] for n, k, e in st.cache.events] == case["cache_events"]


def test_oracle_forest_scores_and_features():
    for case in G.load("forest.json"):
        fo = F.Forest.from_json(case["forest"])
        for row in case["rows"]:
            base = np.full(fo.num_outputs, 1.0 / fo.num_outputs) if fo.residual else None
            assert fo.predict_scores(row["x"], base).tolist() == row["scores"]
        m = case["model"]
        table = F.embedding_table(m["vocab_size"], m["embed_dim"], case["table_seed"])
        for f in case["features"]:
            hist = {int(k): tuple(v) for k, v in f["hist"].items()}
            got = F.features(table, m["num_layers"], m["experts_per_layer"], f["tokens"],
                             f["step"], f["target"], hist)
            assert got.tolist() == f["f"]


def test_oracle_pregate_signal():
    g = G.load("pregate.json")
    tr = G.token_trace(g["trace"])
    for c in g["cases"]:
        got = D.pregate_signal(tr.gates[c["l"] + c["h"]], c["l"], c["h"], c["rate"], c["seed"])
        assert got.tolist() == c["probs"]


def test_oracle_reproduces_readme_golden_csv():
    """pkg/README.md:84-88, reproduced through the oracle stepper."""
    g = G.load("readme.json")
    rows = []
    base = None
    for pj in g["policies"]:
        case = {"model": g["model"], "hw": g["hw"], "policy": pj, "seed": g["run_seed"],
                "trace": g["trace"]}
        m = run_oracle_case(case)
        lat = m.waiting_ns + m.cache_miss_ns
        if base is None:
            base = lat
        red = "" if base == 0 else repr(100.0 * (1.0 - lat / base))
        rows.append(f"0,{m.policy},{m.waiting_ns},{m.cache_miss_ns},{m.total_time_ns},"
                    f"{m.final_step},{m.hit_rate!r},{m.miss_rate!r},{red}")
    want = g["csv"].strip().split("\n")[1:]
    assert rows == want
    assert want == ["0,baseline,38125000,46250000,98125000,0,0.08641975308641975,0.0,0.0",
                    "0,adaptive,0,0,60000000,2,1.0,0.0,100.0"]


def test_oracle_closed_form_kats():
    """tests/test_engine.py:90-103 and :106-115 closed-form timelines."""
    T = 5_000_000
    MB, GB = 1_000_000, 1_000_000_000
    tr = S.TokenTrace(token_ids=(1,),
                      gates=[np.array([0.99 if e == l else 0.01 / 7 for e in range(8)]) for l in range(4)],
                      actual=[(l,) for l in range(4)],
                      group_actual=[((l,),) for l in range(4)], group_sizes=(1,))
    pol = S.Policy("r", "reactive", predictor="oracle", cold_start="preload")
    kw = dict(num_layers=4, experts_per_layer=8, top_k=1, expert_size_bytes=10 * MB,
              device_memory_bytes=GB, layer_compute_ns=T, policy=pol)
    m = S.simulate(trace=tr, link_bw=2 * GB, **kw)
    assert (m.waiting_ns, m.total_time_ns, m.prefetch_ns, m.cold_start_ns) == (0, 4 * T, 3 * T, T)
    m = S.simulate(trace=tr, link_bw=GB, **kw)
    assert (m.waiting_ns, m.total_time_ns, m.stall_events) == (3 * T, 7 * T, 3)
