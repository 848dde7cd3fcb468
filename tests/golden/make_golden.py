"""Generate the golden fixtures from the REAL reference (run in the build
container only; /root/reference does not exist on the GPU box).

    python tests/golden/make_golden.py

Imports ``moesim`` read-only from /root/reference/pkg/src and writes JSON into
tests/golden/.  The fixtures pin the oracle (oracle/) and, through it and
directly, the product's decision logic.  Every case records the inputs it
was produced from, so consumers never need the reference at run time.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import moesim  # noqa: E402
from moesim import (  # noqa: E402
    GB, MB, BandwidthEstimator, ExpertCache, ExpertId, ForestHyper, HardwareSpec,
    ModelSpec, NoiseConfig, PolicyConfig, PredictionCache, Seed, StepState, TIER_HIGH,
    TIER_LOW, TokenBatch, TraceGenConfig, build_embedding_table, build_features,
    compute_step, expected_expert_count, generate_trace, group_requests, model_to_json,
    on_overfetch, on_stall, pregate_signal, route_batch, simulate, swap_in_latency,
    top_experts, train,
)
from moesim.engine import _Sim  # noqa: E402


def dump(name, obj):
    path = os.path.join(HERE, name)
    with open(path, "w") as f:
        json.dump(obj, f, separators=(",", ":"), sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def trace_json(tr):
    return {
        "token_ids": list(tr.batch.token_ids),
        "gates": [list(map(float, g.probs)) for g in tr.per_layer_gate],
        "actual": [list(a) for a in tr.per_layer_actual],
        "group_actual": [[list(g) for g in layer] for layer in tr.per_layer_group_actual],
        "group_sizes": list(tr.group_sizes),
    }


def metrics_json(m):
    return {
        "policy": m.policy, "total_time_ns": m.total_time_ns, "compute_ns": m.compute_ns,
        "waiting_ns": m.waiting_ns, "cache_miss_ns": m.cache_miss_ns,
        "prefetch_ns": m.prefetch_ns, "cold_start_ns": m.cold_start_ns, "hits": m.hits,
        "misses": m.misses, "admissions": m.admissions, "evictions": m.evictions,
        "stall_events": m.stall_events, "overfetch_events": m.overfetch_events,
        "prediction_cache_hits": m.prediction_cache_hits,
        "prediction_cache_misses": m.prediction_cache_misses,
        "bandwidth_estimate": m.bandwidth_estimate, "final_step": m.final_step,
        "n_selected": m.miss_stats.n_selected, "n_total": m.miss_stats.n_total,
        "hit_rate": m.hit_rate, "miss_rate": m.miss_rate,
        "step_history": [list(x) for x in m.step_history],
        "per_layer": [[r.layer, r.start_ns, r.end_ns, r.stall_ns, r.step, list(r.predicted),
                       list(r.actual), r.demand_misses] for r in m.per_layer],
        "samples": [[list(s.token_ids), s.layer_idx, list(s.predicted_experts),
                     list(s.actual_experts), s.step_size] for s in m.samples],
        "events": None if m.events is None else [[e.time_ns, e.kind, e.seq, e.detail] for e in m.events],
    }


def policy_json(p):
    return {"name": p.name, "strategy": p.strategy, "predictor": p.predictor,
            "interval": p.interval, "cache_aware_routing": p.cache_aware_routing,
            "cold_start": p.cold_start, "cum_threshold": p.cum_threshold,
            "stall_threshold": p.stall_threshold, "overfetch_threshold": p.overfetch_threshold,
            "min_step": p.min_step, "max_step": p.max_step, "recent_window": p.recent_window,
            "noise_decay_rate": p.noise.decay_rate,
            "prediction_cache_capacity": p.prediction_cache_capacity}


def model_json(m):
    return {"num_layers": m.num_layers, "experts_per_layer": m.experts_per_layer,
            "top_k": m.top_k, "expert_size_bytes": m.expert_size_bytes,
            "embed_dim": m.embed_dim, "vocab_size": m.vocab_size}


def hw_json(h):
    return {"link_bandwidth_bytes_per_sec": h.link_bandwidth_bytes_per_sec,
            "device_memory_bytes": h.device_memory_bytes,
            "layer_compute_time_sec": h.layer_compute_time_sec}


# ------------------------------------------------------------------ primitives
def primitives():
    rng = Seed(1234).rng()
    out = {"count": [], "top": [], "compute_step": [], "swap": [], "ewma": [], "predcache": [], "route_batch": [], "seed_split": []}
    for i in range(300):
        m = int(rng.integers(1, 65))
        kind = i % 4
        if kind == 0:
            p = rng.dirichlet(np.ones(m) * float(rng.uniform(0.05, 2.0)))
        elif kind == 1:  # many exact ties
            p = rng.integers(0, 4, m).astype(np.float64) + 1.0
            p = p / p.sum()
        elif kind == 2:
            p = np.full(m, 1.0 / m)
        else:
            p = np.zeros(m)
            p[int(rng.integers(0, m))] = 1.0
        thr = float(rng.choice([0.9, 0.5, 0.8, 0.99, 1.0, float(rng.uniform(0.01, 1.0))]))
        out["count"].append({"probs": p.tolist(), "thr": thr, "n": expected_expert_count(p, thr)})
        c = int(rng.integers(0, m + 1))
        out["top"].append({"probs": p.tolist(), "count": c, "sel": list(top_experts(p, c))})
    for i in range(200):
        n_e = int(rng.integers(0, 64))
        e_s = int(rng.integers(1, 700 * MB))
        bw = int(rng.integers(1, 200 * GB))
        t_l = int(rng.integers(1, 10**8))
        lo = int(rng.integers(1, 5))
        hi = lo + int(rng.integers(0, 40))
        out["compute_step"].append({"args": [n_e, e_s, bw, t_l, lo, hi], "float": False,
                                    "s": compute_step(n_e, e_s, bw, t_l, lo, hi)})
        fbw = float(bw) * float(rng.uniform(0.5, 1.5))
        out["compute_step"].append({"args": [n_e, e_s, fbw, t_l, lo, hi], "float": True,
                                    "s": compute_step(n_e, e_s, fbw, t_l, lo, hi)})
        out["swap"].append({"args": [n_e, e_s, bw], "ns": swap_in_latency(n_e, e_s, bw)})
    for i in range(30):
        alpha = float(rng.choice([0.25, 0.5, 1.0, float(rng.uniform(0.01, 1.0))]))
        prior = None if i % 3 == 0 else float(rng.integers(1, 200 * GB))
        est = BandwidthEstimator(initial=prior, alpha=alpha)
        obs, vals = [], []
        for _ in range(int(rng.integers(1, 20))):
            b = int(rng.integers(0, 700 * MB))
            ns = int(rng.integers(1, 10**9))
            obs.append([b, ns])
            vals.append(est.observe(b, ns))
        out["ewma"].append({"alpha": alpha, "prior": prior, "obs": obs, "est": vals})
    for i in range(10):
        cap = int(rng.integers(1, 6))
        pc = PredictionCache(cap)
        ops, res = [], []
        for j in range(80):
            key = ((int(rng.integers(0, 4)),), int(rng.integers(0, 3)), int(rng.integers(1, 3)))
            if rng.integers(0, 2):
                got = pc.get(key)
                ops.append(["get", [list(key[0]), key[1], key[2]]])
                res.append(None if got is None else got)
            else:
                val = int(rng.integers(0, 100))
                pc.put(key, val)
                ops.append(["put", [list(key[0]), key[1], key[2]], val])
                res.append(None)
        out["predcache"].append({"cap": cap, "ops": ops, "res": res, "hits": pc.hits,
                                 "misses": pc.misses})
    for i in range(40):
        n = int(rng.integers(1, 8))
        groups = [(g, tuple(ExpertId(0, int(e)) for e in sorted(set(rng.integers(0, 6, int(rng.integers(1, 4)))))))
                  for g in range(n)]
        resident = {ExpertId(0, int(e)) for e in range(6) if rng.integers(0, 2)}
        order, deferred = route_batch(groups, resident)
        out["route_batch"].append({"groups": [[g, [e.expert for e in d]] for g, d in groups],
                                   "resident": sorted(e.expert for e in resident),
                                   "order": list(order), "deferred": list(deferred)})
    for v, label in [(0, "embeddings"), (1, "trace:0"), (2**63 + 5, "pregate:3:2"), (2**64 - 1, "x")]:
        out["seed_split"].append([v, label, Seed(v).split(label).value])
    dump("primitives.json", out)


def stepstate_cases():
    rng = Seed(77).rng()
    cases = []
    for i in range(20):
        mx = int(rng.integers(1, 12))
        cur = int(rng.integers(1, mx + 1))
        mn = int(rng.integers(1, cur + 1))
        sth, oth = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        st = StepState(current=cur, max_step=mx, min_step=mn, stall_threshold=sth,
                       overfetch_threshold=oth)
        ops = [int(x) for x in rng.integers(0, 2, 60)]
        seq = []
        for o in ops:
            st = on_stall(st) if o else on_overfetch(st)
            seq.append([st.current, st.stall_count, st.overfetch_count])
        cases.append({"current": cur, "max_step": mx, "min_step": mn, "sth": sth, "oth": oth,
                      "ops": ops, "seq": seq})
    dump("stepstate.json", cases)


def cache_cases():
    rng = Seed(4242).rng()
    cases = []
    for i in range(40):
        cap = int(rng.integers(1, 7))
        cache = ExpertCache(cap * MB + int(rng.integers(0, MB)), MB, record_events=True)
        ids = [(int(l), int(e)) for l in range(3) for e in range(4)]
        ops, outs = [], []
        for step in range(120):
            l, e = ids[int(rng.integers(0, len(ids)))]
            op = int(rng.integers(0, 4))
            if op == 0:
                outs.append(cache.access(ExpertId(l, e), step))
                ops.append(["access", l, e, step])
            elif op == 1:
                tier = TIER_HIGH if rng.integers(0, 2) else TIER_LOW
                v = cache.admit(ExpertId(l, e), tier, step)
                outs.append([[x.layer, x.expert] for x in v])
                ops.append(["admit", l, e, tier, step])
            elif op == 2:
                pred = sorted({ids[int(j)] for j in rng.integers(0, len(ids), int(rng.integers(0, 5)))})
                win = int(rng.integers(0, 6))
                cache.reassign_tiers({ExpertId(a, b) for a, b in pred}, win, step)
                outs.append(None)
                ops.append(["reassign", [list(p) for p in pred], win, step])
            else:
                hit = cache.access(ExpertId(l, e), step)
                v = [] if hit else cache.admit(ExpertId(l, e), TIER_LOW, step)
                outs.append([hit, [[x.layer, x.expert] for x in v]])
                ops.append(["touch", l, e, step])
            cur = sorted((x.layer, x.expert, cache.tier_of(x), cache.last_access(x)) for x in cache.resident)
        cases.append({
            "capacity_bytes": cache.capacity_experts * MB, "expert_size": MB,
            "ops": ops, "outs": outs,
            "final": [list(c) for c in cur],
            "counters": [cache.hits, cache.misses, cache.admissions, cache.evictions],
            "events": [[n, k, x.layer, x.expert] for n, k, x in cache.events],
        })
    dump("cache.json", cases)


# ------------------------------------------------------------------ simulate()
def sim_cases():
    cases = []
    models = [
        ModelSpec(4, 8, 2, 3_145_728, 8, 64),      # C1 tiny shape (fp32 expert bytes)
        ModelSpec(8, 16, 2, 10 * MB, 8, 64),       # tests/test_engine.py GEN_MODEL
        ModelSpec(6, 4, 1, MB, 8, 64),
        ModelSpec(12, 16, 2, 10 * MB, 8, 256),     # README example
    ]
    policies = [
        PolicyConfig("static", "static"),
        PolicyConfig("static_pre", "static", cold_start="preload"),
        PolicyConfig("reactive_none", "reactive"),
        PolicyConfig("reactive_oracle", "reactive", predictor="oracle"),
        PolicyConfig("reactive_pregate", "reactive", predictor="pregate", cache_aware_routing=True),
        PolicyConfig("fixed2_pregate", "fixed_interval", predictor="pregate", interval=2),
        PolicyConfig("fixed3_oracle_car", "fixed_interval", predictor="oracle", interval=3,
                     cache_aware_routing=True, cold_start="preload"),
        PolicyConfig("adaptive_oracle", "adaptive", predictor="oracle"),
        PolicyConfig("adaptive_pregate", "adaptive", predictor="pregate", cache_aware_routing=True),
        PolicyConfig("adaptive_pregate_w", "adaptive", predictor="pregate", recent_window=2,
                     noise=NoiseConfig(0.2), max_step=3),
        PolicyConfig("adaptive_none_pre", "adaptive", cold_start="preload", stall_threshold=1,
                     overfetch_threshold=1),
        PolicyConfig("adaptive_forest", "adaptive", predictor="forest", cache_aware_routing=True),
        PolicyConfig("reactive_forest", "reactive", predictor="forest"),
    ]
    for mi, model in enumerate(models):
        root = Seed(900 + mi)
        table_seed = root.split("embeddings")
        table = build_embedding_table(model, table_seed)
        # a small forest trained on this model's own simulated log (offline path)
        train_samples = []
        seen = set()
        for j in range(12):
            toks = tuple(int(t) for t in root.split(f"tok:{j}").rng().integers(0, model.vocab_size, 1 + j % 4))
            if toks in seen:
                continue
            seen.add(toks)
            tr = generate_trace(model, table, TokenBatch.of(model, toks),
                                TraceGenConfig(persistence=0.7), root.split(f"train:{j}"))
            for s in (1 + j % 2,):
                m = simulate(model, HardwareSpec(8 * GB, 40 * model.expert_size_bytes, 0.005), tr,
                             PolicyConfig("t", "fixed_interval", predictor="pregate", interval=s),
                             root.split(f"trs:{j}"))
                train_samples.extend(m.samples)
        X, Y = build_features(group_requests(train_samples), table, model)
        forest = train(X, Y, ForestHyper(num_trees=6, max_depth=6, residual=(mi % 2 == 1)), root.split("forest"))
        forest_text = model_to_json(forest)
        for ti in range(3):
            n_tok = [1, 3, 5][ti]
            toks = tuple(int(t) for t in root.split(f"q:{ti}").rng().integers(0, model.vocab_size, n_tok))
            tr = generate_trace(model, table, TokenBatch.of(model, toks),
                                TraceGenConfig(persistence=[0.3, 0.8, 0.6][ti]), root.split(f"trace:{ti}"))
            for hi, hw in enumerate([
                HardwareSpec(4 * GB, 6 * model.expert_size_bytes + 123, 0.005),
                HardwareSpec(64 * GB, 3 * model.expert_size_bytes, 0.0011),
                HardwareSpec(1 * GB, 20 * model.expert_size_bytes, 0.002),
            ]):
                if hw.device_memory_bytes < model.top_k * model.expert_size_bytes * 2:
                    continue
                for p in policies:
                    seed = root.split(f"run:{ti}:{hi}")
                    fr = forest if p.predictor == "forest" else None
                    tb = table if p.predictor == "forest" else None
                    try:
                        sim = _Sim(model, hw, tr, p, seed, fr, tb, True)
                        m = sim.run()
                    except RuntimeError as exc:
                        cases.append({"model": model_json(model), "hw": hw_json(hw),
                                      "policy": policy_json(p), "seed": seed.value,
                                      "trace": trace_json(tr), "error": str(exc)})
                        continue
                    cases.append({
                        "model": model_json(model), "hw": hw_json(hw), "policy": policy_json(p),
                        "seed": seed.value, "trace": trace_json(tr),
                        "table_seed": table_seed.value if fr is not None else None,
                        "forest": forest_text if fr is not None else None,
                        "metrics": metrics_json(m),
                        "cache_events": [[n, k, x.layer, x.expert] for n, k, x in sim.cache.events],
                    })
    dump("simulate.json", cases)


def forest_cases():
    model = ModelSpec(6, 8, 2, MB, 8, 64)
    root = Seed(31337)
    table_seed = root.split("embeddings")
    table = build_embedding_table(model, table_seed)
    samples = []
    seen = set()
    for j in range(10):
        toks = tuple(int(t) for t in root.split(f"tok:{j}").rng().integers(0, 64, 2))
        if toks in seen:
            continue
        seen.add(toks)
        tr = generate_trace(model, table, TokenBatch.of(model, toks), TraceGenConfig(persistence=0.6),
                            root.split(f"tr:{j}"))
        m = simulate(model, HardwareSpec(8 * GB, 20 * MB, 0.005), tr,
                     PolicyConfig("t", "fixed_interval", predictor="pregate", interval=2), root)
        samples.extend(m.samples)
    X, Y = build_features(group_requests(samples), table, model)
    out = []
    for residual in (False, True):
        forest = train(X, Y, ForestHyper(num_trees=8, max_depth=5, residual=residual), root.split("f"))
        rows = []
        for i in range(min(len(X), 25)):
            base = np.full(8, 1.0 / 8) if residual else None
            rows.append({"x": X[i].tolist(), "scores": forest.predict_scores(X[i], base).tolist()})
        # inference_features on arbitrary histories
        feats = []
        rng = root.split("feat").rng()
        for i in range(15):
            toks = tuple(int(t) for t in rng.integers(0, 64, int(rng.integers(1, 6))))
            target = int(rng.integers(0, 6))
            hist = {int(l): tuple(sorted(set(int(e) for e in rng.integers(0, 8, 2))))
                    for l in range(int(rng.integers(0, 6)))}
            f = moesim.inference_features(model, table, toks, int(rng.integers(1, 4)), target, hist)
            feats.append({"tokens": list(toks), "target": target, "step": int(f[model.embed_dim]),
                          "hist": {str(k): list(v) for k, v in hist.items()}, "f": f.tolist()})
        out.append({"model": model_json(model), "table_seed": table_seed.value,
                    "forest": model_to_json(forest), "rows": rows, "features": feats})
    dump("forest.json", out)


def pregate_cases():
    model = ModelSpec(8, 16, 2, MB, 8, 64)
    table = build_embedding_table(model, Seed(5))
    tr = generate_trace(model, table, TokenBatch.of(model, (1, 2, 3)), TraceGenConfig(), Seed(6))
    out = {"trace": trace_json(tr), "cases": []}
    for l in range(7):
        for h in range(1, 8 - l):
            for rate in (0.0, 0.6, 2.5):
                out["cases"].append({"l": l, "h": h, "rate": rate, "seed": 4711,
                                     "probs": pregate_signal(tr, l, h, NoiseConfig(rate), Seed(4711)).probs.tolist()})
    dump("pregate.json", out)


def readme_case():
    model = ModelSpec(num_layers=12, experts_per_layer=16, top_k=2, expert_size_bytes=10 * MB,
                      embed_dim=8, vocab_size=256)
    hw = HardwareSpec(link_bandwidth_bytes_per_sec=16 * GB, device_memory_bytes=400 * MB,
                      layer_compute_time_sec=0.005)
    table = build_embedding_table(model, Seed(0))
    trace = generate_trace(model, table, TokenBatch.of(model, (3, 17, 40, 101)),
                           TraceGenConfig(persistence=0.8), Seed(1))
    pols = [PolicyConfig("baseline", "static", cold_start="preload"),
            PolicyConfig("adaptive", "adaptive", predictor="oracle", cold_start="preload",
                         cache_aware_routing=True)]
    res = moesim.run_comparison(model, hw, [trace], pols, Seed(2))
    dump("readme.json", {"model": model_json(model), "hw": hw_json(hw),
                         "policies": [policy_json(p) for p in pols],
                         "run_seed": Seed(2).split("workload:0").value,
                         "trace": trace_json(trace), "csv": res.to_csv()})


if __name__ == "__main__":
    primitives()
    stepstate_cases()
    cache_cases()
    sim_cases()
    forest_cases()
    pregate_cases()
    readme_case()
