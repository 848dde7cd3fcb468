"""Replay a B200 engine run through the oracle — TEST INFRASTRUCTURE.

Given the routing the GPU produced (the engine's routing log: per executed
layer the scored fp32 router logits [R, B, M] and the selection [B, k]),
rebuild the scheduler inputs with the canonical adapter of
oracle/numerics.py (fp64 softmax, sequential sums, one group per token) and
run the OracleStepper, which restates /root/reference/pkg/src/moesim/
engine.py:_Sim.  The result must equal the engine's decisions bit for bit:
that is the "given identical fp32 gate logits" parity of the north star.
"""

from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np

from . import numerics as N
from .sim import OracleStepper, Policy, TokenTrace


def token_traces(log, L: int, tokens_per_step: Sequence[Sequence[int]],
                 bias: float = 0.0) -> List[TokenTrace]:
    out = []
    for t, toks in enumerate(tokens_per_step):
        gates, actual, grouped = [], [], []
        for l in range(L):
            logits, sel, mask = log[t * L + l]
            gates.append(N.batch_gate(logits[0], bias, mask))
            g = tuple(tuple(sorted(int(e) for e in row)) for row in sel)
            grouped.append(g)
            actual.append(tuple(sorted(set().union(*g))))
        out.append(TokenTrace(tuple(toks), gates, actual, grouped, tuple([1] * sel.shape[0])))
    return out


def replay(log, *, L, M, k, expert_bytes, link_bw, budget_experts, layer_ns, policy: Policy,
           tokens_per_step, bias: float = 0.0, emit_events=True, mask_tokens=None):
    """Returns (stepper, mask_mismatches, selection_mismatches).
    ``mask_tokens[i]``: the token count the engine's bias-mask top-up rule
    used for log entry i (MoEEngine.routing_x(); 0 for prefill layers);
    default: the entry's batch size."""
    traces = token_traces(log, L, tokens_per_step, bias)
    cur = {"t": 0}
    holder = {}

    def ntok(i):
        return log[i][0].shape[1] if mask_tokens is None else mask_tokens[i]

    def pregate_fn(tt, layer, h):
        i = cur["t"] * L + layer
        logits = log[i][0]
        cache = holder["st"].cache
        mask = N.routing_mask([(layer + h, e) in cache for e in range(M)], M, k, budget_experts,
                              L, ntok(i), logits[h]) if bias else 0
        return N.batch_gate(logits[h], bias, mask)

    st = OracleStepper(num_layers=L, experts_per_layer=M, top_k=k, expert_size_bytes=expert_bytes,
                       link_bw=link_bw, device_memory_bytes=budget_experts * expert_bytes,
                       layer_compute_ns=layer_ns, policy=policy, emit_events=emit_events,
                       pregate_fn=pregate_fn)
    holder["st"] = st
    mask_bad, sel_bad = [], []

    def hook(layer, resident):
        i = cur["t"] * L + layer
        logits, sel, mask = log[i]
        want = N.routing_mask([(layer, e) in resident for e in range(M)], M, k, budget_experts,
                              L, ntok(i), logits[0]) if bias else 0
        if mask != want:
            mask_bad.append((cur["t"], layer, mask, want))
        ref = N.topk_select(logits[0], k, bias, N.mask_bits(want, M) if bias else None)
        if not np.array_equal(ref, sel):
            sel_bad.append((cur["t"], layer))

    st.pre_layer_hook = hook
    for t, tt in enumerate(traces):
        cur["t"] = t
        st.run_token(tt)
    return st, mask_bad, sel_bad


def forward_step(h0: np.ndarray, log, step: int, weights: N.ModelWeights, L: int, k: int,
                 mode: str, xs=None, x_errs: Optional[list] = None) -> np.ndarray:
    """fp64 oracle of one decode step using the GPU's logits for selection.
    With ``xs`` (MoEEngine.routing_x()), the GPU's router input of every layer
    is compared with the oracle's x_l = rmsnorm(h_l): the relative error of
    each layer is appended to ``x_errs`` as (step, layer, err)."""
    h = np.asarray(h0, dtype=np.float64)
    for l in range(L):
        logits, sel, _mask = log[step * L + l]
        out = N.moe_layer(h, weights, l, k, mode, logits_override=logits[0], sel_override=sel)
        if xs is not None and x_errs is not None:
            x_errs.append((step, l, rel_err(xs[step * L + l][0], out["x"])))
        h = out["h_next"]
    return h


def router_row_errors(log, xs, weights: N.ModelWeights, L: int):
    """Every router row the GPU scored — the layer's own row (h = 0) and every
    pre-gate row (h >= 1, layer l+h's router applied to x_l, kernel (b)) —
    against the fp64 product x_l . W_r^(l+h)^T of the GPU's own x_l, so the
    check isolates the router GEMV from the layers before it.  Returns
    [(entry, h, token, rel_err)] with rel_err = ||gpu - ref|| / ||ref|| over
    the M logits of one token."""
    out = []
    for i, ((logits, _sel, _mask), (x, _mt)) in enumerate(zip(log, xs)):
        l = i % L
        x64 = np.asarray(x, np.float64)
        for h in range(logits.shape[0]):
            ref = N.router_logits(x64, weights.router(l + h))
            for t in range(ref.shape[0]):
                out.append((i, h, t, rel_err(logits[h][t], ref[t])))
    return out


def rel_err(got, want) -> float:
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))


def oracle_metrics_dict(st: OracleStepper) -> dict:
    m = st.metrics
    return {
        "total_time_ns": m.total_time_ns, "compute_ns": m.compute_ns, "waiting_ns": m.waiting_ns,
        "cache_miss_ns": m.cache_miss_ns, "prefetch_ns": m.prefetch_ns,
        "cold_start_ns": m.cold_start_ns, "hits": m.hits, "misses": m.misses,
        "admissions": m.admissions, "evictions": m.evictions, "stall_events": m.stall_events,
        "overfetch_events": m.overfetch_events, "prediction_cache_hits": m.prediction_cache_hits,
        "prediction_cache_misses": m.prediction_cache_misses,
        "bandwidth_estimate": m.bandwidth_estimate, "final_step": m.final_step,
        "n_selected": m.n_selected, "n_total": m.n_total,
        "step_history": [tuple(x) for x in m.step_history],
        "per_layer": [(r[0], r[1], r[2], r[3], r[4], tuple(r[5]), tuple(r[6]), r[7])
                      for r in m.per_layer],
        "samples": [(tuple(s[0]), s[1], tuple(s[2]), tuple(s[3]), s[4]) for s in m.samples],
        "events": None if m.events is None else [tuple(e) for e in m.events],
        "cache_events": None if st.cache.events is None else
        [(n, k, e[0], e[1]) for n, k, e in st.cache.events],
    }


def product_metrics_dict(m, cache_events=None) -> dict:
    """Same layout for a product SimMetrics (paper_2510_26730_b200.engine)."""
    return {
        "total_time_ns": m.total_time_ns, "compute_ns": m.compute_ns, "waiting_ns": m.waiting_ns,
        "cache_miss_ns": m.cache_miss_ns, "prefetch_ns": m.prefetch_ns,
        "cold_start_ns": m.cold_start_ns, "hits": m.hits, "misses": m.misses,
        "admissions": m.admissions, "evictions": m.evictions, "stall_events": m.stall_events,
        "overfetch_events": m.overfetch_events, "prediction_cache_hits": m.prediction_cache_hits,
        "prediction_cache_misses": m.prediction_cache_misses,
        "bandwidth_estimate": m.bandwidth_estimate, "final_step": m.final_step,
        "n_selected": m.miss_stats.n_selected, "n_total": m.miss_stats.n_total,
        "step_history": [tuple(x) for x in m.step_history],
        "per_layer": [(r.layer, r.start_ns, r.end_ns, r.stall_ns, r.step, tuple(r.predicted),
                       tuple(r.actual), r.demand_misses) for r in m.per_layer],
        "samples": [(tuple(s.token_ids), s.layer_idx, tuple(s.predicted_experts),
                     tuple(s.actual_experts), s.step_size) for s in m.samples],
        "events": None if m.events is None else
        [(e.time_ns, e.kind, e.seq, e.detail) for e in m.events],
        "cache_events": None if cache_events is None else
        [(n, k, e.layer, e.expert) for n, k, e in cache_events],
    }


def diff_dicts(got: dict, want: dict) -> List[str]:
    return [k for k in want if got.get(k) != want[k]]
