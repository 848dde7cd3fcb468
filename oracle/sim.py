"""Oracle restatement of the reference's layer-step loop, made steppable.

TEST INFRASTRUCTURE (see oracle/__init__.py).

``OracleStepper`` restates ``_Sim`` (/root/reference/pkg/src/moesim/engine.py
:240-690) on a logical integer-ns clock.  ``run_token`` executes the per-layer
body of engine.py:566-659 for one token's trace; the cache, link, transfer
queue, step state and counters persist across calls (multi-token decode, new
behaviour documented in DESIGN.md §4).  With a single ``run_token`` call the
result equals ``moesim.simulate`` field for field — that is what
tests/test_oracle_golden.py pins against fixtures made by the real reference.

Multi-token conventions (T > 1):
  * the cache's logical time is the global layer count ``t * L + l``;
  * only the very first layer of the run uses the "cold" bucket;
  * preload and the initial compute_step happen once, on token 0;
  * predictions, horizons and the adaptive boundary restart per token
    (a horizon never crosses a token boundary, engine.py:454 clips it).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import decisions as D

EVENT_RANK = {  # engine.py:72-80
    "transfer_start": 0, "transfer_end": 1, "prefetch_issue": 2, "stall": 3,
    "overfetch": 4, "layer_start": 5, "layer_end": 6,
}
PRIO_NAME = {D.PRIO_MISS: "miss", D.PRIO_PREFETCH: "prefetch", D.PRIO_EVICT: "evict"}


@dataclass
class Policy:
    """engine.py:95-142 (PolicyConfig)."""
    name: str
    strategy: str
    predictor: str = "none"
    interval: Optional[int] = None
    cache_aware_routing: bool = False
    cold_start: str = "counted"
    cum_threshold: float = 0.9
    stall_threshold: int = 3
    overfetch_threshold: int = 3
    min_step: int = 1
    max_step: Optional[int] = None
    recent_window: Optional[int] = None
    noise_decay_rate: float = 0.6
    prediction_cache_capacity: int = 4096

    def resolved_max_step(self, num_layers: int) -> int:
        return self.max_step if self.max_step is not None else max(1, num_layers - 1)


@dataclass
class TokenTrace:
    """The router->scheduler contract of workload.py:161-179 for one token
    (one decode step of a batch)."""
    token_ids: Tuple[int, ...]
    gates: List[np.ndarray]                      # per layer fp64 [M]
    actual: List[Tuple[int, ...]]                # ascending union per layer
    group_actual: List[Tuple[Tuple[int, ...], ...]]
    group_sizes: Tuple[int, ...]


@dataclass
class Metrics:
    """engine.py:157-189 (SimMetrics), plain fields."""
    policy: str
    total_time_ns: int = 0
    compute_ns: int = 0
    waiting_ns: int = 0
    cache_miss_ns: int = 0
    prefetch_ns: int = 0
    cold_start_ns: int = 0
    hits: int = 0
    misses: int = 0
    admissions: int = 0
    evictions: int = 0
    stall_events: int = 0
    overfetch_events: int = 0
    prediction_cache_hits: int = 0
    prediction_cache_misses: int = 0
    bandwidth_estimate: float = 0.0
    final_step: int = 0
    n_selected: int = 0
    n_total: int = 0
    step_history: List[Tuple[int, int]] = field(default_factory=list)
    per_layer: List[tuple] = field(default_factory=list)   # LayerRecord tuples
    samples: List[tuple] = field(default_factory=list)     # Sample tuples
    events: Optional[List[tuple]] = None                   # (time, kind, seq, detail)

    @property
    def hit_rate(self) -> float:
        n = self.hits + self.misses
        return self.hits / n if n else 0.0

    @property
    def miss_rate(self) -> float:
        if self.n_total == 0:
            return 0.0
        return (self.n_total - self.n_selected) / self.n_total


class _Horizon:
    def __init__(self, first, issue_ns):
        self.first = first
        self.issue_ns = issue_ns
        self.missing = set()
        self.last_arrival_ns = issue_ns
        self.checked = False


class OracleStepper:
    """Steppable restatement of engine.py:_Sim."""

    def __init__(self, *, num_layers, experts_per_layer, top_k, expert_size_bytes,
                 link_bw, device_memory_bytes, layer_compute_ns, policy: Policy,
                 seed_value: int = 0, emit_events=False, forest=None,
                 features_fn=None, pregate_fn: Optional[Callable] = None,
                 bandwidth_feedback: bool = False):
        self.L, self.M, self.k = num_layers, experts_per_layer, top_k
        self.E_s = expert_size_bytes
        self.bw = link_bw
        self.policy = policy
        self.seed_value = seed_value
        self.emit = emit_events
        self.forest = forest
        self.features_fn = features_fn
        # pregate_fn(token_trace, layer, h) -> fp64 probs; None -> the
        # reference's synthetic pregate_signal (engine.py:423-426).
        self.pregate_fn = pregate_fn
        self.bandwidth_feedback = bandwidth_feedback
        self.layer_ns = layer_compute_ns                       # engine.py:263
        if self.layer_ns < 1:
            raise ValueError("layer compute time rounds below 1 ns")
        self.per_expert_ns = D.swap_in_latency(1, self.E_s, link_bw)  # :266
        self.cache = D.ExpertCache(device_memory_bytes, self.E_s, record_events=emit_events)
        self.queue = D.TransferQueue()
        self.queued: Dict[tuple, tuple] = {}
        self.bucket_of: Dict[int, str] = {}
        self.inflight = None     # (expert, prio, bucket, start, end)
        self.link_free = 0
        self.estimator = D.BandwidthEstimator(initial=float(link_bw))
        self.pred_cache = D.PredictionCache(policy.prediction_cache_capacity)
        self.metrics = Metrics(policy=policy.name)
        self.events: List[tuple] = []
        self.event_seq = 0
        self.clock = 0
        self.now = 0             # global logical layer (cache time)
        self.state: Optional[D.StepState] = None
        self.miss_stats = D.MissStats()
        self.unconsumed: Dict[tuple, List[int]] = {}
        self.consumed_ns = 0
        self.tokens_run = 0
        self.miss_guard = 0
        self.miss_guard_limit = 16 * self.L * self.M + 256            # :299
        self.max_step = policy.resolved_max_step(self.L)

    # ------------------------------------------------------------ plumbing
    def _emit(self, t, kind, detail):
        if self.emit:
            self.events.append((t, kind, self.event_seq, detail))
            self.event_seq += 1

    def _request(self, e, prio, bucket):                         # :311-326
        if e in self.cache:
            return
        if self.inflight is not None and self.inflight[0] == e:
            return
        prev = self.queued.get(e)
        if prev is not None and prio >= prev[0]:
            return
        req = self.queue.enqueue(e, prio)
        self.queued[e] = req
        self.bucket_of[req[1]] = bucket
        self._pump(self.clock)

    def _pump(self, t):                                           # :328-354
        while self.inflight is None:
            req = self.queue.next_transfer()
            if req is None:
                return
            prio, seq, e = req
            if self.queued.get(e) is not req:
                self.bucket_of.pop(seq, None)
                continue
            del self.queued[e]
            if e in self.cache:
                self.bucket_of.pop(seq, None)
                continue
            start = max(t, self.link_free)
            self.inflight = (e, prio, self.bucket_of.pop(seq), start, start + self.per_expert_ns)
            self._emit(start, "transfer_start",
                       f"expert={e[0]}:{e[1]} priority={PRIO_NAME[prio]}")

    def _advance_to(self, t):                                     # :356-381
        while self.inflight is not None and self.inflight[4] <= t:
            e, _prio, bucket, start, end = self.inflight
            self.inflight = None
            self.link_free = end
            dur = end - start
            self.estimator.observe(self.E_s, dur)
            self.cache.admit(e, D.HIGH, self.now)
            self.unconsumed.setdefault(e, []).append(dur)
            if bucket == "cold":
                self.metrics.cold_start_ns += dur
            elif bucket == "miss":
                self.metrics.cache_miss_ns += dur
            else:
                self.metrics.prefetch_ns += dur
            hz = self.horizon_by_expert.get(e)
            if hz is not None and e in hz.missing:
                hz.missing.discard(e)
                hz.last_arrival_ns = max(hz.last_arrival_ns, end)
            self._emit(end, "transfer_end", f"expert={e[0]}:{e[1]}")
            self._pump(end)

    def _bucket(self):
        return "cold" if self.now == 0 else "miss"

    def _wait_until_resident(self, required, t):                  # :383-402
        while True:
            self._advance_to(t)
            missing = sorted(e for e in required if e not in self.cache)
            if not missing:
                return t
            for e in missing:
                self._request(e, D.PRIO_MISS, self._bucket())
                self.miss_guard += 1
            if self.miss_guard > self.miss_guard_limit:
                raise RuntimeError("no forward progress: device memory too small")
            if self.inflight is None:
                self._pump(t)
            assert self.inflight is not None, "missing experts but idle link"
            t = max(t, self.inflight[4])

    def _consume(self, required):                                 # :404-408
        for e in sorted(required):
            pend = self.unconsumed.get(e)
            if pend:
                self.consumed_ns += pend.pop(0)

    # ---------------------------------------------------------- prediction
    def _predict_targets(self, tt: TokenTrace, layer, step):      # :412-449
        pol = self.policy
        if pol.predictor == "oracle":
            return [(t, tt.actual[t]) for t in range(layer + 1, layer + step + 1)]
        pregate = None
        if pol.predictor in ("pregate", "forest"):
            if self.pregate_fn is not None:
                pregate = lambda h: self.pregate_fn(tt, layer, h)  # noqa: E731
            else:
                pregate = lambda h: D.pregate_signal(  # noqa: E731
                    tt.gates[layer + h], layer, h, pol.noise_decay_rate, self.seed_value)
        forest = self.forest if pol.predictor == "forest" else None
        feats = None
        if forest is not None:
            feats = lambda s, target, hist: self.features_fn(tt.token_ids, s, target, hist)  # noqa: E731
        known = {x: tt.actual[x] for x in range(layer + 1)}
        return list(D.predict_experts(tt.token_ids, layer, step, tt.gates[layer], pregate,
                                      known, pol.cum_threshold, self.pred_cache,
                                      forest=forest, features_fn=feats, top_k=self.k))

    def _issue_horizon(self, tt, layer, step):                    # :451-482
        step = min(step, self.L - 1 - layer)
        if step < 1:
            return
        targets = self._predict_targets(tt, layer, step)
        if not targets:
            return
        hz = _Horizon(targets[0][0], self.clock)
        for target, experts in targets:
            self.predicted[target] = (tuple(experts), step)
            for x in experts:
                e = (target, x)
                if e not in self.cache:
                    if e not in self.queued and (self.inflight is None or self.inflight[0] != e):
                        self._request(e, D.PRIO_PREFETCH, "prefetch")
                    hz.missing.add(e)
                    self.horizon_by_expert[e] = hz
        self.horizons.append(hz)
        self._emit(self.clock, "prefetch_issue",
                   f"layer={layer} targets={targets[0][0]}..{targets[-1][0]} step={step}")

    def _boundary(self, tt, layer):                               # :484-499
        s = self.policy.strategy
        if s == "static":
            return
        if s == "reactive":
            self._issue_horizon(tt, layer, 1)
        elif s == "fixed_interval":
            if layer % self.policy.interval == 0:
                self._issue_horizon(tt, layer, self.policy.interval)
        elif layer == self.next_boundary:
            if self.bandwidth_feedback and self.state is not None:
                # flagged feedback (not in the reference, whose S is
                # computed once, engine.py:545-556): re-base S on the current
                # estimate at every adaptive boundary
                pol = self.policy
                n_e = D.expected_expert_count(tt.gates[layer], pol.cum_threshold)
                self.state.current = D.compute_step(n_e, self.E_s, self.estimator.estimate,
                                                    self.layer_ns, pol.min_step, self.max_step)
            step = self.state.current
            self._issue_horizon(tt, layer, step)
            self.next_boundary = layer + step

    def _check_overfetch(self, layer, first_exec):                # :501-517
        for hz in self.horizons:
            if hz.first != layer or hz.checked:
                continue
            hz.checked = True
            if hz.missing:
                continue
            margin = first_exec - hz.last_arrival_ns
            if margin > self.layer_ns:
                self.metrics.overfetch_events += 1
                self._emit(first_exec, "overfetch", f"layer={layer} margin_ns={margin}")
                if self.state is not None:
                    self.state.overfetch()

    def _step_in_effect(self):                                    # :532-541
        s = self.policy.strategy
        if s == "adaptive":
            return self.state.current
        if s == "fixed_interval":
            return self.policy.interval
        return 1 if s == "reactive" else 0

    # ----------------------------------------------------------- main loop
    def _start(self, tt: TokenTrace):                             # :543-564
        pol = self.policy
        if pol.strategy == "adaptive":
            n_e = D.expected_expert_count(tt.gates[0], pol.cum_threshold)
            s0 = D.compute_step(n_e, self.E_s, self.estimator.estimate, self.layer_ns,
                                pol.min_step, self.max_step)
            self.state = D.StepState(s0, self.max_step, pol.min_step,
                                     pol.stall_threshold, pol.overfetch_threshold)
        if pol.cold_start == "preload":                           # :521-530
            for x in tt.actual[0]:
                self.cache.admit((0, x), D.HIGH, 0)
            self.metrics.cold_start_ns = D.swap_in_latency(len(tt.actual[0]), self.E_s, self.bw)

    pre_layer_hook = None  # callable(layer, resident_set) before each layer's step

    def run_token(self, tt: TokenTrace) -> None:
        if self.pre_layer_hook is not None:
            self.pre_layer_hook(0, set(self.cache.tier))
        if self.tokens_run == 0:
            self._start(tt)
        # the reference's no-progress guard (:299) lives for one trace = one
        # token; a multi-token decode run re-arms it per token
        self.miss_guard = 0
        self.predicted: Dict[int, tuple] = {}
        self.horizons: List[_Horizon] = []
        self.horizon_by_expert: Dict[tuple, _Horizon] = {}
        self.next_boundary = 0
        pol, m = self.policy, self.metrics
        for layer in range(self.L):                               # :566-659
            if layer and self.pre_layer_hook is not None:
                self.pre_layer_hook(layer, set(self.cache.tier))
            self.now = self.tokens_run * self.L + layer
            t0 = self.clock
            self._advance_to(t0)
            self._emit(t0, "layer_start", f"layer={layer}")
            m.step_history.append((layer, self._step_in_effect()))
            actual = tuple(tt.actual[layer])
            missing = [(layer, x) for x in actual if not self.cache.access((layer, x), self.now)]
            for e in missing:
                self._request(e, D.PRIO_MISS, self._bucket())
            self._boundary(tt, layer)
            if layer in self.predicted:
                pred, step = self.predicted[layer]
                self.miss_stats.observe(pred, actual)
                m.samples.append((tuple(tt.token_ids), layer, pred, actual, step))
            groups = [(g, tuple((layer, x) for x in dem))
                      for g, dem in enumerate(tt.group_actual[layer])]
            if pol.cache_aware_routing:
                order, _ = D.route_batch(groups, set(self.cache.tier))
            else:
                order = tuple(g for g, _ in groups)
            durs = D.group_durations(self.layer_ns, tt.group_sizes)
            chain, stall = t0, 0
            for pos, g in enumerate(order):
                demand = set(groups[g][1])
                avail = self._wait_until_resident(demand, chain)
                if pos == 0:
                    self._check_overfetch(layer, avail)
                if avail > chain:
                    stall += avail - chain
                    self._emit(chain, "stall", f"layer={layer} gap_ns={avail - chain}")
                    chain = avail
                self._consume(demand)
                chain += durs[g]
                self._advance_to(chain)
            m.waiting_ns += stall
            m.compute_ns += self.layer_ns
            if stall > 0:
                m.stall_events += 1
                if self.state is not None:
                    self.state.stall()
            if pol.strategy == "adaptive":                        # :631-644
                window = pol.recent_window if pol.recent_window is not None else self.state.current
                hot = {(t, x) for t, (ex, _s) in self.predicted.items() if t > layer for x in ex}
                self.cache.reassign_tiers(hot, window, self.now)
            self._emit(chain, "layer_end", f"layer={layer}")
            m.per_layer.append((layer, t0, chain, stall, self._step_in_effect(),
                                self.predicted.get(layer, ((), 0))[0], actual, len(missing)))
            self.clock = chain
        self.tokens_run += 1
        self._finish()

    def _finish(self):                                            # :661-689
        m = self.metrics
        m.total_time_ns = self.clock
        m.hits, m.misses = self.cache.hits, self.cache.misses
        m.admissions, m.evictions = self.cache.admissions, self.cache.evictions
        m.prediction_cache_hits = self.pred_cache.hits
        m.prediction_cache_misses = self.pred_cache.misses
        m.bandwidth_estimate = self.estimator.estimate
        m.final_step = self._step_in_effect()
        m.n_selected, m.n_total = self.miss_stats.n_selected, self.miss_stats.n_total
        if self.emit:
            m.events = sorted(self.events, key=lambda ev: (ev[0], EVENT_RANK[ev[1]], ev[2]))
        assert m.total_time_ns == m.compute_ns + m.waiting_ns
        assert self.consumed_ns <= m.total_time_ns


def simulate(*, trace: TokenTrace, **kw) -> Metrics:
    """engine.py:693-716 for one trace."""
    st = OracleStepper(**kw)
    st.run_token(trace)
    return st.metrics
