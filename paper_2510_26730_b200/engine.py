"""Policies, metrics, ``simulate`` and comparisons over the C++ scheduler
stepper (reference /root/reference/pkg/src/moesim/engine.py:67-857).

``simulate`` keeps the reference's signature and semantics (a single
trace-driven pass on the integer-ns logical clock) but executes in
libexpertflow.so.  ``Simulator`` exposes the same stepper persistently across
tokens — the multi-token decode semantics the B200 engine (``MoEEngine``)
uses; with one token it is identical to ``simulate``.
"""

from __future__ import annotations

import csv
import ctypes as C
import io
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Set, Tuple

import numpy as np

from . import _lib as L
from .core import ExpertId, HardwareSpec, ModelSpec, Seed, seconds_to_ns, validate
from .predictor import ForestModel
from .scheduler import MissStats, _Ladder, miss_rate
from .workload import ActivationTrace, EmbeddingTable, NoiseConfig, Sample, pregate_signal

STRATEGIES = ("static", "reactive", "fixed_interval", "adaptive")
PREDICTORS = ("none", "pregate", "forest", "oracle")
COLD_START_MODES = ("counted", "preload")
EVENT_RANK = {"transfer_start": 0, "transfer_end": 1, "prefetch_issue": 2, "stall": 3,
              "overfetch": 4, "layer_start": 5, "layer_end": 6}
_EVENT_NAME = {v: k for k, v in EVENT_RANK.items()}


@dataclass(frozen=True)
class SimEvent:
    time_ns: int
    kind: str
    seq: int
    detail: str

    @property
    def sort_key(self) -> Tuple[int, int, int]:
        return (self.time_ns, EVENT_RANK[self.kind], self.seq)


@dataclass(frozen=True)
class PolicyConfig:
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
    noise: NoiseConfig = field(default_factory=NoiseConfig)
    prediction_cache_capacity: int = 4096

    def check(self, model: ModelSpec) -> None:
        if self.strategy not in STRATEGIES:
            raise ValueError(f"unknown strategy {self.strategy!r}; known: {', '.join(STRATEGIES)}")
        if self.predictor not in PREDICTORS:
            raise ValueError(f"unknown predictor {self.predictor!r}; known: {', '.join(PREDICTORS)}")
        if self.strategy == "fixed_interval" and (self.interval is None or self.interval < 1):
            raise ValueError("fixed_interval needs interval >= 1")
        if self.cold_start not in COLD_START_MODES:
            raise ValueError(f"unknown cold_start {self.cold_start!r}; known: "
                             + ", ".join(COLD_START_MODES))
        if self.strategy == "static" and self.predictor != "none":
            raise ValueError("static strategy takes no predictor")
        hi = self.resolved_max_step(model)
        if not 1 <= self.min_step <= hi:
            raise ValueError(f"bad step bounds [{self.min_step}, {hi}]")

    def resolved_max_step(self, model: ModelSpec) -> int:
        return self.max_step if self.max_step is not None else max(1, model.num_layers - 1)

    def to_c(self, model: ModelSpec, hw: HardwareSpec, seed: Seed, emit_events: bool) -> L.SimCfg:
        c = L.SimCfg()
        c.L, c.M, c.top_k = model.num_layers, model.experts_per_layer, model.top_k
        c.expert_size_bytes = model.expert_size_bytes
        c.link_bw = hw.link_bandwidth_bytes_per_sec
        c.device_memory_bytes = hw.device_memory_bytes
        c.layer_ns = seconds_to_ns(hw.layer_compute_time_sec)
        c.strategy = STRATEGIES.index(self.strategy)
        c.predictor = PREDICTORS.index(self.predictor)
        c.interval = self.interval or 0
        c.cache_aware_routing = int(self.cache_aware_routing)
        c.cold_start_preload = int(self.cold_start == "preload")
        c.cum_threshold = self.cum_threshold
        c.stall_threshold, c.overfetch_threshold = self.stall_threshold, self.overfetch_threshold
        c.min_step = self.min_step
        c.max_step = -1 if self.max_step is None else self.max_step
        c.recent_window = -1 if self.recent_window is None else self.recent_window
        c.prediction_cache_capacity = self.prediction_cache_capacity
        c.emit_events = int(emit_events)
        c.seed = seed.value
        return c


@dataclass(frozen=True)
class LayerRecord:
    layer: int
    start_ns: int
    end_ns: int
    stall_ns: int
    step: int
    predicted: Tuple[int, ...]
    actual: Tuple[int, ...]
    demand_misses: int


@dataclass
class SimMetrics:
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
    miss_stats: MissStats = field(default_factory=MissStats)
    step_history: Tuple[Tuple[int, int], ...] = ()
    per_layer: Tuple[LayerRecord, ...] = ()
    samples: Tuple[Sample, ...] = ()
    events: Optional[Tuple[SimEvent, ...]] = None

    @property
    def hit_rate(self) -> float:
        n = self.hits + self.misses
        return self.hits / n if n else 0.0

    @property
    def miss_rate(self) -> float:
        return miss_rate(self.miss_stats)


def route_batch(groups: Sequence[Tuple[int, Tuple[ExpertId, ...]]],
                resident: Set[ExpertId]) -> Tuple[Tuple[int, ...], Tuple[int, ...]]:
    """Stable ready-first partition of routing groups (engine.py:192-209),
    computed by the C++ runtime (ef_route_batch) over a dense index of the
    demanded experts."""
    groups = list(groups)
    if not groups:
        return (), ()
    ids = {}
    recs = []
    for gid, dem in groups:
        dem = tuple(dem)
        recs += [int(gid), len(dem)] + [ids.setdefault(e, len(ids)) for e in dem]
    mask = np.array([1 if e in resident else 0 for e in ids] or [0], dtype=np.uint8)
    rec = L.i32arr(recs)
    order = np.empty(len(groups), dtype=np.int32)
    deferred = np.empty(len(groups), dtype=np.int32)
    n, nd = C.c_int32(), C.c_int32()
    L.check(L.lib.ef_route_batch(L.as_ptr(rec, C.c_int32), rec.size, L.as_ptr(mask, C.c_uint8),
                                 max(1, len(ids)), L.as_ptr(order, C.c_int32),
                                 L.as_ptr(deferred, C.c_int32), C.byref(n), C.byref(nd)))
    return (tuple(int(g) for g in order[:n.value]), tuple(int(g) for g in deferred[:nd.value]))


# --------------------------------------------------------------- C outputs
def _read_output(fn, handle, kind) -> List[int]:
    n = C.c_int64()
    L.check(fn(handle, kind, None, 0, C.byref(n)))
    buf = np.empty(max(1, n.value), dtype=np.int64)
    L.check(fn(handle, kind, L.as_ptr(buf, C.c_int64), n.value, C.byref(n)))
    return buf[:n.value].tolist()


def collect_metrics(name: str, handle, metrics_fn, output_fn, details_fn,
                    emit_events: bool) -> SimMetrics:
    ints = (C.c_int64 * 17)()
    bw = C.c_double()
    L.check(metrics_fn(handle, ints, 17, C.byref(bw)))
    v = list(ints)
    m = SimMetrics(policy=name, total_time_ns=v[0], compute_ns=v[1], waiting_ns=v[2],
                   cache_miss_ns=v[3], prefetch_ns=v[4], cold_start_ns=v[5], hits=v[6],
                   misses=v[7], admissions=v[8], evictions=v[9], stall_events=v[10],
                   overfetch_events=v[11], prediction_cache_hits=v[12],
                   prediction_cache_misses=v[13], bandwidth_estimate=bw.value, final_step=v[14],
                   miss_stats=MissStats(v[15], v[16]))
    sh = _read_output(output_fn, handle, 0)
    m.step_history = tuple((sh[i], sh[i + 1]) for i in range(0, len(sh), 2))
    pl, recs, p = _read_output(output_fn, handle, 1), [], 0
    while p < len(pl):
        layer, s0, s1, stall, step, dm, npred = pl[p:p + 7]
        pred = tuple(pl[p + 7:p + 7 + npred])
        p += 7 + npred
        nact = pl[p]
        act = tuple(pl[p + 1:p + 1 + nact])
        p += 1 + nact
        recs.append(LayerRecord(layer, s0, s1, stall, step, pred, act, dm))
    m.per_layer = tuple(recs)
    sm, samples, p = _read_output(output_fn, handle, 2), [], 0
    while p < len(sm):
        layer, step, nt = sm[p:p + 3]
        toks = tuple(sm[p + 3:p + 3 + nt])
        p += 3 + nt
        npd = sm[p]
        pred = tuple(sm[p + 1:p + 1 + npd])
        p += 1 + npd
        na = sm[p]
        act = tuple(sm[p + 1:p + 1 + na])
        p += 1 + na
        samples.append(Sample(toks, layer, pred, act, step))
    m.samples = tuple(samples)
    if emit_events:
        ev = _read_output(output_fn, handle, 3)
        n = C.c_int64()
        L.check(details_fn(handle, None, 0, C.byref(n)))
        buf = C.create_string_buffer(max(1, n.value))
        L.check(details_fn(handle, buf, n.value, C.byref(n)))
        details = buf.raw[:n.value].decode().split("\n")[:-1]
        m.events = tuple(SimEvent(ev[3 * i], _EVENT_NAME[ev[3 * i + 1]], ev[3 * i + 2], details[i])
                         for i in range(len(details)))
    return m


def _trace_arrays(trace: ActivationTrace, M: int):
    gates = np.concatenate([L.f64arr(g.probs) for g in trace.per_layer_gate])
    if gates.size != trace.num_layers * M:
        raise ValueError("gate width differs from experts_per_layer")
    actual, groups = [], []
    for layer in range(trace.num_layers):
        a = trace.per_layer_actual[layer]
        actual += [len(a), *a]
        grp = trace.per_layer_group_actual[layer]
        groups.append(len(grp))
        for g in grp:
            groups += [len(g), *g]
    return (gates, L.i32arr(actual), L.i32arr(groups),
            L.i64arr(list(trace.group_sizes) or [0]))


class Simulator:
    """Persistent C++ stepper over trace-driven tokens (engine.py:240-690)."""

    def __init__(self, model: ModelSpec, hw: HardwareSpec, policy: PolicyConfig, seed: Seed,
                 forest: Optional[ForestModel] = None, table: Optional[EmbeddingTable] = None,
                 emit_events: bool = False, pregate=None, bandwidth_feedback: bool = False):
        """``pregate(layer, h) -> probs``: the pre-gate distribution of layer
        layer + h (default: the reference's synthetic ``pregate_signal`` of the
        current trace, engine.py:423-426; an expert-parallel shard passes its
        real router rows, ep.shard_view)."""
        rep = validate(model, hw)
        if not rep.ok:
            raise ValueError("invalid specs: " + "; ".join(rep.violations))
        policy.check(model)
        if policy.predictor == "forest" and (forest is None or table is None):
            raise ValueError("forest predictor needs a trained model and table")
        self.model, self.policy, self.seed, self.emit_events = model, policy, seed, emit_events
        self._trace: Optional[ActivationTrace] = None
        if pregate is None and policy.predictor in ("pregate", "forest"):
            def pregate(layer, h):  # engine.py:423-426
                return pregate_signal(self._trace, layer, h, policy.noise, seed).probs
        self._ladder = _Ladder(L_=model.num_layers, M=model.experts_per_layer, top_k=model.top_k,
                               cum_threshold=policy.cum_threshold,
                               forest=forest if policy.predictor == "forest" else None,
                               table=table if policy.predictor == "forest" else None,
                               pregate=pregate)
        h = L.vp()
        self._cfg = policy.to_c(model, hw, seed, emit_events)
        # bandwidth feedback into S from the logical EWMA; the
        # reference computes S once (engine.py:545-556): off = parity
        self._cfg.bw_feedback = int(bandwidth_feedback)
        L.check(L.lib.ef_sim_create(C.byref(self._cfg), C.byref(self._ladder.cfg), C.byref(h)))
        self._h = L.Handle(h.value, L.lib.ef_sim_destroy)

    def run_token(self, trace: ActivationTrace) -> None:
        if trace.num_layers != self.model.num_layers:
            raise ValueError(f"trace has {trace.num_layers} layers, model {self.model.num_layers}")
        gates, actual, groups, sizes = _trace_arrays(trace, self.model.experts_per_layer)
        toks = L.i64arr(list(trace.batch.token_ids))
        self._trace = trace
        L._pending_exc.clear()
        L.check(L.lib.ef_sim_run_token(
            self._h.ptr, L.as_ptr(toks, C.c_int64), toks.size, L.as_ptr(gates, C.c_double),
            L.as_ptr(actual, C.c_int32), actual.size, L.as_ptr(groups, C.c_int32), groups.size,
            L.as_ptr(sizes, C.c_int64), len(trace.group_sizes)))

    def metrics(self) -> SimMetrics:
        return collect_metrics(self.policy.name, self._h.ptr, L.lib.ef_sim_metrics,
                               L.lib.ef_sim_output, L.lib.ef_sim_event_details, self.emit_events)

    def cache_events(self) -> List[Tuple[int, str, ExpertId]]:
        rows = _read_output(L.lib.ef_sim_output, self._h.ptr, 4)
        names = {0: "miss", 1: "hit", 2: "admit", 3: "evict"}
        return [(rows[i], names[rows[i + 1]], ExpertId(rows[i + 2], rows[i + 3]))
                for i in range(0, len(rows), 4)]


def simulate(model: ModelSpec, hw: HardwareSpec, trace: ActivationTrace, policy: PolicyConfig,
             seed: Seed, forest: Optional[ForestModel] = None,
             table: Optional[EmbeddingTable] = None, emit_events: bool = False) -> SimMetrics:
    """One policy over one trace; deterministic (engine.py:693-716)."""
    rep = validate(model, hw)
    if not rep.ok:
        raise ValueError("invalid specs: " + "; ".join(rep.violations))
    policy.check(model)
    if trace.num_layers != model.num_layers:
        raise ValueError(f"trace has {trace.num_layers} layers, model {model.num_layers}")
    sim = Simulator(model, hw, policy, seed, forest, table, emit_events)
    sim.run_token(trace)
    return sim.metrics()


@dataclass(frozen=True)
class RunRow:
    workload: int
    policy: str
    metrics: SimMetrics

    @property
    def stall_plus_miss_ns(self) -> int:
        return self.metrics.waiting_ns + self.metrics.cache_miss_ns


@dataclass
class ComparisonResult:
    rows: List[RunRow]
    baseline: str
    reduction_pct: Dict[Tuple[int, str], Optional[float]]

    def to_csv(self) -> str:
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(["workload", "policy", "waiting_ns", "cache_miss_ns", "total_ns", "final_step",
                    "hit_rate", "miss_rate", "reduction_pct"])
        for r in self.rows:
            red = self.reduction_pct[(r.workload, r.policy)]
            m = r.metrics
            w.writerow([r.workload, r.policy, m.waiting_ns, m.cache_miss_ns, m.total_time_ns,
                        m.final_step, repr(m.hit_rate), repr(m.miss_rate),
                        "" if red is None else repr(red)])
        return buf.getvalue()


def run_comparison(model: ModelSpec, hw: HardwareSpec, traces: Sequence[ActivationTrace],
                   policies: Sequence[PolicyConfig], seed: Seed,
                   forest: Optional[ForestModel] = None, table: Optional[EmbeddingTable] = None,
                   emit_events: bool = False) -> ComparisonResult:
    """Every policy on every trace with paired seeds (engine.py:777-823)."""
    if not policies:
        raise ValueError("no policies to compare")
    names = [p.name for p in policies]
    if len(set(names)) != len(names):
        raise ValueError(f"duplicate policy names: {names}")
    rows = [RunRow(w, p.name, simulate(model, hw, tr, p, seed.split(f"workload:{w}"), forest,
                                       table, emit_events))
            for w, tr in enumerate(traces) for p in policies]
    red: Dict[Tuple[int, str], Optional[float]] = {}
    for w in range(len(traces)):
        mine = {r.policy: r for r in rows if r.workload == w}
        base = mine[policies[0].name].stall_plus_miss_ns
        for p in policies:
            red[(w, p.name)] = (100.0 * (1.0 - mine[p.name].stall_plus_miss_ns / base)
                                if base > 0 else None)
    return ComparisonResult(rows, policies[0].name, red)


def metrics_csv(rows: Sequence[Tuple[int, SimMetrics]]) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(["workload", "policy", "waiting_ns", "cache_miss_ns", "cold_start_ns", "total_ns",
                "final_step", "hit_rate", "miss_rate"])
    for wl, m in rows:
        w.writerow([wl, m.policy, m.waiting_ns, m.cache_miss_ns, m.cold_start_ns, m.total_time_ns,
                    m.final_step, repr(m.hit_rate), repr(m.miss_rate)])
    return buf.getvalue()
