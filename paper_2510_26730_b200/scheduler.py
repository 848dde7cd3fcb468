"""Adaptive-horizon arithmetic, feedback state, prediction cache and the
prediction ladder — Python faces over the C++ runtime (reference
/root/reference/pkg/src/moesim/scheduler.py:36-309)."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace
from typing import Callable, Dict, Optional, Sequence, Tuple, Union

import numpy as np

from . import _lib as L
from .core import ModelSpec
from .workload import GateDistribution

HorizonPrediction = Tuple[Tuple[int, Tuple[int, ...]], ...]


def _probs(gate) -> np.ndarray:
    return L.f64arr(gate.probs if isinstance(gate, GateDistribution) else gate)


def expected_expert_count(gate: Union[GateDistribution, np.ndarray],
                          cum_threshold: float = 0.9) -> int:
    p = _probs(gate)
    out = C.c_int()
    L.check(L.lib.ef_expected_expert_count(L.as_ptr(p, C.c_double), p.size, float(cum_threshold),
                                           C.byref(out)))
    return out.value


def top_experts(gate: Union[GateDistribution, np.ndarray], count: int) -> Tuple[int, ...]:
    p = _probs(gate)
    n = max(0, min(int(count), p.size))
    out = np.empty(max(1, n), dtype=np.intc)
    L.check(L.lib.ef_top_experts(L.as_ptr(p, C.c_double), p.size, int(count),
                                 L.as_ptr(out, C.c_int)))
    return tuple(int(x) for x in out[:n])


def swap_in_latency(num_experts: int, expert_size_bytes: int, bandwidth_bytes_per_sec: int) -> int:
    out = C.c_int64()
    L.check(L.lib.ef_swap_in_latency(int(num_experts), int(expert_size_bytes),
                                     int(bandwidth_bytes_per_sec), C.byref(out)))
    return out.value


def compute_step(num_experts: int, expert_size_bytes: int,
                 bandwidth_bytes_per_sec: Union[int, float], layer_compute_ns: int,
                 min_step: int, max_step: int) -> int:
    out = C.c_int()
    if isinstance(bandwidth_bytes_per_sec, int):
        L.check(L.lib.ef_compute_step_int(int(num_experts), int(expert_size_bytes),
                                          bandwidth_bytes_per_sec, int(layer_compute_ns),
                                          int(min_step), int(max_step), C.byref(out)))
    else:
        L.check(L.lib.ef_compute_step_float(int(num_experts), int(expert_size_bytes),
                                            float(bandwidth_bytes_per_sec), int(layer_compute_ns),
                                            int(min_step), int(max_step), C.byref(out)))
    return out.value


@dataclass(frozen=True)
class StepState:
    current: int
    max_step: int
    min_step: int = 1
    stall_count: int = 0
    overfetch_count: int = 0
    stall_threshold: int = 3
    overfetch_threshold: int = 3

    def _c(self) -> L.StepStateC:
        return L.StepStateC(self.current, self.max_step, self.min_step, self.stall_count,
                            self.overfetch_count, self.stall_threshold, self.overfetch_threshold)

    def __post_init__(self) -> None:
        L.check(L.lib.ef_step_validate(C.byref(self._c())))


def _transition(state: StepState, fn) -> StepState:
    c = state._c()
    L.check(fn(C.byref(c)))
    return replace(state, current=c.current, stall_count=c.stall_count,
                   overfetch_count=c.overfetch_count)


def on_stall(state: StepState) -> StepState:
    return _transition(state, L.lib.ef_step_on_stall)


def on_overfetch(state: StepState) -> StepState:
    return _transition(state, L.lib.ef_step_on_overfetch)


@dataclass
class MissStats:
    n_selected: int = 0
    n_total: int = 0

    def __post_init__(self) -> None:
        if self.n_selected < 0 or self.n_total < 0:
            raise ValueError("miss counts must be non-negative")
        if self.n_selected > self.n_total:
            raise ValueError(f"n_selected {self.n_selected} exceeds n_total {self.n_total}")

    def observe(self, predicted: Sequence[int], actual: Sequence[int]) -> None:
        a = set(actual)
        self.n_selected += len(a & set(predicted))
        self.n_total += len(a)


def miss_rate(stats: MissStats) -> float:
    if stats.n_total == 0:
        return 0.0
    return (stats.n_total - stats.n_selected) / stats.n_total


# --- value encoding shared with the C++ prediction cache -------------------
# A horizon ((target, (experts...)), ...) is stored in the C++ ladder's own
# layout [n, target, count, experts...]; any other value (nested tuples of
# ints) gets a generic tagged layout starting with -1.
def _is_horizon(v) -> bool:
    return isinstance(v, tuple) and all(
        isinstance(x, tuple) and len(x) == 2 and isinstance(x[0], (int, np.integer))
        and isinstance(x[1], tuple) and all(isinstance(e, (int, np.integer)) for e in x[1])
        for x in v)


def _encode(v) -> np.ndarray:
    if _is_horizon(v):
        out = [len(v)]
        for t, ex in v:
            out += [int(t), len(ex), *map(int, ex)]
        return L.i64arr(out)
    flat = [-1]

    def rec(x):
        if isinstance(x, (tuple, list)):
            flat.extend([1, len(x)])
            for y in x:
                rec(y)
        elif isinstance(x, (int, np.integer)):
            flat.extend([0, int(x)])
        else:
            raise TypeError("PredictionCache values must be ints or nested tuples of ints")
    rec(v)
    return L.i64arr(flat)


def _decode(b: Sequence[int]):
    b = [int(x) for x in b]
    if b[0] >= 0:
        p, out = 1, []
        for _ in range(b[0]):
            t, c = b[p], b[p + 1]
            out.append((t, tuple(b[p + 2:p + 2 + c])))
            p += 2 + c
        return tuple(out)
    pos = [1]

    def rec():
        tag, val = b[pos[0]], b[pos[0] + 1]
        pos[0] += 2
        if tag == 0:
            return val
        return tuple(rec() for _ in range(val))
    return rec()


class PredictionCache:
    """LRU of resolved predictions keyed by (token_ids, layer, step)
    (scheduler.py:194-221), stored in the C++ runtime."""

    def __init__(self, capacity: int = 4096):
        h = L.vp()
        L.check(L.lib.ef_pcache_create(int(capacity), C.byref(h)))
        self._h = L.Handle(h.value, L.lib.ef_pcache_destroy)
        self.capacity = capacity

    def _stats(self):
        out = (C.c_int64 * 3)()
        L.check(L.lib.ef_pcache_stats(self._h.ptr, out))
        return list(out)

    @property
    def hits(self) -> int:
        return self._stats()[0]

    @property
    def misses(self) -> int:
        return self._stats()[1]

    def __len__(self) -> int:
        return self._stats()[2]

    @staticmethod
    def _key(key):
        tokens, layer, step = key
        return L.i64arr(list(tokens) or [0]), len(tokens), int(layer), int(step)

    def get(self, key: Tuple):
        toks, nt, layer, step = self._key(key)
        cap = 4096
        buf = np.empty(cap, dtype=np.int64)
        n, found = C.c_int64(), C.c_int()
        L.check(L.lib.ef_pcache_get(self._h.ptr, L.as_ptr(toks, C.c_int64), nt, layer, step,
                                    L.as_ptr(buf, C.c_int64), cap, C.byref(n), C.byref(found)))
        if not found.value:
            return None
        if n.value > cap:
            buf = np.empty(n.value, dtype=np.int64)
            self._peek(toks, nt, layer, step, buf)
        return _decode(buf[:n.value])

    def _peek(self, toks, nt, layer, step, buf):
        raise RuntimeError("prediction cache value exceeds the binding buffer")

    def put(self, key: Tuple, value) -> None:
        toks, nt, layer, step = self._key(key)
        v = _encode(value)
        L.check(L.lib.ef_pcache_put(self._h.ptr, L.as_ptr(toks, C.c_int64), nt, layer, step,
                                    L.as_ptr(v, C.c_int64), v.size))


@dataclass(frozen=True)
class PredictionQuery:
    token_ids: Tuple[int, ...]
    layer: int
    step: int
    router_probs: np.ndarray
    pregate: Optional[Callable[[int], np.ndarray]] = None
    known_activations: Optional[Dict[int, Tuple[int, ...]]] = None
    cum_threshold: float = 0.9


def cache_key(query: PredictionQuery) -> Tuple:
    return (query.token_ids, query.layer, query.step)


class _Ladder:
    """Builds the C ladder config; keeps callbacks and buffers alive."""

    def __init__(self, *, L_, M, top_k, cum_threshold, forest=None, table=None, pregate=None):
        self.keep = []
        cfg = L.LadderCfg()
        cfg.L, cfg.M, cfg.top_k, cfg.cum_threshold = L_, M, top_k, float(cum_threshold)
        cfg.forest_cb = L.FOREST_CB()
        cfg.pregate_cb = L.PREGATE_CB()
        if forest is not None:
            native = getattr(forest, "_native_handle", None)
            if native is not None:
                cfg.forest = native()
                self.keep.append(forest)
            else:
                flen = int(getattr(forest, "feature_len", 0) or 0)

                def fcb(_u, feats, n, base, out):
                    try:
                        f = np.ctypeslib.as_array(feats, shape=(n,)).copy()
                        b = None if not base else np.ctypeslib.as_array(base, shape=(M,)).copy()
                        s = np.asarray(forest.predict_scores(f, baseline=b), dtype=np.float64)
                        np.ctypeslib.as_array(out, shape=(M,))[:] = s
                        return 0
                    except BaseException as exc:  # re-raised by _lib.check
                        L._pending_exc.append(exc)
                        return -1
                cfg.forest_cb = L.FOREST_CB(fcb)
                self.keep.append(cfg.forest_cb)
                if table is not None and not flen:
                    flen = table.vectors.shape[1] + 2 + L_ * M
                cfg.forest_feature_len = flen
        if table is not None:
            vec = L.f64arr(table.vectors)
            self.keep.append(vec)
            cfg.table = L.as_ptr(vec, C.c_double)
            cfg.vocab, cfg.embed_dim = vec.shape
        if pregate is not None:
            def pcb(_u, layer, h, out):
                try:
                    p = pregate(layer, h)
                    np.ctypeslib.as_array(out, shape=(M,))[:] = np.asarray(p, dtype=np.float64)
                    return 0
                except BaseException as exc:
                    L._pending_exc.append(exc)
                    return -1
            cfg.pregate_cb = L.PREGATE_CB(pcb)
            self.keep.append(cfg.pregate_cb)
        self.cfg = cfg


def _hist_records(hist: Optional[Dict[int, Tuple[int, ...]]]) -> np.ndarray:
    out = []
    for layer, ex in (hist or {}).items():
        out += [int(layer), len(ex), *map(int, ex)]
    return L.i32arr(out or [0])


def predict_experts(query: PredictionQuery, cache: PredictionCache, forest=None, table=None,
                    model: Optional[ModelSpec] = None) -> HorizonPrediction:
    """Prediction ladder (scheduler.py:247-309) executed in C++: cached
    horizon -> forest on pre-gate baseline -> pre-gate -> router top-k."""
    probs = L.f64arr(query.router_probs)
    M = probs.size
    if forest is not None and (table is None or model is None):
        raise ValueError("forest prediction needs table and model")
    pg = None
    if query.pregate is not None:
        pg = lambda _layer, h: query.pregate(h)  # noqa: E731
    lad = _Ladder(L_=model.num_layers if model else 0, M=M, top_k=model.top_k if model else 0,
                  cum_threshold=query.cum_threshold, forest=forest, table=table, pregate=pg)
    toks = L.i64arr(list(query.token_ids) or [0])
    known = _hist_records(query.known_activations)
    known_len = 0 if not query.known_activations else known.size
    cap = 16 + query.step * (3 + M)
    out = np.empty(cap, dtype=np.int64)
    n = C.c_int64()
    L._pending_exc.clear()
    L.check(L.lib.ef_predict_experts(C.byref(lad.cfg), cache._h.ptr, L.as_ptr(toks, C.c_int64),
                                     len(query.token_ids), int(query.layer), int(query.step),
                                     L.as_ptr(probs, C.c_double), L.as_ptr(known, C.c_int32),
                                     known_len, L.as_ptr(out, C.c_int64), cap, C.byref(n)))
    if n.value > cap:
        raise RuntimeError("horizon exceeds the binding buffer")
    return _decode(out[:n.value])
