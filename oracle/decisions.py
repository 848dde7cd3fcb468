"""Oracle restatement of the reference's per-layer decision primitives.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Pure Python on small inputs;
every function cites the reference (paths relative to
/root/reference/pkg/src/moesim).  Objects here use plain tuples
``(layer, expert)`` for expert ids instead of the reference's ``ExpertId``
dataclass; ordering is the same (layer-major, ``core.py:94-116``).
"""

from __future__ import annotations

import hashlib
import heapq
import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

NS_PER_SEC = 1_000_000_000
CUM_EPS = 1e-9  # scheduler.py:24
HIGH, LOW = "high", "low"  # memory.py:24-25
PRIO_MISS, PRIO_PREFETCH, PRIO_EVICT = 0, 1, 2  # memory.py:169-175


# ---------------------------------------------------------------- core.py

def seconds_to_ns(seconds: float) -> int:
    """core.py:41-45 — Python round() of seconds * 1e9 (ties to even)."""
    if seconds < 0:
        raise ValueError("negative duration")
    return round(seconds * NS_PER_SEC)


def seed_split(value: int, label: str) -> int:
    """core.py:63-67 — first 8 bytes of sha256(value_be8 ':' label)."""
    h = hashlib.sha256(value.to_bytes(8, "big") + b":" + label.encode()).digest()
    return int.from_bytes(h[:8], "big")


# ---------------------------------------------------------- scheduler.py

def desc_order(values: Sequence[float]) -> List[int]:
    """Stable descending order (ties -> lower index); the contract of
    ``np.argsort(-p, kind="stable")`` at workload.py:184, scheduler.py:47,59."""
    return sorted(range(len(values)), key=lambda i: (-float(values[i]), i))


def expected_expert_count(probs: Sequence[float], thr: float = 0.9) -> int:
    """scheduler.py:36-53 — shortest descending prefix whose sequential fp64
    sum reaches thr - 1e-9; at least 1 (len(probs) if never reached)."""
    if not 0.0 < thr <= 1.0:
        raise ValueError("cum_threshold must lie in (0, 1]")
    acc = 0.0
    order = desc_order(probs)
    for n, i in enumerate(order, 1):
        acc += float(probs[i])
        if acc >= thr - CUM_EPS:
            return n
    return len(order)


def top_experts(probs: Sequence[float], count: int) -> Tuple[int, ...]:
    """scheduler.py:56-60 — the ``count`` best indices, returned ascending."""
    return tuple(sorted(desc_order(probs)[:count]))


def topk_ranked(values: Sequence[float], k: int) -> Tuple[int, ...]:
    """workload.py:182-185 — the k best indices in rank order."""
    return tuple(desc_order(values)[:k])


def swap_in_latency(n: int, size: int, bw: int) -> int:
    """scheduler.py:63-74 — ceil(n * size * 1e9 / bw) in exact integers."""
    if n < 0 or bw < 1:
        raise ValueError("bad swap_in_latency arguments")
    return -((-n * size * NS_PER_SEC) // bw)


def compute_step(n_e, size, bw, layer_ns, lo, hi) -> int:
    """scheduler.py:77-105 — S = clamp(ceil(n_e*size*1e9 / (bw*layer_ns)))."""
    if layer_ns < 1 or not 1 <= lo <= hi or n_e < 0:
        raise ValueError("bad compute_step arguments")
    numer = n_e * size * NS_PER_SEC
    if isinstance(bw, int):
        if bw < 1:
            raise ValueError("bandwidth must be >= 1 byte/s")
        raw = -((-numer) // (bw * layer_ns))
    else:
        if not bw > 0:
            raise ValueError("bandwidth must be positive")
        raw = math.ceil(numer / (bw * layer_ns))
    return max(lo, min(int(raw), hi))


class StepState:
    """scheduler.py:108-163 — step size with stall / overfetch counters."""

    def __init__(self, current, max_step, min_step=1, stall_threshold=3,
                 overfetch_threshold=3):
        if not (1 <= min_step <= max_step and min_step <= current <= max_step):
            raise ValueError("bad step state")
        if stall_threshold < 1 or overfetch_threshold < 1:
            raise ValueError("feedback thresholds must be >= 1")
        self.current, self.max_step, self.min_step = current, max_step, min_step
        self.stall_threshold = stall_threshold
        self.overfetch_threshold = overfetch_threshold
        self.stall_count = 0
        self.overfetch_count = 0

    def stall(self) -> None:  # on_stall, scheduler.py:142-151
        self.stall_count += 1
        if self.stall_count >= self.stall_threshold:
            self.stall_count = 0
            self.current = min(self.current + 1, self.max_step)

    def overfetch(self) -> None:  # on_overfetch, scheduler.py:154-163
        self.overfetch_count += 1
        if self.overfetch_count >= self.overfetch_threshold:
            self.overfetch_count = 0
            self.current = max(self.current - 1, self.min_step)


class MissStats:
    """scheduler.py:166-191."""

    def __init__(self):
        self.n_selected = 0
        self.n_total = 0

    def observe(self, predicted, actual) -> None:
        a = set(actual)
        self.n_selected += len(a & set(predicted))
        self.n_total += len(a)

    def rate(self) -> float:
        if self.n_total == 0:
            return 0.0
        return (self.n_total - self.n_selected) / self.n_total


class PredictionCache:
    """scheduler.py:194-221 — LRU map of resolved horizons."""

    def __init__(self, capacity: int = 4096):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        self.capacity = capacity
        self.hits = 0
        self.misses = 0
        self._d: Dict[tuple, tuple] = {}

    def get(self, key):
        if key not in self._d:
            self.misses += 1
            return None
        val = self._d.pop(key)
        self._d[key] = val  # re-insert = most recent
        self.hits += 1
        return val

    def put(self, key, value) -> None:
        self._d.pop(key, None)
        self._d[key] = value
        while len(self._d) > self.capacity:
            del self._d[next(iter(self._d))]


def predict_experts(token_ids, layer, step, router_probs, pregate, known,
                    cum_threshold, cache: PredictionCache, forest=None,
                    features_fn=None, top_k=None):
    """scheduler.py:247-309 — the prediction ladder for targets
    layer+1 .. layer+step.  ``pregate(h)`` returns fp64 probs or is None;
    ``forest`` is any object with ``predict_scores(features, baseline)``;
    ``features_fn(step, target, history)`` builds forest features."""
    key = (tuple(token_ids), layer, step)
    hit = cache.get(key)
    if hit is not None:
        return hit
    history = dict(known or {})
    out = []
    for h in range(1, step + 1):
        target = layer + h
        pg = pregate(h) if pregate is not None else None
        if forest is not None:
            scores = np.asarray(
                forest.predict_scores(features_fn(step, target, history), baseline=pg),
                dtype=np.float64)
            mass = np.clip(scores, 0.0, None)
            total = mass.sum()
            if total > 0:
                n = expected_expert_count(mass / total, cum_threshold)
            elif pg is not None:
                n = expected_expert_count(pg, cum_threshold)
            else:
                n = expected_expert_count(router_probs, cum_threshold)
            chosen = top_experts(scores, n)
        elif pg is not None:
            chosen = top_experts(pg, expected_expert_count(pg, cum_threshold))
        else:
            if top_k is None:
                raise ValueError("fallback prediction needs model for top_k")
            chosen = top_experts(router_probs, top_k)
        out.append((target, chosen))
        history[target] = chosen
    result = tuple(out)
    cache.put(key, result)
    return result


# -------------------------------------------------------------- memory.py

class ExpertCache:
    """memory.py:28-156 — two-tier LRU.  Each resident carries (tier, touch
    sequence number); per-tier recency order is ascending touch, which is
    exactly the OrderedDict order the reference maintains (every insertion
    into a tier order takes a fresh, larger touch number)."""

    def __init__(self, capacity_bytes: int, expert_size: int, record_events=False):
        if expert_size < 1:
            raise ValueError("expert_size_bytes must be >= 1")
        self.capacity_experts = capacity_bytes // expert_size
        if self.capacity_experts < 1:
            raise ValueError("capacity cannot hold one expert")
        self.expert_size_bytes = expert_size
        self.hits = self.misses = self.admissions = self.evictions = 0
        self.tier: Dict[tuple, str] = {}
        self.touch: Dict[tuple, int] = {}
        self.last: Dict[tuple, int] = {}
        self._seq = 0
        self.events: Optional[list] = [] if record_events else None

    def __contains__(self, e) -> bool:
        return e in self.tier

    def __len__(self) -> int:
        return len(self.tier)

    def _log(self, now, kind, e):
        if self.events is not None:
            self.events.append((now, kind, e))

    def _stamp(self, e, tier):
        self.tier[e] = tier
        self.touch[e] = self._seq
        self._seq += 1

    def access(self, e, now) -> bool:  # memory.py:94-104
        if e not in self.tier:
            self.misses += 1
            self._log(now, "miss", e)
            return False
        self._stamp(e, HIGH)
        self.last[e] = now
        self.hits += 1
        self._log(now, "hit", e)
        return True

    def _victim(self):
        for tier in (LOW, HIGH):
            members = [x for x in self.tier if self.tier[x] == tier]
            if members:
                return min(members, key=lambda x: self.touch[x])
        raise AssertionError("empty cache has no victim")

    def admit(self, e, tier, now) -> list:  # memory.py:106-129
        if tier not in (HIGH, LOW):
            raise ValueError(f"unknown tier {tier!r}")
        if e in self.tier:
            self._stamp(e, tier)
            self.last[e] = now
            return []
        victims = []
        while len(self.tier) >= self.capacity_experts:
            v = self._victim()
            del self.tier[v], self.touch[v], self.last[v]
            self.evictions += 1
            self._log(now, "evict", v)
            victims.append(v)
        self._stamp(e, tier)
        self.last[e] = now
        self.admissions += 1
        self._log(now, "admit", e)
        return victims

    def reassign_tiers(self, predicted, window, now) -> None:  # memory.py:137-156
        if window < 0:
            raise ValueError("recent_window must be >= 0")
        for e in self.tier:
            hot = e in predicted or (now - self.last[e] < window)
            self.tier[e] = HIGH if hot else LOW


class TransferQueue:
    """memory.py:183-202 — min-heap on (priority, seq)."""

    def __init__(self):
        self._heap = []
        self._seq = 0

    def __len__(self):
        return len(self._heap)

    def enqueue(self, e, prio):
        req = (prio, self._seq, e)
        self._seq += 1
        heapq.heappush(self._heap, req)
        return req

    def next_transfer(self):
        return heapq.heappop(self._heap) if self._heap else None


class BandwidthEstimator:
    """memory.py:205-236 — EWMA; the first observation replaces the prior.
    The rate is the correctly rounded quotient of the exact integers."""

    def __init__(self, initial=None, alpha=0.25):
        if not 0.0 < alpha <= 1.0:
            raise ValueError("alpha must lie in (0, 1]")
        self.alpha = alpha
        self._est = float(initial) if initial is not None else None
        self._seen = False

    @property
    def estimate(self) -> float:
        if self._est is None:
            raise RuntimeError("no estimate")
        return self._est

    def observe(self, nbytes: int, ns: int) -> float:
        if ns < 1 or nbytes < 0:
            raise ValueError("bad observation")
        rate = nbytes * NS_PER_SEC / ns
        if self._seen:
            self._est = self.alpha * rate + (1.0 - self.alpha) * self._est
        else:
            self._est, self._seen = rate, True
        return self._est


# -------------------------------------------------------------- engine.py

def route_batch(groups, resident):
    """engine.py:192-209 — stable ready-first partition of group ids."""
    ready = [g for g, dem in groups if all(e in resident for e in dem)]
    late = [g for g, dem in groups if not all(e in resident for e in dem)]
    return tuple(ready + late), tuple(late)


def group_durations(total_ns: int, sizes: Sequence[int]) -> List[int]:
    """engine.py:212-219 — floor split by token count, remainder to the front."""
    n = sum(sizes)
    d = [total_ns * s // n for s in sizes]
    for g in range(total_ns - sum(d)):
        d[g] += 1
    return d


# ------------------------------------------------------------ workload.py

def noise_weight(decay_rate: float, horizon: int) -> float:
    """workload.py:255-256."""
    return 1.0 - math.exp(-decay_rate * horizon)


def pregate_signal(true_probs, from_layer, horizon, decay_rate, seed_value):
    """workload.py:259-293 — corrupted preview of a future gate.  Uses numpy's
    PCG64 Dirichlet draw seeded by split("pregate:l:h") exactly like the
    reference (numpy is the reference's one dependency, pyproject.toml:10)."""
    true_probs = np.asarray(true_probs, dtype=np.float64)
    m = true_probs.shape[0]
    w = noise_weight(decay_rate, horizon)
    rng = np.random.default_rng(seed_split(seed_value, f"pregate:{from_layer}:{horizon}"))
    r = rng.dirichlet(np.ones(m))
    return (1.0 - w) * ((1.0 - w) * true_probs + w * r) + w * np.full(m, 1.0 / m)
