"""Expert cache, transfer queue and link estimator — thin Python faces over
the C++ runtime in libexpertflow.so (same API as the reference
/root/reference/pkg/src/moesim/memory.py:28-236)."""

from __future__ import annotations

import csv
import ctypes as C
import io
from dataclasses import dataclass
from enum import IntEnum
from typing import Iterable, List, Optional, Set, Tuple

import numpy as np

from . import _lib as L
from .core import ExpertId

TIER_HIGH = "high"
TIER_LOW = "low"
_TIER_CODE = {TIER_HIGH: 1, TIER_LOW: 0}
_TIER_NAME = {1: TIER_HIGH, 0: TIER_LOW}
_EV_NAME = {0: "miss", 1: "hit", 2: "admit", 3: "evict"}


class ExpertCache:
    """Two-tier LRU over fixed-size expert blobs (memory.py:28-156).  State
    lives in the C++ ExpertCache (O(1) per op)."""

    def __init__(self, capacity_bytes: int, expert_size_bytes: int, record_events: bool = False):
        h = L.vp()
        L.check(L.lib.ef_cache_create(int(capacity_bytes), int(expert_size_bytes),
                                      int(bool(record_events)), C.byref(h)))
        self._h = L.Handle(h.value, L.lib.ef_cache_destroy)
        self.expert_size_bytes = expert_size_bytes
        self._record = bool(record_events)

    def _counters(self):
        out = (C.c_int64 * 6)()
        L.check(L.lib.ef_cache_counters(self._h.ptr, out))
        return list(out)

    @property
    def capacity_experts(self) -> int:
        return self._counters()[0]

    @property
    def hits(self) -> int:
        return self._counters()[2]

    @property
    def misses(self) -> int:
        return self._counters()[3]

    @property
    def admissions(self) -> int:
        return self._counters()[4]

    @property
    def evictions(self) -> int:
        return self._counters()[5]

    def __len__(self) -> int:
        return self._counters()[1]

    def __contains__(self, expert: ExpertId) -> bool:
        return self.tier_of(expert) is not None

    @property
    def resident(self) -> Set[ExpertId]:
        n = C.c_int()
        cap = max(1, len(self))
        buf = np.empty(2 * cap, dtype=np.int32)
        L.check(L.lib.ef_cache_resident(self._h.ptr, L.as_ptr(buf, C.c_int32), cap, C.byref(n)))
        return {ExpertId(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(n.value)}

    def _query(self, e: ExpertId):
        tier, last = C.c_int(), C.c_int64()
        L.check(L.lib.ef_cache_query(self._h.ptr, e.layer, e.expert, C.byref(tier), C.byref(last)))
        return tier.value, last.value

    def tier_of(self, expert: ExpertId) -> Optional[str]:
        t, _ = self._query(expert)
        return None if t < 0 else _TIER_NAME[t]

    def last_access(self, expert: ExpertId) -> Optional[int]:
        t, last = self._query(expert)
        return None if t < 0 else last

    def access(self, expert: ExpertId, now: int) -> bool:
        hit = C.c_int()
        L.check(L.lib.ef_cache_access(self._h.ptr, expert.layer, expert.expert, int(now),
                                      C.byref(hit)))
        return bool(hit.value)

    def admit(self, expert: ExpertId, tier: str, now: int) -> List[ExpertId]:
        if tier not in _TIER_CODE:
            raise ValueError(f"unknown tier {tier!r}")
        cap = 64
        buf = np.empty(2 * cap, dtype=np.int32)
        n = C.c_int()
        L.check(L.lib.ef_cache_admit(self._h.ptr, expert.layer, expert.expert, _TIER_CODE[tier],
                                     int(now), L.as_ptr(buf, C.c_int32), cap, C.byref(n)))
        if n.value > cap:
            raise RuntimeError("more victims than the binding buffer")
        return [ExpertId(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(n.value)]

    def reassign_tiers(self, predicted_next: Set[ExpertId], recent_window: int, now: int) -> None:
        pairs = np.array([[e.layer, e.expert] for e in predicted_next] or [[0, 0]], dtype=np.int32)
        L.check(L.lib.ef_cache_reassign_tiers(self._h.ptr, L.as_ptr(pairs, C.c_int32),
                                              len(predicted_next), int(recent_window), int(now)))

    @property
    def events(self) -> Optional[List[Tuple[int, str, ExpertId]]]:
        n = C.c_int64()
        L.check(L.lib.ef_cache_events(self._h.ptr, None, 0, C.byref(n)))
        if n.value < 0:
            return None
        rows = np.empty(max(1, 4 * n.value), dtype=np.int64)
        L.check(L.lib.ef_cache_events(self._h.ptr, L.as_ptr(rows, C.c_int64), n.value, C.byref(n)))
        return [(int(rows[4 * i]), _EV_NAME[int(rows[4 * i + 1])],
                 ExpertId(int(rows[4 * i + 2]), int(rows[4 * i + 3]))) for i in range(n.value)]


def cache_events_csv(events: Iterable[Tuple[int, str, ExpertId]]) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(["logical_time", "event", "layer", "expert"])
    w.writerows([now, kind, e.layer, e.expert] for now, kind, e in events)
    return buf.getvalue()


class Priority(IntEnum):
    MISS = 0
    PREFETCH = 1
    EVICT = 2


@dataclass(frozen=True)
class TransferRequest:
    expert: ExpertId
    priority: Priority
    seq: int


class TransferQueue:
    """MISS < PREFETCH < EVICT, FIFO within a class (memory.py:183-202)."""

    def __init__(self) -> None:
        h = L.vp()
        L.check(L.lib.ef_tqueue_create(C.byref(h)))
        self._h = L.Handle(h.value, L.lib.ef_tqueue_destroy)

    def __len__(self) -> int:
        n = C.c_int64()
        L.check(L.lib.ef_tqueue_len(self._h.ptr, C.byref(n)))
        return n.value

    def enqueue(self, expert: ExpertId, priority: Priority) -> TransferRequest:
        seq = C.c_int64()
        L.check(L.lib.ef_tqueue_enqueue(self._h.ptr, expert.layer, expert.expert, int(priority),
                                        C.byref(seq)))
        return TransferRequest(expert, Priority(int(priority)), seq.value)

    def next_transfer(self) -> Optional[TransferRequest]:
        la, ex, pr, seq, found = C.c_int32(), C.c_int32(), C.c_int(), C.c_int64(), C.c_int()
        L.check(L.lib.ef_tqueue_next(self._h.ptr, C.byref(la), C.byref(ex), C.byref(pr),
                                     C.byref(seq), C.byref(found)))
        if not found.value:
            return None
        return TransferRequest(ExpertId(la.value, ex.value), Priority(pr.value), seq.value)


class BandwidthEstimator:
    """EWMA link-rate estimate (memory.py:205-236)."""

    def __init__(self, initial: Optional[float] = None, alpha: float = 0.25):
        h = L.vp()
        L.check(L.lib.ef_bw_create(int(initial is not None),
                                   float(initial) if initial is not None else 0.0, float(alpha),
                                   C.byref(h)))
        self._h = L.Handle(h.value, L.lib.ef_bw_destroy)
        self.alpha = alpha

    @property
    def estimate(self) -> float:
        out = C.c_double()
        L.check(L.lib.ef_bw_estimate(self._h.ptr, C.byref(out)))
        return out.value

    def observe(self, transferred_bytes: int, elapsed_ns: int) -> float:
        out = C.c_double()
        L.check(L.lib.ef_bw_observe(self._h.ptr, int(transferred_bytes), int(elapsed_ns),
                                    C.byref(out)))
        return out.value
