"""Expert parallelism: expert ownership, token dispatch/combine.

Expert e of every layer lives on rank ``e * G // M`` (contiguous blocks; for
Mixtral-8x22B at G=8 one expert per rank per layer).  Per layer each rank
routes its own tokens, sends every (token, rank-r) row to the expert's owner
(all-to-all), the owner runs the expert FFN on what it received, and the
results come back the same way (all-to-all) to be combined in rank order —
the same deterministic order as the single-GPU combine kernel.

Each rank keeps an independent ExpertCache over the experts it owns (E2), so
the reference scheduler shards naturally: rank r's decisions equal the oracle
fed with r's owned-expert access subsequence.

The exchange runs on ``torch.distributed`` all_to_all_single: NCCL over
NVLink on GPUs, gloo on CPU for the multi-process tests.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist


def owner(expert: int, M: int, G: int) -> int:
    """Rank that owns ``expert`` (contiguous blocks of M/G experts)."""
    return expert * G // M


def owned_experts(rank: int, M: int, G: int) -> List[int]:
    return [e for e in range(M) if owner(e, M, G) == rank]


def home_pool_rank(rank: int, G: int) -> int:
    """GPU whose spare HBM holds the home copies of ``rank``'s owned experts
    (the peer-HBM miss tier): the next rank, so a miss never
    reads its own device and every pool is on a different GPU."""
    return (rank + 1) % G


def peer_pool_ids(rank: int, L: int, M: int, G: int) -> List[int]:
    """Flat expert ids (l*M + e) of every layer's experts owned by ``rank``,
    in (layer, expert) order: the pool that ``home_pool_rank(rank, G)`` fills
    and exports, and the ``peer_pool_ids`` the owner's engine opens it with."""
    own = owned_experts(rank, M, G)
    return [l * M + e for l in range(L) for e in own]


@dataclass
class DispatchPlan:
    """Where each (token, rank) row goes, in a canonical order.

    ``order`` lists flat slots f = t*k + r grouped by destination rank, and
    by f inside a destination, so the exchange is deterministic.
    """
    order: np.ndarray          # [B*k] flat slots sorted by (dest, f)
    send_counts: List[int]     # rows to each rank
    recv_counts: List[int]     # rows from each rank
    recv_experts: np.ndarray   # [sum(recv)] global expert id of every received row


def plan_dispatch(sel: np.ndarray, M: int, G: int) -> Tuple[np.ndarray, List[int]]:
    sel = np.asarray(sel)
    flat = sel.reshape(-1)
    dest = np.array([owner(int(e), M, G) for e in flat], dtype=np.int64)
    order = np.lexsort((np.arange(flat.size), dest)).astype(np.int64)
    counts = [int((dest == r).sum()) for r in range(G)]
    return order, counts


class EPExchange:
    """all-to-all dispatch / combine of token rows for one process group."""

    def __init__(self, M: int, group=None):
        self.M = M
        self.group = group
        self.G = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def _a2a(self, t: torch.Tensor, send: List[int], recv: List[int]) -> torch.Tensor:
        out = torch.empty((sum(recv),) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_to_all_single(out, t.contiguous(), recv, send, group=self.group)
        return out

    def dispatch(self, x: torch.Tensor, sel: np.ndarray) -> Tuple[torch.Tensor, DispatchPlan]:
        """x [B, d] local tokens, sel [B, k] global expert ids ->
        (rows received for my experts [R, d], plan)."""
        B, k = np.asarray(sel).shape
        order, send = plan_dispatch(sel, self.M, self.G)
        dev = x.device
        send_t = torch.tensor(send, dtype=torch.int64, device=dev)
        recv_t = torch.empty_like(send_t)
        dist.all_to_all_single(recv_t, send_t, group=self.group)
        recv = [int(v) for v in recv_t.tolist()]
        rows = x[torch.as_tensor(order // k, device=dev)]
        experts = torch.as_tensor(np.asarray(sel).reshape(-1)[order], dtype=torch.int64,
                                  device=dev).reshape(-1, 1)
        got = self._a2a(rows, send, recv)
        got_e = self._a2a(experts, send, recv).reshape(-1).cpu().numpy()
        return got, DispatchPlan(order, send, recv, got_e)

    def combine(self, y_recv: torch.Tensor, plan: DispatchPlan, wts: torch.Tensor,
                residual: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Return every processed row to its token's rank and sum in rank
        order: out[t] = residual[t] + sum_r wts[t, r] * y[t, r]."""
        back = self._a2a(y_recv, plan.recv_counts, plan.send_counts)
        B, k = wts.shape
        y = torch.empty((B * k,) + tuple(back.shape[1:]), dtype=back.dtype, device=back.device)
        y[torch.as_tensor(plan.order, device=back.device)] = back
        y = y.reshape(B, k, -1)
        out = residual.clone() if residual is not None else torch.zeros(
            B, y.shape[-1], dtype=y.dtype, device=y.device)
        for r in range(k):  # rank order, like ef_combine
            out += wts[:, r:r + 1].to(y.dtype) * y[:, r]
        return out


def local_groups(recv_experts: np.ndarray) -> List[Tuple[int, np.ndarray]]:
    """(expert, row indices) for the rows a rank received, experts ascending,
    rows in arrival order (stable)."""
    out = []
    for e in sorted(set(int(v) for v in recv_experts)):
        out.append((e, np.nonzero(recv_experts == e)[0]))
    return out


def shard_budget(total_budget: int, M: int, G: int, L: int) -> int:
    """Per-rank expert-cache capacity for a global budget (E4): the budget
    split in proportion to the experts each rank owns (equal for G | M)."""
    return max(1, total_budget * len(owned_experts(0, M, G)) // M)
