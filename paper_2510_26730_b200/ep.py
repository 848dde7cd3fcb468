"""Expert parallelism: ownership, shard shapes, and the
host side of the expert-parallel decode step.

Expert e of every layer lives on rank ``e * G // M`` (contiguous blocks; for
Mixtral-8x22B at G=8 one expert per rank per layer).  ``MoEEngine(...,
ep_rank=r, ep_world=G)`` runs the step in C++/CUDA (engine.cu ``ep_step_on``):
each rank routes its own B tokens, the routing blocks (x, logits, selection,
weights) are all-gathered, every rank runs its owned experts for all G*B
tokens from its own slab under its own scheduler, and the outputs return by
an all-to-all to be combined in rank order — the single-GPU combine's order.

The collectives are NCCL on the engine's stream (one process per GPU:
``nccl_unique_id`` on rank 0, broadcast to the others), or a host transport
(``TorchCollective``: any torch.distributed group, e.g. gloo) so G ranks can
share one GPU in tests — NCCL refuses two ranks on one device.

Each rank's scheduler sees only its owned experts (local ids 0..M/G-1): the
batch gate of all G*B tokens restricted to them (``ef_ep_shard_view``), one
routing group per global token.  The reference scheduler therefore shards
naturally: rank r's decisions equal the oracle fed with r's view
(oracle/ep_shard.py).
"""

from __future__ import annotations

import ctypes as C
from typing import List, Sequence, Tuple

import numpy as np

from . import _lib as L
from .core import ModelSpec


def owner(expert: int, M: int, G: int) -> int:
    """Rank that owns ``expert`` (contiguous blocks of M/G experts)."""
    return expert * G // M


def owned_experts(rank: int, M: int, G: int) -> List[int]:
    return [e for e in range(M) if owner(e, M, G) == rank]


def shard_model(model: ModelSpec, G: int) -> ModelSpec:
    """The scheduler shape of one rank: M/G experts per layer, top_k
    min(k, M/G) (its ladder predicts over its own experts)."""
    if model.experts_per_layer % G:
        raise ValueError(f"expert parallelism needs G | M (M={model.experts_per_layer}, G={G})")
    ms = model.experts_per_layer // G
    return ModelSpec(model.num_layers, ms, min(model.top_k, ms), model.expert_size_bytes,
                     model.embed_dim, model.vocab_size)


def shard_budget(total_budget: int, M: int, G: int, L: int) -> int:
    """Per-rank expert-cache capacity for a global budget (E4): the budget
    split in proportion to the experts each rank owns (equal for G | M)."""
    return max(1, total_budget * len(owned_experts(0, M, G)) // M)


def home_pool_rank(rank: int, G: int) -> int:
    """GPU whose spare HBM holds the home copies of ``rank``'s owned experts
    (the peer-HBM miss tier): the next rank, so a miss never
    reads its own device and every pool is on a different GPU."""
    return (rank + 1) % G


def peer_pool_ids(rank: int, L: int, M: int, G: int) -> List[int]:
    """Flat expert ids (l*M + e) of every layer's experts owned by ``rank``,
    in (layer, expert) order: the home copies a single-GPU engine's peer pool
    holds for that rank's experts.  An expert-parallel engine's own pool uses
    its local ids (l * M/G + j)."""
    own = owned_experts(rank, M, G)
    return [l * M + e for l in range(L) for e in own]


def shard_view(logits: np.ndarray, sel: np.ndarray, M: int, k: int, G: int, rank: int
               ) -> Tuple[np.ndarray, Tuple[Tuple[int, ...], ...], Tuple[int, ...]]:
    """The shard's view of one layer (ef_ep_shard_view): (gate [M/G] fp64,
    per-token owned experts as local ids, ascending union)."""
    lg = np.ascontiguousarray(logits, dtype=np.float32)
    sl = np.ascontiguousarray(sel, dtype=np.int32)
    GB = lg.shape[0]
    ms = M // G
    gate = np.empty(ms, dtype=np.float64)
    groups = np.empty((GB, k), dtype=np.int32)
    actual = np.empty(ms, dtype=np.int32)
    n = C.c_int32()
    L.check(L.lib.ef_ep_shard_view(L.as_ptr(lg, C.c_float), L.as_ptr(sl, C.c_int32), GB, M, k, G,
                                   rank, L.as_ptr(gate, C.c_double), L.as_ptr(groups, C.c_int32),
                                   L.as_ptr(actual, C.c_int32), C.byref(n)))
    g = tuple(tuple(int(e) for e in row if e >= 0) for row in groups)
    return gate, g, tuple(int(e) for e in actual[:n.value])


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id of a new EP group (call on rank 0 only)."""
    buf = C.create_string_buffer(128)
    L.check(L.lib.ef_ep_nccl_unique_id(buf))
    return buf.raw


def nccl_group_id(group=None) -> bytes:
    """The NCCL id of an EP group, agreed over a torch.distributed group."""
    import torch.distributed as dist
    box = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    return box[0]


class TorchCollective:
    """Host transport of the EP collectives over a torch.distributed group
    (``MoEEngine(..., ep_collective=TorchCollective(group))``): the device
    buffers are staged through host memory and exchanged with the group's
    backend (gloo in the multi-process tests, several ranks per GPU)."""

    def __init__(self, group=None, device=0):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.world = dist.get_world_size(group)
        self.device = torch.device("cuda", device)
        self.calls = 0

    def _view(self, ptr: int, nbytes: int):
        from .runtime import _raw_device_view
        return _raw_device_view(ptr, nbytes, self.device)

    def __call__(self, op: int, send: int, recv: int, nbytes: int, stream: int) -> None:
        torch, dist = self.torch, self.dist
        torch.cuda.synchronize(self.device)  # the engine's stream has produced `send`
        G = self.world
        if op == 0:  # all-gather: recv[g] = rank g's send
            src = self._view(send, nbytes).cpu()
            out = torch.empty(G * nbytes, dtype=torch.uint8)
            dist.all_gather(list(out.view(G, nbytes).unbind(0)), src, group=self.group)
        elif op == 1:  # all-to-all: recv[g] = rank g's send[me]
            src = self._view(send, G * nbytes).cpu()
            out = torch.empty(G * nbytes, dtype=torch.uint8)
            dist.all_to_all_single(out, src, group=self.group)
        else:
            raise ValueError(f"unknown collective op {op}")
        self._view(recv, G * nbytes).copy_(out)
        torch.cuda.synchronize(self.device)
        self.calls += 1
