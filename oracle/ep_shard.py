"""Expert-parallel shard oracle — TEST INFRASTRUCTURE (see oracle/__init__.py).

Under expert parallelism rank r of G owns experts
[r*M/G, (r+1)*M/G) of every layer and runs the reference scheduler over
them alone.  The reference has no multi-GPU code; its
per-layer loop (/root/reference/pkg/src/moesim/engine.py:566-659) and
ExpertCache (memory.py:28-156) are applied per shard to the shard's view of
the routing:

  gate    the batch gate of all G*B tokens (numerics.batch_gate, bias 0:
          token-weighted mean of per-token fp64 softmax, workload.py:215-223)
          restricted to the owned experts and renormalised by a sequential sum;
  groups  one routing group per global token, holding its owned experts as
          local ids (ascending; empty when it routes elsewhere);
  actual  the ascending union.

The shard's ModelSpec has M/G experts per layer and top_k min(k, M/G).
"""

from __future__ import annotations

from typing import List, Sequence

import numpy as np

from . import numerics as N
from .sim import OracleStepper, Policy, TokenTrace


def shard_gate(logits: np.ndarray, M: int, G: int, rank: int) -> np.ndarray:
    ms, e0 = M // G, rank * (M // G)
    full = N.batch_gate(np.asarray(logits, np.float32))
    s = 0.0
    for j in range(ms):
        s += float(full[e0 + j])
    return np.array([float(full[e0 + j]) / s for j in range(ms)], dtype=np.float64)


def shard_view(logits, sel, M: int, G: int, rank: int):
    ms, e0 = M // G, rank * (M // G)
    groups = tuple(tuple(sorted(int(e) - e0 for e in row if e0 <= int(e) < e0 + ms))
                   for row in np.asarray(sel))
    actual = tuple(sorted(set().union(*groups))) if groups else ()
    return shard_gate(logits, M, G, rank), groups, actual


def shard_traces(log, L: int, tokens_per_step: Sequence[Sequence[int]], M: int, G: int,
                 rank: int) -> List[TokenTrace]:
    """Per decode step, the shard's TokenTrace from the global routing log
    [(logits [R][G*B][M], sel [G*B][k], mask)] of an expert-parallel engine."""
    out = []
    for t, toks in enumerate(tokens_per_step):
        gates, actual, grouped = [], [], []
        for l in range(L):
            logits, sel, _ = log[t * L + l]
            g, grp, a = shard_view(logits[0], sel, M, G, rank)
            gates.append(g)
            grouped.append(grp)
            actual.append(a)
        out.append(TokenTrace(tuple(toks), gates, actual, grouped,
                              tuple([1] * log[t * L][1].shape[0])))
    return out


def replay_shard(log, *, L, M, k, G, rank, expert_bytes, link_bw, budget_experts, layer_ns,
                 policy: Policy, tokens_per_step, emit_events=True) -> OracleStepper:
    ms = M // G
    traces = shard_traces(log, L, tokens_per_step, M, G, rank)
    cur = {"t": 0}

    def pregate_fn(tt, layer, h):
        return shard_gate(log[cur["t"] * L + layer][0][h], M, G, rank)

    st = OracleStepper(num_layers=L, experts_per_layer=ms, top_k=min(k, ms),
                       expert_size_bytes=expert_bytes, link_bw=link_bw,
                       device_memory_bytes=budget_experts * expert_bytes, layer_compute_ns=layer_ns,
                       policy=policy, emit_events=emit_events, pregate_fn=pregate_fn)
    for t, tt in enumerate(traces):
        cur["t"] = t
        st.run_token(tt)
    return st
