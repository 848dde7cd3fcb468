"""Oracle for the MoE-layer arithmetic: float64 restatement on the CPU.

TEST INFRASTRUCTURE (see oracle/__init__.py).  PARITY UNPINNED by the
reference: the reference charges a constant T_l per layer
(/root/reference/pkg/src/moesim/engine.py:263, :606) and contains no router
GEMV, softmax weights, SwiGLU experts, permute or combine.
This module fixes the canonical semantics the product implements (DESIGN.md
§3) and evaluates them in float64:

  x      = rmsnorm(h)                         (weight 1, eps 1e-6)
  logits = x . W_r^T                          (fp32 on device)
  sel    = top-k of (logits + bias * resident) keyed (value desc, index asc)
  w      = "mixtral": softmax over the k selected raw logits
           "softmax_topk": softmax over all M raw logits, gathered (no renorm)
  xe     = T(x); a = T(silu(xe.W1^T) * (xe.W3^T)); y = a.W2^T
  moe    = sum_r w[t,r] * y[t,r]   (rank order)  [+ gate_t * shared(xe)]
  h'     = h + moe

Weights come from a counter-based generator (splitmix64 finaliser) that the
CUDA kernel ``ef_fill_uniform`` reproduces bit for bit, so the oracle can
regenerate any expert without copying it off the device.
"""

from __future__ import annotations

import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
C1 = np.uint64(0xBF58476D1CE4E5B9)
C2 = np.uint64(0x94D049BB133111EB)
MAT_W1, MAT_W3, MAT_W2, MAT_ROUTER, MAT_SHARED_W1, MAT_SHARED_W3, MAT_SHARED_W2, MAT_SHARED_GATE, MAT_INPUT = range(9)


def _mix(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * C1
    z = z ^ (z >> np.uint64(27))
    z = z * C2
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, layer: int, expert: int, mat: int) -> int:
    """Key of one weight tensor; mirrored by ef_stream_key() in csrc."""
    with np.errstate(over="ignore"):
        tag = np.array([(layer << 32) | (expert << 8) | mat], dtype=np.uint64)
        s = np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)
        return int(_mix(s ^ _mix(tag + GOLDEN))[0])


def uniform_scale(var: float) -> np.float32:
    """fp32 step so that values span U[-a, a) with a^2/3 = var."""
    return np.float32(math.sqrt(3.0 * var) / 8388608.0)


def fan_scale(fan_in: int) -> np.float32:
    """Weight step for variance 1/fan_in; same double expression as engine.cu."""
    return np.float32(math.sqrt(3.0 / fan_in) / 8388608.0)


def fill_uniform(key: int, n: int, scale: np.float32, offset: int = 0) -> np.ndarray:
    """Element i = float32(int24(mix(key + (offset+i+1)*GOLDEN)) - 2^23) * scale."""
    with np.errstate(over="ignore"):
        i = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        h = _mix(np.uint64(key) + i * GOLDEN)
    u = (h >> np.uint64(40)).astype(np.int64) - 8388608
    return u.astype(np.float32) * np.float32(scale)


def to_bf16(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as float32 values."""
    b = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) << np.uint64(16)
    return r.astype(np.uint32).view(np.float32)


def cast(a: np.ndarray, dtype: str) -> np.ndarray:
    return to_bf16(a) if dtype == "bf16" else np.asarray(a, dtype=np.float32)


class ModelWeights:
    """Lazily regenerates the synthetic weights of a model shape."""

    def __init__(self, *, L, M, d, ff, dtype, seed, shared_ff=0, shared_gate=False,
                 cache: bool = False):
        self.L, self.M, self.d, self.ff, self.dtype, self.seed = L, M, d, ff, dtype, seed
        self.shared_ff, self.shared_gate = shared_ff, shared_gate
        self._cache = {} if cache else None  # regenerated matrices (large shapes, tests)

    def _mat(self, layer, expert, mat, rows, cols, fan_in):
        ck = (layer, expert, mat)
        if self._cache is not None and ck in self._cache:
            return self._cache[ck]
        key = stream_key(self.seed, layer, expert, mat)
        v = fill_uniform(key, rows * cols, fan_scale(fan_in))
        m = cast(v, self.dtype).reshape(rows, cols)
        if self._cache is not None:
            self._cache[ck] = m
        return m

    def expert(self, layer, e):
        d, ff = self.d, self.ff
        return (self._mat(layer, e, MAT_W1, ff, d, d), self._mat(layer, e, MAT_W3, ff, d, d),
                self._mat(layer, e, MAT_W2, d, ff, ff))

    def router(self, layer):
        return self._mat(layer, 0, MAT_ROUTER, self.M, self.d, self.d)

    def shared(self, layer):
        if not self.shared_ff:
            return None
        d, ff = self.d, self.shared_ff
        w1 = self._mat(layer, 0, MAT_SHARED_W1, ff, d, d)
        w3 = self._mat(layer, 0, MAT_SHARED_W3, ff, d, d)
        w2 = self._mat(layer, 0, MAT_SHARED_W2, d, ff, ff)
        g = self._mat(layer, 0, MAT_SHARED_GATE, 1, d, d)[0] if self.shared_gate else None
        return w1, w3, w2, g


def input_hidden(seed: int, step: int, B: int, d: int) -> np.ndarray:
    """Synthetic decode input h_0 for step ``step``: U with variance 1, fp32."""
    key = stream_key(seed, step, 0, MAT_INPUT)
    return fill_uniform(key, B * d, uniform_scale(1.0)).reshape(B, d)


def rmsnorm(h: np.ndarray, eps: float = 1e-6) -> np.ndarray:
    h = np.asarray(h, dtype=np.float64)
    return h / np.sqrt((h * h).mean(axis=1, keepdims=True) + eps)


def router_logits(x: np.ndarray, wr: np.ndarray) -> np.ndarray:
    return np.asarray(x, np.float64) @ np.asarray(wr, np.float64).T


def routing_mask(resident, M: int, k: int, budget_experts: int, L: int, ntok: int,
                 logits: Optional[np.ndarray] = None) -> int:
    """Experts that get the cache-aware routing bias in one layer (engine.cu
    ``residency_mask`` + kernels.cu ``topup_mask``): the layer's residents;
    when the batch could touch more than the layer's share of the cache
    (ntok*k > U, U = max(k, budget // L)) and fewer than k experts are
    resident, topped up to U experts by router votes over the layer's fp32
    ``logits`` [B, M]: the non-resident experts in the most tokens' UNBIASED
    top-k (value desc, index asc), then the largest logit over the batch,
    then the lower index — the set that changes the fewest tokens'
    selections.  Decode steps only: the engine's prefill passes ntok = 0
    (residents only).  No reference counterpart (the reference's cache-aware
    routing only reorders groups, engine.py:192-209)."""
    mask = 0
    n = 0
    for e in range(M):
        if resident[e]:
            mask |= 1 << e
            n += 1
    U = min(max(k, budget_experts // L), M)
    if ntok * k > U and n < k:
        if logits is None:
            raise ValueError("the top-up needs the layer's router logits")
        lg = np.asarray(logits, dtype=np.float32)
        votes = np.zeros(M, dtype=np.int64)
        for row in topk_select(lg, k):
            votes[row] += 1
        mx = lg.max(axis=0)
        order = sorted((e for e in range(M) if not (mask >> e) & 1),
                       key=lambda e: (-int(votes[e]), -float(mx[e]), e))
        for e in order[:max(0, U - n)]:
            mask |= 1 << e
    return mask


def mask_bits(mask: int, M: int) -> np.ndarray:
    return np.array([(mask >> e) & 1 for e in range(M)], dtype=bool)


def topk_select(logits: np.ndarray, k: int, bias: float = 0.0,
                resident: Optional[np.ndarray] = None) -> np.ndarray:
    """Rank-ordered top-k keyed on fp32 (logit + bias*resident); ties -> low
    index (selection keys on logits, same order as
    scheduler.py:56-60 applied to softmax)."""
    logits = np.asarray(logits, dtype=np.float32)
    B, M = logits.shape
    key = logits.copy()
    if resident is not None and bias != 0.0:
        key = (key + np.float32(bias) * resident.astype(np.float32)).astype(np.float32)
    out = np.empty((B, k), dtype=np.int32)
    for t in range(B):
        out[t] = sorted(range(M), key=lambda e: (-float(key[t, e]), e))[:k]
    return out


def route_weights(logits: np.ndarray, sel: np.ndarray, mode: str) -> np.ndarray:
    lg = np.asarray(logits, np.float64)
    if mode == "mixtral":
        picked = np.take_along_axis(lg, sel, axis=1)
        z = np.exp(picked - picked.max(axis=1, keepdims=True))
        return z / z.sum(axis=1, keepdims=True)
    z = np.exp(lg - lg.max(axis=1, keepdims=True))
    p = z / z.sum(axis=1, keepdims=True)
    return np.take_along_axis(p, sel, axis=1)


def permute(sel: np.ndarray, M: int):
    """Stable permutation by (expert, token, rank): counts, offsets[M+1],
    perm[B*k] (flat slot t*k+r), inv[B,k] (position of (t,r))."""
    B, k = sel.shape
    flat = sel.reshape(-1)
    counts = np.bincount(flat, minlength=M).astype(np.int32)
    offsets = np.zeros(M + 1, dtype=np.int32)
    offsets[1:] = np.cumsum(counts)
    perm = np.argsort(flat, kind="stable").astype(np.int32)
    inv = np.empty(B * k, dtype=np.int32)
    inv[perm] = np.arange(B * k, dtype=np.int32)
    return counts, offsets, perm, inv.reshape(B, k)


def swiglu(xe: np.ndarray, w1, w3, w2, dtype: str) -> np.ndarray:
    xe = np.asarray(xe, np.float64)
    g = xe @ np.asarray(w1, np.float64).T
    u = xe @ np.asarray(w3, np.float64).T
    a = cast((g / (1.0 + np.exp(-g))) * u, dtype).astype(np.float64)
    return a @ np.asarray(w2, np.float64).T


def moe_layer(h, weights: ModelWeights, layer, k, mode, bias=0.0, resident=None,
              logits_override=None, sel_override=None):
    """One layer of the canonical MoE forward; returns dict of intermediates.
    ``logits_override``/``sel_override`` replay the device's fp32 logits and
    selection (the "given identical fp32 gate logits" condition)."""
    x = rmsnorm(h)
    wr = weights.router(layer)
    logits = router_logits(x, wr)
    lg32 = np.asarray(logits if logits_override is None else logits_override, np.float32)
    sel = topk_select(lg32, k, bias, resident) if sel_override is None else \
        np.asarray(sel_override, dtype=np.int32)
    w = route_weights(lg32, sel, mode)
    xe = cast(x.astype(np.float32), weights.dtype)
    B = h.shape[0]
    moe = np.zeros((B, weights.d), dtype=np.float64)
    ys = {}
    for e in sorted(set(sel.reshape(-1).tolist())):
        rows = [t for t in range(B) if e in sel[t]]
        w1, w3, w2 = weights.expert(layer, e)
        y = swiglu(xe[rows], w1, w3, w2, weights.dtype)
        for i, t in enumerate(rows):
            ys[(t, e)] = y[i]
    for t in range(B):
        for r in range(k):
            moe[t] += w[t, r] * ys[(t, int(sel[t, r]))]
    sh = weights.shared(layer)
    if sh is not None:
        w1, w3, w2, g = sh
        ysh = swiglu(xe, w1, w3, w2, weights.dtype)
        if g is not None:
            gate = 1.0 / (1.0 + np.exp(-(x @ np.asarray(g, np.float64))))
            ysh = ysh * gate[:, None]
        moe += ysh
    return {"x": x, "logits": logits, "sel": sel, "w": w,
            "h_next": np.asarray(h, np.float64) + moe}


def softmax64(logits_row: Sequence[float]) -> List[float]:
    """Canonical fp64 softmax of fp32 logits: glibc exp (math.exp), sequential
    sum — the normalisation order SURVEY H6 pins for N_e."""
    vals = [float(v) for v in logits_row]
    m = max(vals)
    ex = [math.exp(v - m) for v in vals]
    s = 0.0
    for v in ex:
        s += v
    return [v / s for v in ex]


def biased_keys(logits: np.ndarray, bias: float = 0.0, mask: int = 0) -> np.ndarray:
    """fp32 router keys: logit + bias for experts in the residency bit mask
    (the key the route kernel selects on)."""
    key = np.asarray(logits, dtype=np.float32).copy()
    if bias != 0.0:
        cols = [e for e in range(key.shape[-1]) if (mask >> e) & 1]
        key[..., cols] = key[..., cols] + np.float32(bias)
    return key


def batch_gate(logits: np.ndarray, bias: float = 0.0, mask: int = 0) -> np.ndarray:
    """Token-weighted batch gate (workload.py:215-223 with per-token groups):
    mean of per-token softmax64 of the (biased) fp32 keys, renormalised by a
    sequential sum."""
    logits = biased_keys(logits, bias, mask)
    B, M = logits.shape
    w = 1.0 / B
    mixed = [0.0] * M
    for t in range(B):
        p = softmax64(logits[t])
        for e in range(M):
            mixed[e] += w * p[e]
    s = 0.0
    for v in mixed:
        s += v
    return np.array([v / s for v in mixed], dtype=np.float64)


class CpuPortLayerSample:
    """Timed CPU port of the decode layer (the bench's cpu_baseline and
    ``--impl reference`` arm): the same canonical semantics as moe_layer in
    float32 numpy/BLAS on all host threads, over a bounded sample of layers
    whose routed experts are generated once and then kept in host memory."""

    def __init__(self, weights: ModelWeights, layers, B: int, k: int, mode: str, seed: int = 0):
        self.w, self.layers, self.k, self.mode = weights, list(layers), k, mode
        self.h0 = input_hidden(seed, 0, B, weights.d).astype(np.float32)
        self.router = {l: weights.router(l).astype(np.float32) for l in self.layers}
        self.experts = {}
        self.shared = {l: weights.shared(l) for l in self.layers}
        h = self.h0
        for l in self.layers:  # first pass: find and materialise the routed experts
            x = rmsnorm(h).astype(np.float32)
            sel = topk_select(x @ self.router[l].T, k)
            for e in sorted(set(sel.reshape(-1).tolist())):
                self.experts[(l, e)] = tuple(np.ascontiguousarray(m, np.float32)
                                             for m in weights.expert(l, e))
            h = self._layer(h, l)

    def _swiglu(self, xe, w1, w3, w2):
        g = xe @ w1.T
        u = xe @ w3.T
        a = cast((g / (np.float32(1) + np.exp(-g))) * u, self.w.dtype)
        return a @ w2.T

    def _layer(self, h, l):
        x = (h / np.sqrt((h * h).mean(axis=1, keepdims=True) + np.float32(1e-6))).astype(np.float32)
        lg = x @ self.router[l].T
        sel = topk_select(lg, self.k)
        wts = route_weights(lg, sel, self.mode).astype(np.float32)
        xe = cast(x, self.w.dtype)
        out = h.copy()
        for t in range(h.shape[0]):
            for r in range(self.k):
                w1, w3, w2 = self.experts.get((l, int(sel[t, r]))) or tuple(
                    np.asarray(m, np.float32) for m in self.w.expert(l, int(sel[t, r])))
                out[t] += wts[t, r] * self._swiglu(xe[t:t + 1], w1, w3, w2)[0]
        sh = self.shared[l]
        if sh is not None:
            w1, w3, w2, g = sh
            ys = self._swiglu(xe, np.asarray(w1, np.float32), np.asarray(w3, np.float32),
                              np.asarray(w2, np.float32))
            if g is not None:
                ys = ys * (1.0 / (1.0 + np.exp(-(x @ np.asarray(g, np.float32)))))[:, None]
            out += ys
        return out

    def run(self):
        h = self.h0
        for l in self.layers:
            h = self._layer(h, l)
        return h
