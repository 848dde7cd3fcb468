"""CPU decode port: the whole MoE decode step on the host cores.

TEST AND BASELINE INFRASTRUCTURE (see oracle/__init__.py).  bench.py times it
as the CPU implementation of the path (its ``cpu_baseline`` leg and the
``--impl reference`` arm); tests check it against the float64 oracle.

One ``step(h)`` is a full L-layer decode step of the same workload the GPU
engine runs:

  * the reference's scheduler decisions — ``OracleStepper``, the restatement of
    ``_Sim`` (/root/reference/pkg/src/moesim/engine.py:543-690) pinned to the
    reference's golden vectors — driven layer by layer by this port's own
    routing, with the cache-aware routing bias mask of the engine
    (numerics.routing_mask) taken from the stepper's cache at each layer start
    and the pre-gate predictor fed from the future layers' router rows
    (kernel (b) semantics: x_l . W_r^(l+h));
  * the layer arithmetic of oracle/numerics.py in fp32: router
    GEMV, top-k keyed on fp32 logits (value desc, index asc), routing
    weights, SwiGLU experts on bf16 weights widened on the fly (oracle/cport.c,
    OpenMP over the host cores), rank-order combine, shared experts.

Expert weights are generated on first touch into host RAM in the slab's blob
layout (bf16, [W1 | W3 | W2]) by the counter generator the device uses; the
generation time is reported separately and excluded from ``compute_s``.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import time
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import numerics as N
from .sim import OracleStepper, Policy, TokenTrace

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libcport.so")


def build(force: bool = False) -> str:
    """gcc -O3 -fopenmp oracle/cport.c -> oracle/_build/libcport.so."""
    import subprocess
    src = os.path.join(HERE, "cport.c")
    if not force and os.path.exists(LIB_PATH) and \
            os.path.getmtime(LIB_PATH) >= os.path.getmtime(src):
        return LIB_PATH
    os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
    subprocess.run(["gcc", "-O3", "-fopenmp", "-shared", "-fPIC", src, "-o", LIB_PATH, "-lm"],
                   check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int, C.c_int64
        _lib.cp_fill_bf16.argtypes = [vp, i64, C.c_uint64, C.c_float, i64]
        _lib.cp_gemv.argtypes = [vp, i32, i32, i32, vp, i32, vp]
        _lib.cp_swiglu.argtypes = [vp, i32, i32, i32, vp, i32, vp, vp]
        _lib.cp_num_threads.restype = i32
    return _lib


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def fill(key: int, n: int, scale, dtype: str) -> np.ndarray:
    """One weight tensor: bf16 bits (uint16) or fp32 values."""
    if dtype == "bf16":
        out = np.empty(n, dtype=np.uint16)
        lib().cp_fill_bf16(_p(out), n, key, float(scale), 0)
        return out
    return N.fill_uniform(key, n, scale)


def gemv(w: np.ndarray, rows: int, cols: int, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.empty((x.shape[0], rows), dtype=np.float32)
    lib().cp_gemv(_p(w), 1 if w.dtype == np.uint16 else 0, rows, cols, _p(x), x.shape[0], _p(y))
    return y


def swiglu(blob: np.ndarray, d: int, ff: int, xe: np.ndarray) -> np.ndarray:
    xe = np.ascontiguousarray(xe, dtype=np.float32)
    n = xe.shape[0]
    act = np.empty((n, ff), dtype=np.float32)
    y = np.empty((n, d), dtype=np.float32)
    lib().cp_swiglu(_p(blob), 1 if blob.dtype == np.uint16 else 0, d, ff, _p(xe), n, _p(act),
                    _p(y))
    return y


class CpuDecodePort:
    """The engine's decode step (MoEEngine.step) on the host cores."""

    def __init__(self, *, L, M, k, d, ff, dtype, route_mode, shared_ff=0, shared_gate=False,
                 seed=0, budget_experts, policy: Policy, link_bw, layer_ns, bias=0.0):
        self.L, self.M, self.k, self.d, self.ff = L, M, k, d, ff
        self.dtype, self.mode, self.seed, self.bias = dtype, route_mode, seed, float(bias)
        self.shared_ff, self.shared_gate = shared_ff, shared_gate
        self.budget = budget_experts
        self.gen_s = 0.0
        t0 = time.perf_counter()
        self.router = [fill(N.stream_key(seed, l, 0, N.MAT_ROUTER), M * d, N.fan_scale(d), dtype)
                       for l in range(L)]
        self.shared = []
        for l in range(L):
            if not shared_ff:
                self.shared.append(None)
                continue
            blob = np.concatenate([
                fill(N.stream_key(seed, l, 0, N.MAT_SHARED_W1), shared_ff * d, N.fan_scale(d), dtype),
                fill(N.stream_key(seed, l, 0, N.MAT_SHARED_W3), shared_ff * d, N.fan_scale(d), dtype),
                fill(N.stream_key(seed, l, 0, N.MAT_SHARED_W2), shared_ff * d,
                     N.fan_scale(shared_ff), dtype)])
            g = None
            if shared_gate:
                g = fill(N.stream_key(seed, l, 0, N.MAT_SHARED_GATE), d, N.fan_scale(d), dtype)
            self.shared.append((blob, g))
        self.gen_s += time.perf_counter() - t0
        self.experts: Dict[Tuple[int, int], np.ndarray] = {}
        self.st = OracleStepper(num_layers=L, experts_per_layer=M, top_k=k,
                                expert_size_bytes=3 * d * ff * (2 if dtype == "bf16" else 4),
                                link_bw=int(link_bw),
                                device_memory_bytes=budget_experts * 3 * d * ff *
                                (2 if dtype == "bf16" else 4),
                                layer_compute_ns=int(layer_ns), policy=policy,
                                pregate_fn=self._pregate)
        self.steps = 0
        self.compute_s = 0.0   # layer arithmetic (router, pre-gate rows, experts, combine)
        self.sched_s = 0.0     # the reference scheduler's per-layer decisions
        self.layers_run = 0
        self.expert_bytes = 0  # routed expert weight bytes streamed

    # ------------------------------------------------------------ weights
    def expert(self, l: int, e: int) -> np.ndarray:
        w = self.experts.get((l, e))
        if w is None:
            t0 = time.perf_counter()
            d, ff, s = self.d, self.ff, self.seed
            w = np.concatenate([
                fill(N.stream_key(s, l, e, N.MAT_W1), ff * d, N.fan_scale(d), self.dtype),
                fill(N.stream_key(s, l, e, N.MAT_W3), ff * d, N.fan_scale(d), self.dtype),
                fill(N.stream_key(s, l, e, N.MAT_W2), ff * d, N.fan_scale(ff), self.dtype)])
            self.experts[(l, e)] = w
            self.gen_s += time.perf_counter() - t0
        return w

    def _x_in_dtype(self, x):
        return N.cast(x, self.dtype)

    # ------------------------------------------------------------ routing
    def _mask(self, layer, logits):
        if not self.bias:
            return 0
        res = [(layer, e) in self.st.cache for e in range(self.M)]
        return N.routing_mask(res, self.M, self.k, self.budget, self.L, logits.shape[0], logits)

    def _pregate(self, tt, layer, h):
        t0 = time.perf_counter()
        key = (layer, h)
        lg = self._pg.get(key)
        if lg is None:
            lg = gemv(self.router[layer + h], self.M, self.d, self._x[layer])
            self._pg[key] = lg
        self._pg_s += time.perf_counter() - t0
        return N.batch_gate(lg, self.bias, self._mask(layer + h, lg))

    # ------------------------------------------------------------ one step
    def step(self, h: np.ndarray, token_ids: Optional[Sequence[int]] = None) -> np.ndarray:
        """h[B, d] fp32 -> the MoE stack applied to it (returns a new array)."""
        B = h.shape[0]
        L, M, k = self.L, self.M, self.k
        tt = TokenTrace(tuple(token_ids) if token_ids else (-(self.steps + 1),),
                        [None] * L, [None] * L, [None] * L, tuple([1] * B))
        state = {"h": np.array(h, dtype=np.float32)}
        self._x, self._pg, self._pg_s = {}, {}, 0.0
        self.last_sel = {}
        hook_s = [0.0]
        gen0 = self.gen_s

        def hook(layer, resident):
            t0 = time.perf_counter()
            hh = state["h"]
            x = (hh / np.sqrt((hh * hh).mean(axis=1, keepdims=True) + np.float32(1e-6))).astype(
                np.float32)
            self._x[layer] = x
            lg = gemv(self.router[layer], M, self.d, x)
            self._pg[(layer, 0)] = lg
            mask = self._mask(layer, lg)
            sel = N.topk_select(lg, k, self.bias, N.mask_bits(mask, M) if self.bias else None)
            w = N.route_weights(lg, sel, self.mode).astype(np.float32)
            xe = self._x_in_dtype(x)
            out = hh.copy()
            ys = {}
            for e in sorted(set(sel.reshape(-1).tolist())):
                rows = [t for t in range(B) if e in sel[t]]
                y = swiglu(self.expert(layer, e), self.d, self.ff, xe[rows])
                self.expert_bytes += self.experts[(layer, e)].nbytes
                for i, t in enumerate(rows):
                    ys[(t, e)] = y[i]
            for t in range(B):
                for r in range(k):
                    out[t] += w[t, r] * ys[(t, int(sel[t, r]))]
            sh = self.shared[layer]
            if sh is not None:
                blob, g = sh
                y = swiglu(blob, self.d, self.shared_ff, xe)
                if g is not None:
                    gl = gemv(g, 1, self.d, x)[:, 0]
                    y = y * (1.0 / (1.0 + np.exp(-gl)))[:, None].astype(np.float32)
                out += y
            state["h"] = out
            self.last_sel[layer] = (lg, sel)
            g_sel = tuple(tuple(sorted(int(e) for e in row)) for row in sel)
            tt.gates[layer] = N.batch_gate(lg, self.bias, mask)
            tt.group_actual[layer] = g_sel
            tt.actual[layer] = tuple(sorted(set().union(*g_sel)))
            hook_s[0] += time.perf_counter() - t0

        self.st.pre_layer_hook = hook
        t0 = time.perf_counter()
        self.st.run_token(tt)
        total = time.perf_counter() - t0
        gen = self.gen_s - gen0
        compute = hook_s[0] + self._pg_s - gen
        self.compute_s += compute
        self.sched_s += total - hook_s[0] - self._pg_s
        self.layers_run += L
        self.steps += 1
        return state["h"]

    @property
    def threads(self) -> int:
        return int(lib().cp_num_threads())
