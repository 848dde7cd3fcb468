"""MoEEngine — the B200 decode engine behind ``step()``.

PyTorch supplies device memory for activations and the CUDA stream; all
decisions and data movement happen in libexpertflow.so (engine.cu): the
Stepper decides hits / misses / prefetches exactly as the reference
scheduler would on a logical clock, the slab + copy stream make those
decisions physical, and the sm_100a kernels compute the MoE layers.
"""

from __future__ import annotations

import ctypes as C
import math
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib as L
from .configs import PRESETS, MoEConfig  # noqa: F401  (re-exported)
from .core import HardwareSpec, ModelSpec, Seed, seconds_to_ns
from .engine import PolicyConfig, SimMetrics, collect_metrics
from .predictor import ForestModel
from .scheduler import _Ladder
from .workload import EmbeddingTable

DTYPES = {"f32": 0, "bf16": 1}
ROUTE_MODES = {"mixtral": 0, "softmax_topk": 1}


class MoEEngine:
    """One decode engine on one GPU.

    ``budget_experts``: HBM expert-cache capacity in experts (the logical
    cache of the reference, ``ExpertCache`` slots).  ``link_bw`` (bytes/s)
    and ``layer_time_s`` parameterise the scheduler's logical clock exactly
    like ``HardwareSpec`` does in the reference; the bench measures them.
    """

    def __init__(self, cfg: MoEConfig, *, budget_experts: int, policy: PolicyConfig,
                 link_bw: int, layer_time_s: float, max_batch: int = 1, seed: int = 0,
                 routing_bias: float = 0.0, staging_slots: Optional[int] = None,
                 forest: Optional[ForestModel] = None, table: Optional[EmbeddingTable] = None,
                 emit_events: bool = False, timing: bool = False, record_routing: bool = False,
                 device: int = 0, max_prefill: int = 0, host_store_shm: Optional[str] = None,
                 host_store_attach: bool = False, peer_device: Optional[int] = None,
                 peer_pool_experts: int = 0, peer_ipc_handle: Optional[bytes] = None,
                 peer_pool_ids: Optional[Sequence[int]] = None, ep_rank: int = 0,
                 ep_world: int = 0, ep_nccl_id: Optional[bytes] = None,
                 ep_collective=None, bandwidth_feedback: bool = False,
                 peer_pool_export: bool = False, peer_ipc_layout_hash: Optional[int] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("MoEEngine needs a CUDA device (no CPU fallback)")
        self.cfg, self.policy = cfg, policy
        self.max_batch = max_batch
        self.max_prefill = max_prefill
        self.emit_events = emit_events
        self.device = torch.device("cuda", device)
        # expert parallelism: this engine is rank ep_rank of
        # ep_world and schedules only its owned experts (ep.shard_model);
        # budget_experts is the shard's budget (ep.shard_budget)
        self.ep_world, self.ep_rank = int(ep_world), int(ep_rank)
        if self.ep_world:
            from .ep import shard_model
            model = shard_model(cfg.model_spec(), self.ep_world)
        else:
            model = cfg.model_spec()
        self.sched_model = model
        hw = HardwareSpec(int(link_bw), int(budget_experts) * cfg.expert_bytes, float(layer_time_s))
        policy.check(model)
        if policy.predictor == "oracle":
            raise ValueError("the oracle predictor needs future routing; use simulate()")
        if policy.predictor == "forest" and (forest is None or table is None):
            raise ValueError("forest predictor needs a trained model and table")
        self.hw = hw
        self._ladder = _Ladder(L_=cfg.num_layers, M=model.experts_per_layer, top_k=model.top_k,
                               cum_threshold=policy.cum_threshold,
                               forest=forest if policy.predictor == "forest" else None,
                               table=table if policy.predictor == "forest" else None)
        sim = policy.to_c(model, hw, Seed(seed), emit_events)
        # physical bandwidth feedback into S; off = parity mode
        self.bandwidth_feedback = bool(bandwidth_feedback)
        sim.bw_feedback = int(self.bandwidth_feedback)
        ec = L.EngineCfg()
        ec.L, ec.M, ec.top_k = cfg.num_layers, cfg.num_experts, cfg.top_k
        ec.d, ec.ff, ec.dtype = cfg.d_model, cfg.d_ff, DTYPES[cfg.dtype]
        ec.route_mode = ROUTE_MODES[cfg.route_mode]
        ec.max_batch = max_batch
        ec.shared_ff, ec.shared_gate = cfg.shared_ff, int(cfg.shared_gate)
        ec.budget_slots = budget_experts
        # landing slot for the one in-flight transfer + slots pinned by the
        # current layer after an in-layer eviction
        ec.staging_slots = staging_slots or (
            2 + min(max(max_batch, max_prefill) * cfg.top_k * max(1, self.ep_world),
                    model.experts_per_layer))
        ec.routing_bias = routing_bias
        ec.seed = seed
        ec.device = device
        ec.timing = int(timing)
        ec.record_routing = int(record_routing)
        ec.max_prefill = int(max_prefill)
        # one pinned host store per node for replica ranks: the first process
        # creates and fills it, the others attach (bench.py --gpus N)
        self._shm_name = host_store_shm.encode() if host_store_shm else None
        ec.host_store_shm = self._shm_name
        ec.host_store_attach = int(host_store_attach)
        # peer-HBM miss tier (E3): home copies of experts [0, peer_pool_experts)
        # on peer_device (default: this device, the one-GPU stand-in)
        if peer_pool_experts < 0:
            raise ValueError("peer_pool_experts must be >= 0")
        ec.peer_device = device if peer_device is None else int(peer_device)
        ec.peer_pool_experts = int(peer_pool_experts)
        self._peer_ids = None
        if peer_pool_ids is not None:
            ids = [int(i) for i in peer_pool_ids]
            if len(ids) != peer_pool_experts:
                raise ValueError("peer_pool_ids must list peer_pool_experts flat expert ids")
            self._peer_ids = (C.c_int32 * max(len(ids), 1))(*ids)
            ec.peer_pool_ids = self._peer_ids
        # a pool another process (one process per GPU) created on peer_device:
        # its 64-byte handle from that engine's peer_pool_handle()
        self._peer_ipc = None
        ec.peer_pool_export = int(bool(peer_pool_export))
        if peer_ipc_handle is not None:
            if len(peer_ipc_handle) != 64:
                raise ValueError("peer_ipc_handle must be the 64-byte handle of peer_pool_handle()")
            if peer_ipc_layout_hash is None:
                raise ValueError("opening a peer pool needs the exporter's peer_ipc_layout_hash")
            ec.peer_ipc_layout_hash = int(peer_ipc_layout_hash)
            self._peer_ipc = C.create_string_buffer(bytes(peer_ipc_handle), 64)
            ec.peer_ipc_handle = C.cast(self._peer_ipc, L.vp)
        ec.ep_world, ec.ep_rank = self.ep_world, self.ep_rank
        self._ep_id = None
        if ep_nccl_id is not None:
            if len(ep_nccl_id) != 128:
                raise ValueError("ep_nccl_id must be the 128-byte id of ep.nccl_unique_id()")
            self._ep_id = C.create_string_buffer(bytes(ep_nccl_id), 128)
            ec.ep_nccl_id = C.cast(self._ep_id, L.vp)
        self._ep_cb = None
        if ep_collective is not None:
            # ep_collective(op, send_ptr, recv_ptr, nbytes, stream_ptr): a host
            # transport (ep.TorchCollective); exceptions surface from step()
            def _cb(user, op, send, recv, nbytes, stream):
                try:
                    ep_collective(int(op), send or 0, recv or 0, int(nbytes), stream or 0)
                    return 0
                except BaseException as exc:  # noqa: BLE001 - re-raised after the C call
                    L._pending_exc.append(exc)
                    return -1
            self._ep_cb = L.COLLECTIVE_CB(_cb)
            ec.ep_collective = self._ep_cb
        torch.cuda.set_device(device)
        torch.cuda.init()
        h = L.vp()
        L._pending_exc.clear()
        L.check(L.lib.ef_engine_create(C.byref(ec), C.byref(sim), C.byref(self._ladder.cfg),
                                       C.byref(h)))
        self._h = L.Handle(h.value, L.lib.ef_engine_destroy)
        self._ec = ec
        self._seed = seed
        self._sim = sim

    def reset(self, policy: PolicyConfig, routing_bias: float = 0.0) -> None:
        """Start over with a fresh scheduler (``policy``) and routing bias on
        the same slab, weights and pinned host store: the cache is emptied as
        in a new engine, the routing log cleared; ``stats()`` counters keep
        accumulating.  The prediction ladder's threshold and forest stay."""
        model = self.sched_model
        policy.check(model)
        if policy.predictor == "oracle":
            raise ValueError("the oracle predictor needs future routing; use simulate()")
        if policy.cum_threshold != self.policy.cum_threshold or \
                (policy.predictor == "forest") != (self.policy.predictor == "forest"):
            raise ValueError("reset keeps the engine's prediction ladder: same cum_threshold "
                             "and forest use required")
        sim = policy.to_c(model, self.hw, Seed(self._seed), self.emit_events)
        sim.bw_feedback = int(self.bandwidth_feedback)
        L._pending_exc.clear()
        L.check(L.lib.ef_engine_reset(self._h.ptr, C.byref(sim), float(routing_bias)))
        self._sim = sim
        self.policy = policy

    # ------------------------------------------------------------------ API
    def step(self, h: torch.Tensor, token_ids: Optional[Sequence[int]] = None) -> torch.Tensor:
        """One decode step: h[B, d] (fp32, on this device) <- MoE stack(h),
        in place on the current stream; returns h."""
        if h.device != self.device or h.dtype != torch.float32 or not h.is_contiguous():
            raise ValueError("h must be a contiguous fp32 tensor on the engine's device")
        B, d = h.shape
        if d != self.cfg.d_model:
            raise ValueError(f"hidden width {d} != d_model {self.cfg.d_model}")
        toks = L.i64arr(list(token_ids) if token_ids else [0])
        stream = torch.cuda.current_stream(self.device).cuda_stream
        L._pending_exc.clear()
        L.check(L.lib.ef_engine_step(self._h.ptr, C.c_void_p(stream), C.c_void_p(h.data_ptr()),
                                     B, L.as_ptr(toks, C.c_int64),
                                     len(token_ids) if token_ids else 0))
        return h

    def prefill(self, h: torch.Tensor, token_ids: Optional[Sequence[int]] = None) -> torch.Tensor:
        """Prefill T <= max_prefill tokens: h[T, d] (fp32, on this device) <- MoE
        stack(h), in place.  One scheduler step with one routing group per
        token; the expert FFNs run on the tcgen05/TMA grouped GEMM (bf16
        engines only).  Later step() calls continue from the same cache."""
        if h.device != self.device or h.dtype != torch.float32 or not h.is_contiguous():
            raise ValueError("h must be a contiguous fp32 tensor on the engine's device")
        T, d = h.shape
        if d != self.cfg.d_model:
            raise ValueError(f"hidden width {d} != d_model {self.cfg.d_model}")
        toks = L.i64arr(list(token_ids) if token_ids else [0])
        stream = torch.cuda.current_stream(self.device).cuda_stream
        L._pending_exc.clear()
        L.check(L.lib.ef_engine_prefill(self._h.ptr, C.c_void_p(stream), C.c_void_p(h.data_ptr()),
                                        T, L.as_ptr(toks, C.c_int64),
                                        len(token_ids) if token_ids else 0))
        return h

    def step_host(self, h_in: torch.Tensor, h_out: Optional[torch.Tensor] = None,
                  token_ids: Optional[Sequence[int]] = None) -> torch.Tensor:
        """step() with the hidden state in pinned host memory: h_in[B, d] fp32
        (pinned CPU tensor) is read and h_out (default: h_in) written by the
        GPU over PCIe, ordered on the current stream — synchronise the stream
        before reading h_out.  Unlike a cudaMemcpy of the input, this never
        queues behind an expert swap-in on the copy engine."""
        h_out = h_in if h_out is None else h_out
        for t in (h_in, h_out):
            if t.device.type != "cpu" or not t.is_pinned() or t.dtype != torch.float32 \
                    or not t.is_contiguous():
                raise ValueError("h_in / h_out must be contiguous pinned fp32 CPU tensors")
        B, d = h_in.shape
        if d != self.cfg.d_model or tuple(h_out.shape) != (B, d):
            raise ValueError(f"hidden width {d} != d_model {self.cfg.d_model}")
        toks = L.i64arr(list(token_ids) if token_ids else [0])
        stream = torch.cuda.current_stream(self.device).cuda_stream
        L._pending_exc.clear()
        L.check(L.lib.ef_engine_step_host(self._h.ptr, C.c_void_p(stream),
                                          C.c_void_p(h_in.data_ptr()),
                                          C.c_void_p(h_out.data_ptr()), B,
                                          L.as_ptr(toks, C.c_int64),
                                          len(token_ids) if token_ids else 0))
        return h_out

    def activation_log(self) -> List[str]:
        """The engine's prediction samples as activation-log lines in the
        reference's wire format (workload.py:1-16, ``format_log_line``): one
        line per (token batch, layer) the predictor scored, with the token ids
        passed to step()/prefill(), the predicted and the actual expert sets
        and the horizon in effect — the input of the reference's offline forest
        training (``moesim train``), whose JSON model ``model_from_json`` loads
        back into ``MoEEngine(..., forest=...)``."""
        from .workload import format_log_line
        return [format_log_line(s) for s in self.metrics().samples]

    def metrics(self) -> SimMetrics:
        return collect_metrics(self.policy.name, self._h.ptr, L.lib.ef_engine_metrics,
                               L.lib.ef_engine_output, L.lib.ef_engine_event_details,
                               self.emit_events)

    def cache_events(self):
        from .engine import _read_output
        from .core import ExpertId
        rows = _read_output(L.lib.ef_engine_output, self._h.ptr, 4)
        names = {0: "miss", 1: "hit", 2: "admit", 3: "evict"}
        return [(rows[i], names[rows[i + 1]], ExpertId(rows[i + 2], rows[i + 3]))
                for i in range(0, len(rows), 4)]

    def peer_pool_handle(self):
        """(64-byte CUDA IPC handle, layout hash) of this engine's peer pool,
        for the engines of other processes (``peer_ipc_handle=``,
        ``peer_ipc_layout_hash=``) to serve misses from it."""
        buf = C.create_string_buffer(64)
        h = C.c_uint64()
        L.check(L.lib.ef_engine_peer_pool_handle(self._h.ptr, buf, C.byref(h)))
        return buf.raw, h.value

    def stats(self) -> dict:
        keys = ["steps", "copies", "copy_bytes", "stall_ms", "phys_slots", "logical_capacity",
                "staging_slots", "kernel_launches", "host_decision_ms", "ffn_ms", "step_ms",
                "preload_copies", "d2h_bytes", "ffn_bytes", "ffn_launches", "gate_wait_ms",
                "fast_layers", "peer_copies", "peer_bytes", "prefetch_admitted", "prefetch_used",
                "prefetch_wasted", "bw_physical_Bps", "bw_physical_transfers", "layer_kernel_steps"]
        out = (C.c_double * len(keys))()
        L.check(L.lib.ef_engine_stats(self._h.ptr, out, len(keys)))
        return dict(zip(keys, list(out)))

    def routing_log(self):
        """[(logits[R,B,M] fp32, sel[B,k] int32, resident_mask int)] per executed layer."""
        n = C.c_int64()
        R, B, lo, hi = C.c_int32(), C.c_int32(), C.c_uint64(), C.c_uint64()
        L.check(L.lib.ef_engine_routing_log(self._h.ptr, -1, None, 0, None, 0, C.byref(R),
                                            C.byref(B), C.byref(lo), C.byref(hi), C.byref(n)))
        out = []
        M, k = self.cfg.num_experts, self.cfg.top_k
        for i in range(n.value):
            L.check(L.lib.ef_engine_routing_log(self._h.ptr, i, None, 0, None, 0, C.byref(R),
                                                C.byref(B), C.byref(lo), C.byref(hi),
                                                C.byref(n)))
            lg = np.empty(max(1, R.value * B.value * M), dtype=np.float32)
            sel = np.empty(max(1, B.value * k), dtype=np.int32)
            L.check(L.lib.ef_engine_routing_log(self._h.ptr, i, L.as_ptr(lg, C.c_float), lg.size,
                                                L.as_ptr(sel, C.c_int32), sel.size, C.byref(R),
                                                C.byref(B), C.byref(lo), C.byref(hi),
                                                C.byref(n)))
            r, b = R.value, B.value
            out.append((lg[:r * b * M].reshape(r, b, M).copy(), sel[:b * k].reshape(b, k).copy(),
                        lo.value | (hi.value << 64)))
        return out

    def set_record_routing(self, mode) -> None:
        """Routing-log recording: False/0 off, True/1 logits + selection +
        router input x (routing_x), 2 logits + selection only."""
        L.check(L.lib.ef_engine_set_record(self._h.ptr, int(mode)))

    def routing_x(self):
        """[(x[B, d] fp32, mask_tokens)] per executed layer, aligned with
        routing_log(): the router input the GPU computed for that layer and the
        token count the bias mask's top-up rule used (0 for prefill)."""
        n = C.c_int64()
        R, B, lo, hi = C.c_int32(), C.c_int32(), C.c_uint64(), C.c_uint64()
        L.check(L.lib.ef_engine_routing_log(self._h.ptr, -1, None, 0, None, 0, C.byref(R),
                                            C.byref(B), C.byref(lo), C.byref(hi), C.byref(n)))
        out = []
        d = self.cfg.d_model
        for i in range(n.value):
            nx, mt = C.c_int64(), C.c_int32()
            L.check(L.lib.ef_engine_routing_x(self._h.ptr, i, None, 0, C.byref(nx), C.byref(mt)))
            x = np.empty(max(1, nx.value), dtype=np.float32)
            L.check(L.lib.ef_engine_routing_x(self._h.ptr, i, L.as_ptr(x, C.c_float), x.size,
                                              C.byref(nx), C.byref(mt)))
            out.append((x[:nx.value].reshape(-1, d).copy(), mt.value))
        return out

    def device_ptr(self, which: int) -> int:
        p = L.vp()
        L.check(L.lib.ef_engine_ptr(self._h.ptr, which, C.byref(p)))
        return p.value or 0

    def slab_view(self, slot: int) -> torch.Tensor:
        """uint8 view of one physical slab slot (for checks; no copy)."""
        base = self.device_ptr(0) + slot * self.cfg.expert_bytes
        return _raw_device_view(base, self.cfg.expert_bytes, self.device)

    def slot_of(self, layer: int, expert: int) -> int:
        s = C.c_int32()
        L.check(L.lib.ef_engine_slot_of(self._h.ptr, layer, expert, C.byref(s)))
        return s.value

    def close(self) -> None:
        self._h = None


class _RawDevice:
    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


def _raw_device_view(ptr: int, nbytes: int, device) -> torch.Tensor:
    return torch.as_tensor(_RawDevice(ptr, nbytes), device=device)


def synthetic_hidden(cfg: MoEConfig, seed: int, step: int, B: int, device) -> torch.Tensor:
    """Deterministic decode input h_0 (oracle/numerics.py input_hidden)."""
    h = torch.empty(B, cfg.d_model, dtype=torch.float32, device=device)
    key = L.lib.ef_stream_key(seed, step, 0, 8)
    scale = np.float32(math.sqrt(3.0) / 8388608.0)
    stream = torch.cuda.current_stream(device).cuda_stream
    L.check(L.lib.ef_fill_uniform(C.c_void_p(stream), C.c_void_p(h.data_ptr()), 0, h.numel(),
                                  key, float(scale), 0))
    return h


def compare_engines(cfg: MoEConfig, policies: Sequence[PolicyConfig],
                    workloads: Sequence[Sequence[torch.Tensor]], *,
                    token_ids: Optional[Sequence[Sequence[Sequence[int]]]] = None,
                    **engine_kw) -> "ComparisonResult":
    """``moesim compare`` for real decode (engine.py:777-823 report schema):
    every policy runs a fresh MoEEngine over the same hidden-state sequence of
    every workload; rows carry the engines' SimMetrics and the reduction of
    waiting + miss time against the first policy, so ``to_csv()`` prints the
    reference's comparison table.  Also returns the device time per run in
    ``device_ms[(workload, policy)]``."""
    from .engine import ComparisonResult, RunRow
    if not policies:
        raise ValueError("no policies to compare")
    names = [p.name for p in policies]
    if len(set(names)) != len(names):
        raise ValueError(f"duplicate policy names: {names}")
    rows, device_ms = [], {}
    for w, steps in enumerate(workloads):
        for p in policies:
            eng = MoEEngine(cfg, policy=p, max_batch=max(int(h.shape[0]) for h in steps),
                            **engine_kw)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for t, h in enumerate(steps):
                eng.step(h.clone(), token_ids[w][t] if token_ids else None)
            e.record()
            torch.cuda.synchronize()
            device_ms[(w, p.name)] = s.elapsed_time(e)
            rows.append(RunRow(w, p.name, eng.metrics()))
            eng.close()
    red = {}
    for w in range(len(workloads)):
        mine = {r.policy: r for r in rows if r.workload == w}
        base = mine[policies[0].name].stall_plus_miss_ns
        for p in policies:
            red[(w, p.name)] = (100.0 * (1.0 - mine[p.name].stall_plus_miss_ns / base)
                                if base > 0 else None)
    out = ComparisonResult(rows, policies[0].name, red)
    out.device_ms = device_ms
    return out
