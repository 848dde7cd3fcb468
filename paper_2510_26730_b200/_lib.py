"""ctypes binding of libexpertflow.so (include/expertflow.h).

There is no Python fallback: if the library is missing or fails to load,
importing the package raises ImportError naming the build command.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libexpertflow.so")

EF_OK, EF_ERUNTIME, EF_ECUDA, EF_ENOMEM, EF_EINVAL = 0, -1, -5, -12, -22

# The engine's pipeline keeps a kernel spinning on a host flag; kernels must
# not be loaded lazily behind it (see preload_pipeline_kernels in kernels.cu).
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_2510_26730_b200/build.py` "
        "(the product path has no CPU fallback)")
lib = C.CDLL(LIB_PATH)

i32, i64, u64, f32, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double
vp = C.c_void_p
P = C.POINTER


class StepStateC(C.Structure):
    _fields_ = [(n, i32) for n in ("current", "max_step", "min_step", "stall_count",
                                   "overfetch_count", "stall_threshold", "overfetch_threshold")]


PREGATE_CB = C.CFUNCTYPE(C.c_int, vp, i32, i32, P(f64))
COLLECTIVE_CB = C.CFUNCTYPE(C.c_int, vp, C.c_int, vp, vp, i64, vp)
FOREST_CB = C.CFUNCTYPE(C.c_int, vp, P(f64), i32, P(f64), P(f64))


class LadderCfg(C.Structure):
    _fields_ = [("L", i32), ("M", i32), ("top_k", i32), ("cum_threshold", f64),
                ("forest", vp), ("forest_cb", FOREST_CB), ("forest_user", vp),
                ("forest_feature_len", i32), ("table", P(f64)), ("vocab", i64),
                ("embed_dim", i32), ("pregate_cb", PREGATE_CB), ("pregate_user", vp)]


class SimCfg(C.Structure):
    _fields_ = [("L", i32), ("M", i32), ("top_k", i32), ("expert_size_bytes", i64),
                ("link_bw", i64), ("device_memory_bytes", i64), ("layer_ns", i64),
                ("strategy", i32), ("predictor", i32), ("interval", i32),
                ("cache_aware_routing", i32), ("cold_start_preload", i32),
                ("cum_threshold", f64), ("stall_threshold", i32), ("overfetch_threshold", i32),
                ("min_step", i32), ("max_step", i32), ("recent_window", i32),
                ("prediction_cache_capacity", i32), ("emit_events", i32), ("seed", u64),
                ("bw_feedback", i32)]


class EngineCfg(C.Structure):
    _fields_ = [("L", i32), ("M", i32), ("top_k", i32), ("d", i32), ("ff", i32), ("dtype", i32),
                ("route_mode", i32), ("max_batch", i32), ("shared_ff", i32),
                ("shared_gate", i32), ("budget_slots", i64), ("staging_slots", i32),
                ("routing_bias", f32), ("seed", u64), ("device", i32), ("timing", i32),
                ("record_routing", i32), ("max_prefill", i32), ("host_store_shm", C.c_char_p),
                ("host_store_attach", i32), ("peer_device", i32), ("peer_pool_experts", i64),
                ("peer_pool_ids", P(i32)), ("peer_ipc_handle", vp),
                ("ep_world", i32), ("ep_rank", i32), ("ep_nccl_id", vp),
                ("ep_collective", COLLECTIVE_CB), ("ep_user", vp),
                ("peer_pool_export", i32), ("peer_ipc_layout_hash", u64)]


_SIGS = {
    "ef_last_error": (C.c_char_p, []),
    "ef_abi_version": (C.c_int, []),
    "ef_expected_expert_count": (C.c_int, [P(f64), C.c_int, f64, P(C.c_int)]),
    "ef_top_experts": (C.c_int, [P(f64), C.c_int, C.c_int, P(C.c_int)]),
    "ef_swap_in_latency": (C.c_int, [i64, i64, i64, P(i64)]),
    "ef_compute_step_int": (C.c_int, [i64, i64, i64, i64, C.c_int, C.c_int, P(C.c_int)]),
    "ef_compute_step_float": (C.c_int, [i64, i64, f64, i64, C.c_int, C.c_int, P(C.c_int)]),
    "ef_step_validate": (C.c_int, [P(StepStateC)]),
    "ef_step_on_stall": (C.c_int, [P(StepStateC)]),
    "ef_step_on_overfetch": (C.c_int, [P(StepStateC)]),
    "ef_cache_create": (C.c_int, [i64, i64, C.c_int, P(vp)]),
    "ef_cache_destroy": (None, [vp]),
    "ef_cache_access": (C.c_int, [vp, i32, i32, i64, P(C.c_int)]),
    "ef_cache_admit": (C.c_int, [vp, i32, i32, C.c_int, i64, P(i32), C.c_int, P(C.c_int)]),
    "ef_cache_reassign_tiers": (C.c_int, [vp, P(i32), C.c_int, i64, i64]),
    "ef_cache_query": (C.c_int, [vp, i32, i32, P(C.c_int), P(i64)]),
    "ef_cache_counters": (C.c_int, [vp, P(i64)]),
    "ef_cache_resident": (C.c_int, [vp, P(i32), C.c_int, P(C.c_int)]),
    "ef_cache_events": (C.c_int, [vp, P(i64), i64, P(i64)]),
    "ef_tqueue_create": (C.c_int, [P(vp)]),
    "ef_tqueue_destroy": (None, [vp]),
    "ef_tqueue_enqueue": (C.c_int, [vp, i32, i32, C.c_int, P(i64)]),
    "ef_tqueue_next": (C.c_int, [vp, P(i32), P(i32), P(C.c_int), P(i64), P(C.c_int)]),
    "ef_tqueue_len": (C.c_int, [vp, P(i64)]),
    "ef_xfer_create": (C.c_int, [i32, i32, P(vp)]),
    "ef_xfer_destroy": (None, [vp]),
    "ef_xfer_submit": (C.c_int, [vp, i32, i32, i32, vp, vp, i64, P(i64)]),
    "ef_xfer_pump": (C.c_int, [vp, P(i32)]),
    "ef_xfer_poll": (C.c_int, [vp, P(i64), i32, P(i32)]),
    "ef_xfer_wait": (C.c_int, [vp, i64]),
    "ef_xfer_stream_wait": (C.c_int, [vp, i64, vp]),
    "ef_xfer_bandwidth": (C.c_int, [vp, P(C.c_double), P(i64)]),
    "ef_bw_create": (C.c_int, [C.c_int, f64, f64, P(vp)]),
    "ef_bw_destroy": (None, [vp]),
    "ef_bw_observe": (C.c_int, [vp, i64, i64, P(f64)]),
    "ef_bw_estimate": (C.c_int, [vp, P(f64)]),
    "ef_pcache_create": (C.c_int, [C.c_int, P(vp)]),
    "ef_pcache_destroy": (None, [vp]),
    "ef_pcache_get": (C.c_int, [vp, P(i64), C.c_int, i64, i64, P(i64), i64, P(i64), P(C.c_int)]),
    "ef_pcache_put": (C.c_int, [vp, P(i64), C.c_int, i64, i64, P(i64), i64]),
    "ef_pcache_stats": (C.c_int, [vp, P(i64)]),
    "ef_forest_create": (C.c_int, [C.c_int, P(i64), P(i32), P(f64), P(i32), P(i32), P(f64), i32,
                                   i32, C.c_int, P(vp)]),
    "ef_forest_destroy": (None, [vp]),
    "ef_forest_predict": (C.c_int, [vp, P(f64), P(f64), P(f64)]),
    "ef_inference_features": (C.c_int, [P(f64), i64, i32, i32, i32, P(i64), C.c_int, i32, i32,
                                        P(i32), i64, P(f64)]),
    "ef_predict_experts": (C.c_int, [P(LadderCfg), vp, P(i64), C.c_int, i32, i32, P(f64), P(i32),
                                     i64, P(i64), i64, P(i64)]),
    "ef_route_batch": (C.c_int, [P(i32), i64, P(C.c_uint8), i32, P(i32), P(i32), P(i32), P(i32)]),
    "ef_sim_create": (C.c_int, [P(SimCfg), P(LadderCfg), P(vp)]),
    "ef_sim_destroy": (None, [vp]),
    "ef_sim_run_token": (C.c_int, [vp, P(i64), C.c_int, P(f64), P(i32), i64, P(i32), i64, P(i64),
                                   i32]),
    "ef_sim_metrics": (C.c_int, [vp, P(i64), i32, P(f64)]),
    "ef_sim_output": (C.c_int, [vp, i32, P(i64), i64, P(i64)]),
    "ef_sim_event_details": (C.c_int, [vp, C.c_char_p, i64, P(i64)]),
    "ef_fill_uniform": (C.c_int, [vp, vp, C.c_int, i64, u64, f32, i64]),
    "ef_stream_key": (u64, [u64, i32, i32, i32]),
    "ef_rmsnorm": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, f32]),
    "ef_router_logits": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp]),
    "ef_route_permute": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, f32, u64, u64, vp,
                                   vp, vp, vp, vp, vp]),
    "ef_expert_ffn_decode": (C.c_int, [vp, vp, vp, C.c_int, vp, i64, P(i32), P(i32), P(i32),
                                       C.c_int, C.c_int, C.c_int, C.c_int, vp, vp]),
    "ef_combine": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, f32]),
    "ef_gather_rows_bf16": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, vp]),
    "ef_grouped_gemm_bf16": (C.c_int, [vp, vp, i64, C.c_int, vp, i64, i64, vp, C.c_int, C.c_int,
                                       C.c_int, vp, C.c_int]),
    "ef_engine_create": (C.c_int, [P(EngineCfg), P(SimCfg), P(LadderCfg), P(vp)]),
    "ef_engine_destroy": (None, [vp]),
    "ef_engine_step": (C.c_int, [vp, vp, vp, C.c_int, P(i64), C.c_int]),
    "ef_engine_step_host": (C.c_int, [vp, vp, vp, vp, C.c_int, P(i64), C.c_int]),
    "ef_engine_prefill": (C.c_int, [vp, vp, vp, C.c_int, P(i64), C.c_int]),
    "ef_engine_metrics": (C.c_int, [vp, P(i64), i32, P(f64)]),
    "ef_engine_output": (C.c_int, [vp, i32, P(i64), i64, P(i64)]),
    "ef_engine_event_details": (C.c_int, [vp, C.c_char_p, i64, P(i64)]),
    "ef_engine_stats": (C.c_int, [vp, P(f64), C.c_int]),
    "ef_engine_peer_pool_handle": (C.c_int, [vp, vp, P(u64)]),
    "ef_engine_ptr": (C.c_int, [vp, C.c_int, P(vp)]),
    "ef_engine_slot_of": (C.c_int, [vp, i32, i32, P(i32)]),
    "ef_engine_routing_log": (C.c_int, [vp, i64, P(f32), i64, P(i32), i64, P(i32), P(i32), P(u64),
                                        P(u64), P(i64)]),
    "ef_engine_set_record": (C.c_int, [vp, i32]),
    "ef_ep_nccl_unique_id": (C.c_int, [vp]),
    "ef_ep_shard_view": (C.c_int, [P(f32), P(i32), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   P(f64), P(i32), P(i32), P(i32)]),
    "ef_ep_comm_create": (C.c_int, [C.c_int, C.c_int, vp, COLLECTIVE_CB, vp, P(vp)]),
    "ef_ep_comm_destroy": (None, [vp]),
    "ef_ep_dispatch": (C.c_int, [vp, vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                 C.c_int, i64, vp, vp]),
    "ef_ep_owner": (C.c_int, [vp, vp, i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                              C.c_int, C.c_int, C.c_int, vp, vp, vp, vp]),
    "ef_ep_combine": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, vp,
                                vp]),
    "ef_engine_reset": (C.c_int, [vp, P(SimCfg), f32]),
    "ef_engine_routing_x": (C.c_int, [vp, i64, P(f32), i64, P(i64), P(i32)]),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)  # AttributeError here means the .so is out of date
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_SIGS)


class CallbackError(RuntimeError):
    pass


_pending_exc = []  # exceptions raised inside Python callbacks, re-raised after the call


def check(status: int) -> None:
    if status == EF_OK:
        return
    if _pending_exc:
        exc = _pending_exc.pop()
        _pending_exc.clear()
        raise exc
    msg = (lib.ef_last_error() or b"").decode(errors="replace")
    if status == EF_EINVAL:
        raise ValueError(msg)
    if status == EF_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def as_ptr(arr: np.ndarray, ctype):
    return arr.ctypes.data_as(P(ctype))


def f64arr(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def i32arr(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


def i64arr(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64))


class Handle:
    """Owns an opaque C object; destroys it with ``destroy`` on GC."""

    def __init__(self, ptr, destroy):
        self._ptr = ptr
        self._destroy = destroy

    @property
    def ptr(self):
        return self._ptr

    def __del__(self):
        if getattr(self, "_ptr", None):
            try:
                self._destroy(self._ptr)
            except Exception:
                pass
            self._ptr = None
