"""CPU tests of the engine's host-side API surface: the product path has no
CPU fallback (it fails loudly without a CUDA device), argument validation of
the new entry points, and the C-ABI engine struct layout."""

import ctypes as C

import pytest
import torch

import paper_2510_26730_b200 as ef
from paper_2510_26730_b200 import _lib as L
from paper_2510_26730_b200.runtime import PRESETS, MoEEngine


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_engine_refuses_to_run_without_cuda():
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        MoEEngine(PRESETS["tiny"], budget_experts=16, policy=ef.PolicyConfig("s", "static"),
                  link_bw=ef.GB, layer_time_s=1e-4)


def test_compare_engines_validates_policies():
    cfg = PRESETS["tiny"]
    with pytest.raises(ValueError, match="no policies"):
        ef.compare_engines(cfg, [], [])
    p = ef.PolicyConfig("a", "adaptive", predictor="pregate")
    with pytest.raises(ValueError, match="duplicate"):
        ef.compare_engines(cfg, [p, p], [])


def test_engine_cfg_struct_matches_header():
    """ef_engine_cfg in include/expertflow.h and the ctypes mirror agree on
    field order (the last fields were appended for prefill and the shared
    host store)."""
    names = [f[0] for f in L.EngineCfg._fields_]
    assert names[-7:] == ["max_prefill", "host_store_shm", "host_store_attach", "peer_device",
                          "peer_pool_experts", "peer_pool_ids", "peer_ipc_handle"]
    hdr = open(__import__("os").path.join(__import__("os").path.dirname(__file__), "..",
                                          "include", "expertflow.h")).read()
    body = hdr[hdr.index("typedef struct ef_engine_cfg"):hdr.index("} ef_engine_cfg;")]
    pos = [body.index(n) for n in ("record_routing", "max_prefill", "host_store_shm",
                                   "host_store_attach", "peer_device", "peer_pool_experts",
                                   "peer_pool_ids", "peer_ipc_handle")]
    assert pos == sorted(pos)
    assert C.sizeof(L.EngineCfg) >= 96


def test_new_entry_points_exported():
    for name in ("ef_engine_prefill", "ef_engine_step_host", "ef_grouped_gemm_bf16"):
        assert hasattr(L.lib, name)


def test_bench_reference_arm_contract():
    """bench.py --impl reference prints one JSON line with the contract's keys
    (tiny config, one step, so it runs in seconds on the CPU)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                          "--config", "tiny", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1


def test_routing_mask_top_up_rule():
    """Cache-aware routing mask (oracle/numerics.py routing_mask, engine.cu
    residency_mask): residents only, unless the batch could exceed the layer's
    cache share (ntok*k > U) and fewer than k experts are resident; then the
    lowest-index non-resident experts top it up to U = max(k, budget // L)."""
    from oracle import numerics as N
    M, k, L, budget = 8, 2, 4, 12  # U = 3
    res = [False, False, True, False, False, False, False, False]
    assert N.routing_mask(res, M, k, budget, L, 1) == 1 << 2          # 1*2 <= 3: residents only
    assert N.routing_mask(res, M, k, budget, L, 2) == 0b111           # top up to 3 experts
    two = [True, False, False, True, False, False, False, False]
    assert N.routing_mask(two, M, k, budget, L, 32) == 0b1001         # k resident: no top-up
    assert N.routing_mask([False] * M, M, k, 0, L, 32) == 0b11        # U = k when budget < L
    assert N.mask_bits(0b101, 4).tolist() == [True, False, True, False]
