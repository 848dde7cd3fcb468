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
    """ef_engine_cfg in include/expertflow.h and the ctypes mirror declare the
    same fields in the same order."""
    import os
    import re
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "expertflow.h")).read()
    body = hdr[hdr.index("typedef struct ef_engine_cfg {") + len("typedef struct ef_engine_cfg {"):
               hdr.index("} ef_engine_cfg;")]
    body = re.sub(r"/\*.*?\*/", " ", body, flags=re.S)
    names = []
    for stmt in body.split(";"):
        stmt = stmt.replace("*", " ").strip()
        if not stmt:
            continue
        chunks = stmt.split(",")
        names.append(chunks[0].split()[-1])
        names += [c.strip() for c in chunks[1:]]
    assert names == [f[0] for f in L.EngineCfg._fields_]
    assert names[-7:-2] == ["ep_world", "ep_rank", "ep_nccl_id", "ep_collective", "ep_user"]


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
    # run the arm in-process of a child that reports whether the product
    # library was ever mapped (the reference arm must not load it)
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', "
            "'tiny', '--steps', '2', '--warmup', '1']; runpy.run_path('bench.py', "
            "run_name='__main__'); print('MAPPED', any('libexpertflow' in l "
            "for l in open('/proc/self/maps')), 'TORCH', 'torch' in sys.modules)")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["reference_scheduler_us_per_layer"] > 0
    assert "MAPPED False TORCH False" in out.stdout, out.stdout[-500:]


def test_routing_mask_top_up_rule():
    """Cache-aware routing mask (oracle/numerics.py routing_mask, engine.cu
    residency_mask + kernels.cu topup_mask): residents only, unless the batch
    could exceed the layer's cache share (ntok*k > U) and fewer than k experts
    are resident; then the non-residents with the most unbiased top-k votes
    (ties: larger max logit, then lower index) top it up to U = max(k, budget // L)."""
    import numpy as np
    from oracle import numerics as N
    M, k, L, budget = 8, 2, 4, 12  # U = 3
    lg = np.array([[0.1, 0.9, 0.0, 0.8, 0.2, 0.0, 0.0, 0.0],
                   [0.0, 0.7, 0.0, 0.1, 0.0, 0.0, 0.6, 0.0]], dtype=np.float32)
    # votes: e1 = 2, e3 = 1, e6 = 1 (max logit 0.8 vs 0.6)
    res = [False, False, True, False, False, False, False, False]
    assert N.routing_mask(res, M, k, budget, L, 1, lg[:1]) == 1 << 2          # 1*2 <= 3
    assert N.routing_mask(res, M, k, budget, L, 2, lg) == (1 << 2) | (1 << 1) | (1 << 3)
    none = [False] * M
    assert N.routing_mask(none, M, k, budget, L, 2, lg) == (1 << 1) | (1 << 3) | (1 << 6)
    two = [True, False, False, True, False, False, False, False]
    assert N.routing_mask(two, M, k, budget, L, 32, lg) == 0b1001         # k resident: no top-up
    assert N.routing_mask(none, M, k, 0, L, 32, lg) == (1 << 1) | (1 << 3)  # U = k
    tie = np.zeros((2, M), dtype=np.float32)                              # all equal: index order
    assert N.routing_mask(none, M, k, budget, L, 2, tie) == 0b111
    assert N.mask_bits(0b101, 4).tolist() == [True, False, True, False]
