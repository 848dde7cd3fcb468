"""The CPU decode port (oracle/cpu_port.py + oracle/cport.c) — the CPU
implementation bench.py times beside the GPU — against the float64 oracle
(oracle/numerics.py) and the reference scheduler restatement."""

import numpy as np
import pytest

from oracle import cpu_port as CP
from oracle import numerics as N
from oracle.sim import Policy


def test_fill_matches_numpy_generator():
    key = N.stream_key(5, 3, 2, 1)
    got = CP.fill(key, 4099, N.fan_scale(512), "bf16")
    want = N.to_bf16(N.fill_uniform(key, 4099, N.fan_scale(512)))
    assert np.array_equal((got.astype(np.uint32) << 16).view(np.float32), want)


@pytest.mark.parametrize("dtype,shape", [("f32", (4, 8, 2, 256, 1024, 0, False, "mixtral")),
                                         ("bf16", (2, 16, 4, 512, 256, 512, True, "softmax_topk"))])
def test_decode_port_matches_fp64_oracle(dtype, shape):
    L, M, k, d, ff, sff, sg, mode = shape
    pol = Policy("adaptive", "adaptive", predictor="pregate")
    port = CP.CpuDecodePort(L=L, M=M, k=k, d=d, ff=ff, dtype=dtype, route_mode=mode, shared_ff=sff,
                            shared_gate=sg, seed=3, budget_experts=L * M // 2, policy=pol,
                            link_bw=4_000_000_000, layer_ns=200_000, bias=0.0)
    w = N.ModelWeights(L=L, M=M, d=d, ff=ff, dtype=dtype, seed=3, shared_ff=sff, shared_gate=sg)
    tol = 1e-5 if dtype == "f32" else 2e-2
    for t in range(3):
        h0 = N.input_hidden(3, t, 3, d)
        got = port.step(h0)
        h = h0.astype(np.float64)
        for l in range(L):
            lg, sel = port.last_sel[l]
            ref = N.moe_layer(h, w, l, k, mode)
            assert np.array_equal(ref["sel"], sel) or np.allclose(ref["logits"], lg, atol=1e-4)
            h = N.moe_layer(h, w, l, k, mode, logits_override=lg, sel_override=sel)["h_next"]
        err = np.linalg.norm(got - h) / np.linalg.norm(h)
        assert err < tol, (t, err)
    m = port.st.metrics
    assert m.hits + m.misses > 0 and port.layers_run == 3 * L
    assert port.compute_s > 0 and port.sched_s > 0


def test_decode_port_bias_routes_to_residents():
    """With the residency-first bias the port routes like the engine: every
    selected expert of a layer is resident whenever >= k are."""
    L, M, k = 4, 8, 2
    pol = Policy("adaptive", "adaptive", predictor="pregate", cache_aware_routing=True)
    port = CP.CpuDecodePort(L=L, M=M, k=k, d=256, ff=512, dtype="bf16", route_mode="mixtral",
                            seed=1, budget_experts=16, policy=pol, link_bw=2_000_000_000,
                            layer_ns=100_000, bias=1e4)
    for t in range(6):
        port.step(N.input_hidden(1, t, 1, 256))
    m = port.st.metrics
    assert m.hits / (m.hits + m.misses) > 0.5
