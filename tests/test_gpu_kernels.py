"""Kernel-level parity on the B200 through the C ABI: each sm_100a kernel
against the CPU oracle (oracle/numerics.py) on the same seeded inputs."""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2510_26730_b200 as ef  # noqa: E402
from paper_2510_26730_b200 import _lib as L  # noqa: E402
from oracle import numerics as N  # noqa: E402

DEV = "cuda:0"


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return C.c_void_p(t.data_ptr())


def fill(n, key, scale, dtype):
    t = torch.empty(n, dtype=torch.bfloat16 if dtype == "bf16" else torch.float32, device=DEV)
    L.check(L.lib.ef_fill_uniform(stream(), ptr(t), 1 if dtype == "bf16" else 0, n, key,
                                  float(scale), 0))
    return t


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_fill_uniform_bit_exact(dtype):
    for layer, expert, mat, n in [(0, 0, 0, 4096), (3, 7, 2, 10007), (31, 5, 8, 1 << 16)]:
        key = N.stream_key(1234, layer, expert, mat)
        assert key == L.lib.ef_stream_key(1234, layer, expert, mat)
        scale = N.fan_scale(4096)
        got = fill(n, key, scale, dtype).float().cpu().numpy()
        want = N.cast(N.fill_uniform(key, n, scale), dtype)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("dtype,B,M,d,R", [("f32", 1, 8, 256, 1), ("bf16", 3, 60, 2048, 4),
                                           ("bf16", 32, 64, 2048, 2), ("bf16", 1, 8, 6144, 5)])
def test_router_logits(dtype, B, M, d, R):
    key = N.stream_key(9, 0, 0, 3)
    w = fill(R * M * d, key, N.fan_scale(d), dtype)
    x = torch.randn(B, d, device=DEV, dtype=torch.float32)
    out = torch.empty(R, B, M, device=DEV)
    L.check(L.lib.ef_router_logits(stream(), ptr(x), ptr(w), 1 if dtype == "bf16" else 0, R, B, d,
                                   M, ptr(out)))
    wr = N.cast(N.fill_uniform(key, R * M * d, N.fan_scale(d)), dtype).reshape(R, M, d)
    want = np.einsum("bd,rmd->rbm", x.cpu().numpy().astype(np.float64), wr.astype(np.float64))
    got = out.cpu().numpy()
    assert np.abs(got - want).max() <= 1e-5 * np.abs(want).max() + 1e-6


def run_route(logits, k, mode, bias=0.0, mask=0):
    B, M = logits.shape
    lg = torch.tensor(logits, device=DEV)
    sel = torch.empty(B, k, dtype=torch.int32, device=DEV)
    wts = torch.empty(B, k, device=DEV)
    counts = torch.empty(M, dtype=torch.int32, device=DEV)
    offs = torch.empty(M + 1, dtype=torch.int32, device=DEV)
    perm = torch.empty(B * k, dtype=torch.int32, device=DEV)
    inv = torch.empty(B * k, dtype=torch.int32, device=DEV)
    L.check(L.lib.ef_route_permute(stream(), ptr(lg), B, M, k, 0 if mode == "mixtral" else 1,
                                   float(bias), mask & ((1 << 64) - 1), mask >> 64, ptr(sel),
                                   ptr(wts), ptr(counts), ptr(offs), ptr(perm), ptr(inv)))
    return [t.cpu().numpy() for t in (sel, wts, counts, offs, perm, inv)]


@pytest.mark.parametrize("B,M,k,mode", [(1, 8, 2, "mixtral"), (7, 60, 4, "softmax_topk"),
                                        (32, 64, 6, "softmax_topk"), (2048, 64, 6, "softmax_topk"),
                                        (1, 8, 8, "mixtral"), (5, 128, 16, "mixtral")])
def test_route_permute_bit_exact(B, M, k, mode):
    rng = np.random.default_rng(B * 1000 + M)
    logits = rng.standard_normal((B, M)).astype(np.float32)
    logits[:, ::7] = logits[:, :1]  # planted exact ties -> lower index wins
    if B > 1:
        logits[1] = 0.5  # a fully tied row
    sel, wts, counts, offs, perm, inv = run_route(logits, k, mode)
    want_sel = N.topk_select(logits, k)
    assert np.array_equal(sel, want_sel)
    assert np.abs(wts - N.route_weights(logits, want_sel, mode)).max() < 2e-6
    c, o, p, i = N.permute(want_sel, M)
    assert np.array_equal(counts, c) and np.array_equal(offs, o)
    assert np.array_equal(perm, p) and np.array_equal(inv.reshape(B, k), i)


def test_route_cache_aware_bias():
    rng = np.random.default_rng(3)
    B, M, k = 6, 60, 4
    logits = rng.standard_normal((B, M)).astype(np.float32)
    resident = rng.random(M) < 0.4
    mask = sum(1 << e for e in range(M) if resident[e])
    for bias in (0.5, 3.0, 100.0):
        sel, *_ = run_route(logits, k, "softmax_topk", bias, mask)
        assert np.array_equal(sel, N.topk_select(logits, k, bias, resident))
    sel, *_ = run_route(logits, k, "softmax_topk", 100.0, mask)
    assert resident[sel].all()


@pytest.mark.parametrize("dtype,d,ff,rows", [("f32", 256, 1024, [1, 2]),
                                              ("bf16", 2048, 1408, [1, 3, 5, 2]),
                                              ("bf16", 4096, 14336, [1, 1]),
                                              ("bf16", 2048, 1408, [9, 12, 1]),
                                              ("f32", 512, 768, [4, 8, 3])])
def test_expert_ffn_decode(dtype, d, ff, rows):
    E = len(rows)
    es = 2 if dtype == "bf16" else 4
    stride = 3 * d * ff * es
    slab = torch.empty(E + 1, stride, dtype=torch.uint8, device=DEV)
    slots = list(range(E, 0, -1))  # non-identity slot mapping
    w_cpu = []
    for i, s in enumerate(slots):
        mats = []
        for m, (r, c, fan) in enumerate([(ff, d, d), (ff, d, d), (d, ff, ff)]):
            key = N.stream_key(77, 0, i, m)
            t = fill(r * c, key, N.fan_scale(fan), dtype)
            off = (0, ff * d, 2 * ff * d)[m] * es
            slab[s, off:off + r * c * es] = t.view(torch.uint8)
            mats.append(N.cast(N.fill_uniform(key, r * c, N.fan_scale(fan)), dtype).reshape(r, c))
        w_cpu.append(mats)
    n = sum(rows)
    k = 1
    x = torch.randn(n, d, device=DEV)
    perm = torch.arange(n, dtype=torch.int32, device=DEV)
    act = torch.empty(n, ff, dtype=torch.bfloat16 if dtype == "bf16" else torch.float32, device=DEV)
    y = torch.empty(n, d, device=DEV)
    offs = np.cumsum([0] + rows[:-1]).astype(np.int32)
    a_slot, a_off, a_rows = L.i32arr(slots), L.i32arr(offs), L.i32arr(rows)
    L.check(L.lib.ef_expert_ffn_decode(
        stream(), ptr(x), ptr(perm), k, ptr(slab), stride, L.as_ptr(a_slot, C.c_int32),
        L.as_ptr(a_off, C.c_int32), L.as_ptr(a_rows, C.c_int32), E, d, ff,
        1 if dtype == "bf16" else 0, ptr(act), ptr(y)))
    got = y.cpu().numpy()
    xe = N.cast(x.cpu().numpy(), dtype)
    tol = 1e-5 if dtype == "f32" else 2e-2
    for i in range(E):
        r0, r1 = offs[i], offs[i] + rows[i]
        want = N.swiglu(xe[r0:r1], *w_cpu[i], dtype)
        err = np.linalg.norm(got[r0:r1] - want) / np.linalg.norm(want)
        assert err < tol, (i, err)


def test_combine_and_rmsnorm():
    B, d, k = 5, 2048, 4
    rng = np.random.default_rng(1)
    h = rng.standard_normal((B, d)).astype(np.float32)
    y = rng.standard_normal((B * k + 3, d)).astype(np.float32)
    inv = rng.permutation(B * k).astype(np.int32)
    wts = rng.random((B, k)).astype(np.float32)
    ys = rng.standard_normal((B, d)).astype(np.float32)
    gl = rng.standard_normal(B).astype(np.float32)
    th = torch.tensor(h, device=DEV)
    tx = torch.empty(B, d, device=DEV)
    # keep every device buffer alive until the kernel has run
    ty, tinv, tw, tys, tgl = (torch.tensor(a, device=DEV) for a in (y, inv, wts, ys, gl))
    L.check(L.lib.ef_combine(stream(), ptr(th), ptr(tx), ptr(ty), ptr(tinv), ptr(tw), ptr(tys),
                             ptr(tgl), B, d, k, 1e-6))
    torch.cuda.synchronize()
    inv2 = inv.reshape(B, k)
    want = h.astype(np.float64).copy()
    for t in range(B):
        for r in range(k):
            want[t] += wts[t, r] * y[inv2[t, r]]
        want[t] += ys[t] / (1.0 + np.exp(-float(gl[t])))
    assert np.abs(th.cpu().numpy() - want).max() < 1e-4
    assert np.abs(tx.cpu().numpy() - N.rmsnorm(want)).max() < 1e-5
    t2 = torch.empty(B, d, device=DEV)
    th2 = torch.tensor(h, device=DEV)
    L.check(L.lib.ef_rmsnorm(stream(), ptr(th2), ptr(t2), B, d, 1e-6))
    torch.cuda.synchronize()
    assert np.abs(t2.cpu().numpy() - N.rmsnorm(h)).max() < 1e-5


@pytest.mark.gpu
def test_transfer_engine_priority_order_and_bandwidth():
    """ef_xfer_*: copies land byte-exact, issue in TransferQueue order (every
    MISS before any PREFETCH, FIFO within a class; memory.py:184-202) on the
    one-copy link, device-side waits order a consumer stream after a copy,
    and the measured rate reaches the bandwidth estimate."""
    import torch
    n, nbytes = 6, 8 << 20
    src = [torch.randint(0, 255, (nbytes,), dtype=torch.uint8).pin_memory() for _ in range(n)]
    dst = [torch.empty(nbytes, dtype=torch.uint8, device="cuda") for _ in range(n)]
    x = C.c_void_p()
    L.check(L.lib.ef_xfer_create(0, 1, C.byref(x)))
    try:
        prios = [1, 1, 0, 1, 0, 0]  # PREFETCH, PREFETCH, MISS, PREFETCH, MISS, MISS
        tick = []
        for i, p in enumerate(prios):
            t = C.c_int64()
            L.check(L.lib.ef_xfer_submit(x, 0, i, p, C.c_void_p(src[i].data_ptr()),
                                         C.c_void_p(dst[i].data_ptr()), nbytes, C.byref(t)))
            tick.append(t.value)
        assert tick == list(range(n))
        st = torch.cuda.Stream()
        L.check(L.lib.ef_xfer_pump(x, None))
        L.check(L.lib.ef_xfer_stream_wait(x, 2, C.c_void_p(st.cuda_stream)))  # the first MISS
        with torch.cuda.stream(st):
            probe = dst[2].sum(dtype=torch.int64)
        L.check(L.lib.ef_xfer_wait(x, 3))  # the last PREFETCH: everything has landed
        buf = (C.c_int64 * n)()
        got = C.c_int32()
        L.check(L.lib.ef_xfer_poll(x, buf, n, C.byref(got)))
        assert list(buf[:got.value]) == [2, 4, 5, 0, 1, 3], list(buf[:got.value])
        st.synchronize()
        assert int(probe) == int(src[2].sum(dtype=torch.int64))
        for i in range(n):
            assert torch.equal(dst[i].cpu(), src[i])
        bw, done = C.c_double(), C.c_int64()
        L.check(L.lib.ef_xfer_bandwidth(x, C.byref(bw), C.byref(done)))
        assert done.value == n and 1e9 < bw.value < 1e12, bw.value
    finally:
        L.lib.ef_xfer_destroy(x)
