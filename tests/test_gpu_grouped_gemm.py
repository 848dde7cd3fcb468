"""TMA + tcgen05 grouped GEMM (prefill expert FFN) against the CPU oracle on
ragged expert segments, through the C ABI."""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2510_26730_b200 import _lib as L  # noqa: E402
from oracle import numerics as N  # noqa: E402

DEV = "cuda:0"


def tiles_for(segments, n_cols, b_rows_of, bm=128, bn=128):
    """(expert, n, m) ordered tiles: {a_row0, b_row0, m_valid, n0}."""
    out = []
    row = 0
    for e, n in enumerate(segments):
        for n0 in range(0, n_cols, bn):
            for m0 in range(0, n, bm):
                out.append((row + m0, b_rows_of(e), min(bm, n - m0), n0))
        row += n
    return np.array(out, dtype=np.int32).reshape(-1, 4)


def run(A, B, tiles, K, dual, dual_off, out):
    t = torch.tensor(tiles, device=DEV)
    L.check(L.lib.ef_grouped_gemm_bf16(
        C.c_void_p(torch.cuda.current_stream().cuda_stream), C.c_void_p(A.data_ptr()),
        A.shape[0], K, C.c_void_p(B.data_ptr()), B.shape[0], B.shape[1],
        C.c_void_p(t.data_ptr()), tiles.shape[0], int(dual), dual_off,
        C.c_void_p(out.data_ptr()), out.shape[1]))
    torch.cuda.synchronize()


@pytest.mark.parametrize("K,NF,segments", [(256, 128, [128]), (512, 256, [37, 200, 0, 5, 128]),
                                           (2048, 1408, [192, 64, 300])])
def test_grouped_gemm_dual_swiglu(K, NF, segments):
    torch.manual_seed(0)
    E = len(segments)
    rows = sum(segments)
    A = (torch.randn(rows, K, device=DEV) / 4).to(torch.bfloat16)
    # slab view: expert e = [W1 (NF rows) | W3 (NF rows) | pad], pitch K
    per = 3 * NF
    B = (torch.randn(E * per, K, device=DEV) / K ** 0.5).to(torch.bfloat16)
    tiles = tiles_for(segments, NF, lambda e: e * per)
    out = torch.zeros(rows, NF, device=DEV, dtype=torch.bfloat16)
    run(A, B, tiles, K, True, NF, out)
    a = A.float().cpu().numpy().astype(np.float64)
    b = B.float().cpu().numpy().astype(np.float64)
    got = out.float().cpu().numpy()
    r0 = 0
    for e, n in enumerate(segments):
        if n == 0:
            continue
        w1 = b[e * per:e * per + NF]
        w3 = b[e * per + NF:e * per + 2 * NF]
        g, u = a[r0:r0 + n] @ w1.T, a[r0:r0 + n] @ w3.T
        want = N.to_bf16((g / (1 + np.exp(-g)) * u).astype(np.float32))
        err = np.linalg.norm(got[r0:r0 + n] - want) / np.linalg.norm(want)
        assert err < 2e-2, (e, err)
        r0 += n


@pytest.mark.parametrize("K,ND,segments", [(1408, 2048, [192, 7, 129]), (256, 256, [1])])
def test_grouped_gemm_down_fp32(K, ND, segments):
    torch.manual_seed(1)
    E = len(segments)
    rows = sum(segments)
    A = (torch.randn(rows, K, device=DEV) / 4).to(torch.bfloat16)
    B = (torch.randn(E * ND, K, device=DEV) / K ** 0.5).to(torch.bfloat16)
    tiles = tiles_for(segments, ND, lambda e: e * ND)
    out = torch.zeros(rows, ND, device=DEV, dtype=torch.float32)
    run(A, B, tiles, K, False, 0, out)
    a = A.float().cpu().numpy().astype(np.float64)
    b = B.float().cpu().numpy().astype(np.float64)
    got = out.cpu().numpy()
    r0 = 0
    for e, n in enumerate(segments):
        want = a[r0:r0 + n] @ b[e * ND:(e + 1) * ND].T
        err = np.linalg.norm(got[r0:r0 + n] - want) / np.linalg.norm(want)
        assert err < 1e-3, (e, err)  # bf16 inputs, fp32 accumulation
        r0 += n
