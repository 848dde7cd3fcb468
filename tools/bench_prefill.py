"""C4 prefill expert-FFN measurement: DeepSeek-V2-Lite shape (d=2048, ff=1408,
64 experts, top-6), 2048-token prefill; routing from the fp32 router on
random hidden states; weights in a slot slab; the TMA + tcgen05 grouped GEMM
(gate/up with fused SiLU*up, then down).  Prints one JSON line with
TFLOP/s (vs measured dense bf16 peak) and weight GB/s (vs measured HBM peak).

    python tools/bench_prefill.py [--tokens 2048] [--reps 20]
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_26730_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=2048)
ap.add_argument("--experts", type=int, default=64)
ap.add_argument("--topk", type=int, default=6)
ap.add_argument("--d", type=int, default=2048)
ap.add_argument("--ff", type=int, default=1408)
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
T, M, k, d, ff = args.tokens, args.experts, args.topk, args.d, args.ff
dev = torch.device("cuda", 0)
torch.manual_seed(0)
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)

# routing: fp32 router on random hidden states, top-k per token (kernel (a))
x = torch.randn(T, d, device=dev)
wr = (torch.randn(M, d, device=dev) / d ** 0.5).to(torch.bfloat16)
logits = torch.empty(1, T, M, device=dev)
L.check(L.lib.ef_router_logits(st, C.c_void_p(x.data_ptr()), C.c_void_p(wr.data_ptr()), 1, 1, T,
                               d, M, C.c_void_p(logits.data_ptr())))
sel = torch.topk(logits[0], k, dim=1).indices.cpu().numpy()
counts = np.bincount(sel.reshape(-1), minlength=M)
rows = int(counts.sum())
A = (torch.randn(rows, d, device=dev) / 2).to(torch.bfloat16)  # permuted tokens
stride_rows_up = 3 * ff          # slab view with pitch d: [W1 | W3 | W2-as-rows]
slab = (torch.randn(M, 3 * ff * d, device=dev) / d ** 0.5).to(torch.bfloat16)
act = torch.empty(rows, ff, device=dev, dtype=torch.bfloat16)
y = torch.empty(rows, d, device=dev, dtype=torch.float32)


def tiles(n_cols, b_row_of):
    out, r = [], 0
    for e in range(M):
        n = int(counts[e])
        for n0 in range(0, n_cols, 128):
            for m0 in range(0, n, 128):
                out.append((r + m0, b_row_of(e), min(128, n - m0), n0))
        r += n
    return torch.tensor(np.array(out, dtype=np.int32), device=dev)


t_up = tiles(ff, lambda e: e * 3 * ff)                   # W1/W3 rows in the pitch-d view
t_dn = tiles(d, lambda e: e * 3 * d + 2 * d)             # W2 rows in the pitch-ff view
slab_rows_d = M * 3 * ff
slab_rows_ff = M * 3 * d


def run():
    L.check(L.lib.ef_grouped_gemm_bf16(st, C.c_void_p(A.data_ptr()), rows, d,
                                       C.c_void_p(slab.data_ptr()), slab_rows_d, d,
                                       C.c_void_p(t_up.data_ptr()), t_up.shape[0], 1, ff,
                                       C.c_void_p(act.data_ptr()), ff))
    L.check(L.lib.ef_grouped_gemm_bf16(st, C.c_void_p(act.data_ptr()), rows, ff,
                                       C.c_void_p(slab.data_ptr()), slab_rows_ff, ff,
                                       C.c_void_p(t_dn.data_ptr()), t_dn.shape[0], 0, 0,
                                       C.c_void_p(y.data_ptr()), d))


for _ in range(3):
    run()
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ms = []
for _ in range(args.reps):
    flush.zero_()  # evict the slab from L2 between reps
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    run()
    e.record()
    torch.cuda.synchronize()
    ms.append(s.elapsed_time(e))
med = float(np.median(ms))
flops = 2.0 * rows * d * 2 * ff + 2.0 * rows * ff * d
wbytes = float((counts > 0).sum()) * 3 * d * ff * 2
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}
# spot-check the result against a torch reference on one expert
e0 = int(np.argmax(counts))
r0 = int(counts[:e0].sum())
n0 = int(counts[e0])
xa = A[r0:r0 + n0].float()
w = slab[e0].view(3 * ff, d).float()
g, u = xa @ w[:ff].T, xa @ w[ff:2 * ff].T
ref_act = (torch.nn.functional.silu(g) * u)
err = float((act[r0:r0 + n0].float() - ref_act).norm() / ref_act.norm())
tflops = flops / (med / 1e3) / 1e12
print(json.dumps({
    "what": "C4 prefill routed-expert FFN (grouped tcgen05 GEMM: up+SiLU, down)",
    "tokens": T, "rows": rows, "active_experts": int((counts > 0).sum()),
    "ms": med, "tflops": tflops, "tensor_frac": tflops / peaks["bf16_tflops"],
    "weight_GBps": wbytes / (med / 1e3) / 1e9,
    "hbm_frac": wbytes / (med / 1e3) / 1e9 / peaks["hbm_gbs"],
    "gflop": flops / 1e9, "weight_MB": wbytes / 1e6, "rel_err_act_vs_torch": err,
    "roofline_ms": max(flops / (peaks["bf16_tflops"] * 1e12), wbytes / (peaks["hbm_gbs"] * 1e9)) * 1e3,
}))
