"""Lab: decode-FFN pair (gate/up+SiLU, down) throughput through the C ABI
(ef_expert_ffn_decode) — the tensor-core path vs the GEMV pair
(EF_FFN_MMA=0 in a second process).  Prints GB/s of streamed expert weights."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_26730_b200 import _lib as L  # noqa: E402

CASES = [  # name, d, ff, experts, tokens per expert
    ("mixtral B1", 4096, 14336, 2, 1),
    ("qwen B1", 2048, 1408, 4, 1),
    ("qwen shared B1", 2048, 5632, 1, 1),
    ("qwen B8", 2048, 1408, 24, 1),
    ("qwen B32 routed", 2048, 1408, 49, 3),
    ("qwen B32 hot", 2048, 1408, 16, 8),
    ("qwen shared B32", 2048, 5632, 1, 32),
    ("mixtral B8", 4096, 14336, 8, 2),
]


def run(d, ff, E, n):
    es = 3 * d * ff * 2
    slab = torch.empty(E, es, dtype=torch.uint8, device="cuda")
    slab.view(torch.bfloat16).normal_(0, 0.02)
    rows = E * n
    x = torch.randn(rows, d, device="cuda")
    perm = torch.arange(rows, dtype=torch.int32, device="cuda")
    act = torch.empty(rows, ff, dtype=torch.bfloat16, device="cuda")
    y = torch.empty(rows, d, device="cuda")
    sl, off, nr = L.i32arr(range(E)), L.i32arr([i * n for i in range(E)]), L.i32arr([n] * E)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def go():
        L.check(L.lib.ef_expert_ffn_decode(st, C.c_void_p(x.data_ptr()), C.c_void_p(perm.data_ptr()), 1,
                                          C.c_void_p(slab.data_ptr()), es, L.as_ptr(sl, C.c_int32),
                                          L.as_ptr(off, C.c_int32), L.as_ptr(nr, C.c_int32), E, d, ff, 1,
                                          C.c_void_p(act.data_ptr()), C.c_void_p(y.data_ptr())))
    for _ in range(3):
        go()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        go()
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 20 / 1e3
    return E * es / t / 1e9, t * 1e6


tag = os.environ.get("EF_FFN_MMA", "1")
only = sys.argv[1] if len(sys.argv) > 1 else None
for name, d, ff, E, n in CASES:
    if only and name != only:
        continue
    gbs, us = run(d, ff, E, n)
    print(f"mma={tag} {name:18s} {us:8.1f} us {gbs:7.0f} GB/s", flush=True)
