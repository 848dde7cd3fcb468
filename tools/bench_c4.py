"""C4 end to end: DeepSeek-V2-Lite shape (26 MoE layers, 64 experts top-6,
2 shared experts, bf16 random-init), 40 % expert-cache budget, a 2K-token
prefill through MoEEngine.prefill() (expert FFNs on the tcgen05/TMA grouped
GEMM), then batch-1 decode steps from the same cache.  One JSON line.

    python tools/bench_c4.py [--tokens 2048] [--decode 32] [--bias 1e4]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_26730_b200 as ef  # noqa: E402
from paper_2510_26730_b200.runtime import PRESETS, MoEEngine, synthetic_hidden  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=2048)
ap.add_argument("--decode", type=int, default=32)
ap.add_argument("--budget-frac", type=float, default=0.4)
ap.add_argument("--bias", type=float, default=1e4)
ap.add_argument("--link-gbps", type=float, default=55.0)
args = ap.parse_args()
cfg = PRESETS["deepseek-v2-lite"]
dev = torch.device("cuda", 0)
budget = int(round(args.budget_frac * cfg.total_experts))
pol = ef.PolicyConfig("adaptive_pregate", "adaptive", predictor="pregate", cache_aware_routing=True)
t0 = time.perf_counter()
eng = MoEEngine(cfg, budget_experts=budget, policy=pol, link_bw=int(args.link_gbps * 1e9),
                layer_time_s=6e-5, max_batch=1, routing_bias=args.bias, timing=True,
                max_prefill=args.tokens)
init_s = time.perf_counter() - t0
T = args.tokens
h = synthetic_hidden(cfg, 0, 0, T, dev)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st0 = eng.stats()
s.record()
eng.prefill(h, list(range(T)))
e.record()
torch.cuda.synchronize()
pre_ms = s.elapsed_time(e)
st1 = eng.stats()
m1 = eng.metrics()
finite = bool(torch.isfinite(h).all())
xs = [synthetic_hidden(cfg, 0, 1 + t, 1, dev) for t in range(args.decode + 4)]
for t in range(4):
    eng.step(xs[t], [T + t])
torch.cuda.synchronize()
st2 = eng.stats()
s.record()
for t in range(4, 4 + args.decode):
    eng.step(xs[t], [T + t])
e.record()
torch.cuda.synchronize()
dec_ms = s.elapsed_time(e)
st3 = eng.stats()
gemm_flop = 2.0 * T * cfg.top_k * cfg.d_model * 3 * cfg.d_ff + 2.0 * T * cfg.d_model * 3 * cfg.shared_ff
print(json.dumps({
    "what": "C4 DeepSeek-V2-Lite shape: 2K prefill (grouped tcgen05 GEMM) + batch-1 decode, "
            f"budget {budget}/{cfg.total_experts} experts",
    "prefill_tokens": T, "prefill_ms": pre_ms, "prefill_tokens_per_s": T / (pre_ms / 1e3),
    "prefill_copies": st1["copies"] - st0["copies"],
    "prefill_copy_GB": (st1["copy_bytes"] - st0["copy_bytes"]) / 1e9,
    "prefill_h2d_GBps": (st1["copy_bytes"] - st0["copy_bytes"]) / (pre_ms / 1e3) / 1e9,
    "prefill_expert_gemm_gflop": gemm_flop * cfg.num_layers / 1e9,
    "prefill_logical_stall_pct": 100.0 * m1.waiting_ns / max(1, m1.total_time_ns),
    "prefill_output_finite": finite,
    "decode_steps": args.decode, "decode_tokens_per_s": args.decode / (dec_ms / 1e3),
    "decode_copies_per_step": (st3["copies"] - st2["copies"]) / args.decode,
    "decode_fast_layers": st3["fast_layers"] - st2["fast_layers"],
    "routing_bias": args.bias, "engine_init_s": round(init_s, 1),
}))
