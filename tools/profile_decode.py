"""Small decode driver for ncu / launch lists (run with EF_PIPE_DEBUG=1 under
ncu: ncu serialises launches, so the host must publish each layer's decision
before the gate kernel is launched).

    EF_PIPE_DEBUG=1 python tools/profile_decode.py --layers 2 --steps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2510_26730_b200 as ef  # noqa: E402
from paper_2510_26730_b200.runtime import PRESETS, MoEConfig, MoEEngine, synthetic_hidden  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mixtral-8x7b")
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--bias", type=float, default=1e4)
ap.add_argument("--policy", default="static")
ap.add_argument("--budget-frac", type=float, default=1.0)
args = ap.parse_args()
base = PRESETS[args.config]
cfg = MoEConfig(base.name + f"-{args.layers}l", args.layers, base.num_experts, base.top_k,
                base.d_model, base.d_ff, base.dtype, base.route_mode, base.shared_ff,
                base.shared_gate)
pol = ef.PolicyConfig("p", args.policy, predictor="pregate" if args.policy != "static" else "none")
eng = MoEEngine(cfg, budget_experts=max(cfg.top_k, int(args.budget_frac * cfg.total_experts)),
                policy=pol,
                link_bw=55_000_000_000, layer_time_s=1e-4, max_batch=args.batch,
                routing_bias=args.bias, timing=True)
h = synthetic_hidden(cfg, 0, 0, args.batch, torch.device("cuda", 0))
for _ in range(args.steps):
    eng.step(h)
torch.cuda.synchronize()
print(eng.stats())
