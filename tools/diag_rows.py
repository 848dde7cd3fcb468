"""Diagnostic: per-entry router-row and layer-input errors of a B=1 engine
run against the fp64 oracle, under the EF_FUSE / EF_PDL setting of the env."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_26730_b200 as ef
from paper_2510_26730_b200.runtime import MoEConfig, MoEEngine, synthetic_hidden
from oracle import numerics as N, replay as R

shape = sys.argv[1] if len(sys.argv) > 1 else "qwen"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
if shape == "qwen":
    cfg = MoEConfig("qwen-2l", 2, 60, 4, 2048, 1408, route_mode="softmax_topk", shared_ff=5632,
                    shared_gate=True)
    budget = 48
elif shape == "qwen-noshared":
    cfg = MoEConfig("qwen-2l-ns", 2, 60, 4, 2048, 1408, route_mode="softmax_topk")
    budget = 48
else:
    cfg = MoEConfig("ds-2l", 2, 64, 6, 2048, 1408, route_mode="softmax_topk", shared_ff=2816)
    budget = 51
dev = torch.device("cuda", 0)
eng = MoEEngine(cfg, budget_experts=budget, policy=ef.PolicyConfig("a", "adaptive", predictor="pregate"),
                link_bw=50 * ef.GB, layer_time_s=1e-4, max_batch=B, seed=4, routing_bias=1e4,
                record_routing=True, timing=True)
hin, hout = [], []
for t in range(4):
    h = synthetic_hidden(cfg, 4, t, B, dev)
    hin.append(h.cpu().numpy())
    eng.step(h)
    torch.cuda.synchronize()
    hout.append(h.cpu().numpy())
log, xs = eng.routing_log(), eng.routing_x()
w = N.ModelWeights(L=2, M=cfg.num_experts, d=2048, ff=1408, dtype="bf16", seed=4,
                   shared_ff=cfg.shared_ff, shared_gate=cfg.shared_gate, cache=True)
errs = R.router_row_errors(log, xs, w, 2)
tag = f"{shape} B={B} FUSE={os.environ.get('EF_FUSE','27')} PDL={os.environ.get('EF_PDL','1')}"
print(tag, "fast_layers", eng.stats()["fast_layers"])
for e in errs:
    print("  row entry %d h %d tok %d rel %.3e" % e)
for t in range(4):
    xe = []
    ref = R.forward_step(hin[t], log, t, w, 2, cfg.top_k, cfg.route_mode, xs=xs, x_errs=xe)
    print("  step", t, "x errs", ["%.2e" % e for _, _, e in xe], "out", "%.2e" % R.rel_err(hout[t], ref))
