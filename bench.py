"""Benchmark: decode tokens/s and expert-stall % of step at a fixed HBM
expert-cache budget (BASELINE.json metric) on the Mixtral-8x7B shape,
batch-1 decode, cache budget 40 % of experts (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0.  `value` is device-timed throughput with each
step's input already in HBM; `e2e` is the same through MoEEngine.step_host()
with the input read from and the output written to pinned host memory inside
the timed region.  `roofline` is the routed expert FFN (the dominant kernel
pair) against the measured HBM copy peak; `h2d_roofline` the expert swap-ins
against the measured host-link peak.  `cpu_baseline` is the CPU decode port
(oracle/cpu_port.py: the reference scheduler restatement + the layer
arithmetic on every host core) over a bounded sample of full decode steps.
`routing_grid` separates the cache-aware routing bias from prefetching:
{reactive, adaptive} x bias {0, 1, 4, 1e4} + static at 1e4 on the same
engine and inputs, with routing fidelity against unbiased routing.

`--impl reference` runs the CPU decode port alone (no product library is
loaded in that process) on the same config, policy, bias and inputs.
"""

from __future__ import annotations

import argparse
import importlib.util
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tokens/s and expert-stall % of step at fixed HBM expert-cache budget"
UNIT = "tokens/s"
# logical-clock parameters of the scheduler in the CPU arm (no GPU to measure
# them on): the GPU arm's measured host-link rate and layer time at C2 (round 1)
REF_LINK_BW = 55_000_000_000
REF_LAYER_NS = 130_000


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=24)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mixtral-8x7b")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--budget-frac", type=float, default=0.4)
    ap.add_argument("--strategy", default="adaptive")
    ap.add_argument("--predictor", default="pregate")
    ap.add_argument("--bias", type=float, default=1e4,
                    help="cache-aware routing logit bias (headline: residency-first)")
    ap.add_argument("--rho", type=float, default=0.8,
                    help="temporal correlation of successive decode inputs (AR(1))")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-grid", action="store_true", help="skip the routing grid")
    ap.add_argument("--grid-steps", type=int, default=6)
    ap.add_argument("--cpu-steps", type=int, default=2, help="timed CPU-port steps (cpu_baseline)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--no-peer-tier", action="store_true",
                    help="expert parallelism without home copies in the next GPU's HBM")
    return ap.parse_args()


def load_configs():
    """paper_2510_26730_b200/configs.py loaded on its own: no package import,
    so the reference arm never maps libexpertflow.so."""
    path = os.path.join(ROOT, "paper_2510_26730_b200", "configs.py")
    spec = importlib.util.spec_from_file_location("ef_configs_standalone", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod  # dataclasses look their module up
    spec.loader.exec_module(mod)
    return mod.PRESETS


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def budget_of(cfg, frac):
    return max(cfg.top_k, int(round(frac * cfg.total_experts)))


def maybe_launch_ranks(args):
    """`bench.py --gpus N` outside torchrun launches N ranks itself."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(29500 + os.getpid() % 1000), os.path.abspath(__file__),
           *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


# --------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.rows, self.proc, self.index = [], None, index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows if len(r) >= 7
                          for n, v in zip(names, r[3:7]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# --------------------------------------------------------------------- CPU path
def host_inputs(cfg, args, B, n, rank=0):
    """The decode inputs of both arms: AR(1) in time, unit variance, fp32
    (the same counter generator as runtime.synthetic_hidden)."""
    from oracle import numerics as N
    xs = [N.input_hidden(args.seed + 1000 * rank, 0, B, cfg.d_model)]
    for t in range(1, n):
        eps = N.input_hidden(args.seed + 1000 * rank, t, B, cfg.d_model)
        xs.append((args.rho * xs[-1] + math.sqrt(1 - args.rho ** 2) * eps).astype("float32"))
    return xs


def make_port(cfg, args, bias, budget):
    from oracle.cpu_port import CpuDecodePort
    from oracle.sim import Policy
    pol = Policy(f"{args.strategy}_{args.predictor}", args.strategy,
                 predictor=args.predictor if args.strategy != "static" else "none",
                 cache_aware_routing=True)
    return CpuDecodePort(L=cfg.num_layers, M=cfg.num_experts, k=cfg.top_k, d=cfg.d_model,
                         ff=cfg.d_ff, dtype=cfg.dtype, route_mode=cfg.route_mode,
                         shared_ff=cfg.shared_ff, shared_gate=cfg.shared_gate, seed=args.seed,
                         budget_experts=budget, policy=pol, link_bw=REF_LINK_BW,
                         layer_ns=REF_LAYER_NS, bias=bias)


def time_port(port, inputs, warm, steps):
    """tokens/s of full decode steps on the CPU port (expert generation on
    first touch excluded), and the reference scheduler's share."""
    for t in range(warm):
        port.step(inputs[t])
    c0, s0, n0, g0 = port.compute_s, port.sched_s, port.layers_run, port.gen_s
    b0 = port.expert_bytes
    for t in range(warm, warm + steps):
        port.step(inputs[t])
    comp, sched = port.compute_s - c0, port.sched_s - s0
    layers = port.layers_run - n0
    B = inputs[0].shape[0]
    sec = comp + sched
    return {"tokens_per_s": B * steps / sec, "s_per_step": sec / steps,
            "scheduler_us_per_layer": 1e6 * sched / layers,
            "arithmetic_ms_per_step": 1e3 * comp / steps,
            "expert_GBps": (port.expert_bytes - b0) / comp / 1e9 if comp > 0 else None,
            "expert_generation_s_excluded": port.gen_s - g0,
            "hit_rate": _rate(port.st.cache.hits, port.st.cache.misses),
            "threads": port.threads}


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return {i.get("internal_api", "?"): i.get("num_threads") for i in threadpool_info()}
    except Exception:
        return None


def run_reference(args, cfg, bias):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    budget = budget_of(cfg, args.budget_frac)
    port = make_port(cfg, args, bias, budget)
    inputs = host_inputs(cfg, args, args.batch, args.warmup + args.steps)
    r = time_port(port, inputs, args.warmup, args.steps)
    value = r["tokens_per_s"]
    desc = (f"{args.steps} full {cfg.num_layers}-layer B={args.batch} {cfg.name} decode steps "
            f"after {args.warmup} warm-up steps: the reference scheduler (OracleStepper, the "
            f"restatement of moesim _Sim, 1 core) + router / top-k / SwiGLU experts on bf16 "
            f"weights / combine on {r['threads']} OpenMP threads (oracle/cport.c); expert "
            f"weights generated into host RAM on first touch, generation time excluded")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * args.batch / value, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
            "config": {"workload": f"{cfg.name} shape, bf16 random-init, batch-{args.batch} "
                                   f"decode, cache budget {budget}/{cfg.total_experts} experts, "
                                   f"CPU decode port", "model": cfg.name,
                       "policy": port.st.policy.name, "routing_bias": bias, "rho": args.rho},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["threads"], "kind": "port",
                             "sample": desc, "blas_threads": blas_threads(),
                             "host_cores": os.cpu_count()},
            "reference_scheduler_us_per_layer": r["scheduler_us_per_layer"],
            "cpu_detail": r,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- GPU arm
def measure_h2d(torch, nbytes):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    bw = 3 * nbytes / (s.elapsed_time(e) / 1e3)
    del h, d
    return int(bw)


def measure_layer_time(torch, cfg, B):
    """Device time of one layer's routed expert FFN at the roofline-bound
    kernel speed (top_k experts, B rows) + router/combine, on a scratch slab."""
    import ctypes as C
    from paper_2510_26730_b200 import _lib as L
    k = cfg.top_k
    n_act = min(cfg.num_experts, B * k)
    slab = torch.empty(n_act, cfg.expert_bytes, dtype=torch.uint8, device="cuda")
    x = torch.randn(B, cfg.d_model, device="cuda")
    perm = torch.arange(B * k, dtype=torch.int32, device="cuda")
    act = torch.empty(B * k, cfg.d_ff * cfg.elem_bytes, dtype=torch.uint8, device="cuda")
    y = torch.empty(B * k, cfg.d_model, device="cuda")
    slab.view(torch.bfloat16 if cfg.dtype == "bf16" else torch.float32).normal_(0, 0.01)
    rows = [B * k // n_act] * n_act
    rows[0] += B * k - sum(rows)
    offs = [sum(rows[:i]) for i in range(n_act)]
    a_slot, a_off, a_rows = L.i32arr(range(n_act)), L.i32arr(offs), L.i32arr(rows)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def go():
        L.check(L.lib.ef_expert_ffn_decode(
            st, C.c_void_p(x.data_ptr()), C.c_void_p(perm.data_ptr()), k,
            C.c_void_p(slab.data_ptr()), cfg.expert_bytes, L.as_ptr(a_slot, C.c_int32),
            L.as_ptr(a_off, C.c_int32), L.as_ptr(a_rows, C.c_int32), n_act, cfg.d_model,
            cfg.d_ff, 1 if cfg.dtype == "bf16" else 0, C.c_void_p(act.data_ptr()),
            C.c_void_p(y.data_ptr())))
    for _ in range(3):
        go()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        go()
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 10 / 1e3
    del slab
    return t + 15e-6  # + router, route/permute, combine launches


def _rate(h, m):
    return h / (h + m) if h + m else 0.0


def grid_cell(eng, ef, torch, args, cfg, strategy, bias, inputs, W, n):
    """One {policy, bias} cell on the reused engine (reset: cold cache)."""
    import numpy as np
    pol = ef.PolicyConfig(f"{strategy}", strategy,
                          predictor="pregate" if strategy != "static" else "none",
                          cache_aware_routing=strategy != "reactive")
    eng.reset(pol, bias)
    for t in range(W):
        eng.step(inputs[t].clone())
    torch.cuda.synchronize()
    st0, m0 = eng.stats(), eng.metrics()
    eng.set_record_routing(2)
    outs = []
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = 0.0
    for t in range(W, W + n):
        h = inputs[t].clone()
        s.record()
        eng.step(h)
        e.record()
        torch.cuda.synchronize()
        ms += s.elapsed_time(e)
        outs.append(h.cpu().numpy())
    eng.set_record_routing(0)
    st1, m1 = eng.stats(), eng.metrics()
    # routing agreement with the unbiased top-k of the same fp32 logits
    k = cfg.top_k
    agree = tot = 0
    for lg, sel, _mask in eng.routing_log():
        unb = np.argsort(-lg[0], axis=1, kind="stable")[:, :k]
        for a, b in zip(sel, unb):
            agree += len(set(a.tolist()) & set(b.tolist()))
            tot += k
    adm = st1["prefetch_admitted"] - st0["prefetch_admitted"]
    used = st1["prefetch_used"] - st0["prefetch_used"]
    wasted = st1["prefetch_wasted"] - st0["prefetch_wasted"]
    sel_n = m1.miss_stats.n_selected - m0.miss_stats.n_selected
    tot_n = m1.miss_stats.n_total - m0.miss_stats.n_total
    return {"policy": strategy, "bias": bias, "tokens_per_s": args.batch * n / (ms / 1e3),
            "expert_stall_pct": 100.0 * (st1["stall_ms"] - st0["stall_ms"]) / ms,
            "copies_per_step": (st1["copies"] - st0["copies"]) / n,
            "hit_rate": _rate(m1.hits - m0.hits, m1.misses - m0.misses),
            "prediction_miss_rate": (1.0 - sel_n / tot_n) if tot_n else None,
            "prefetch_admitted": adm, "prefetch_used": used, "prefetch_wasted": wasted,
            "prefetch_precision": used / (used + wasted) if used + wasted else None,
            "topk_agreement_vs_unbiased": agree / tot if tot else None,
            "_outs": outs}


def routing_grid(eng, ef, torch, args, cfg, inputs, W):
    import numpy as np
    cells = [(s, b) for s in ("reactive", "adaptive") for b in (0.0, 1.0, 4.0, 1e4)]
    cells.append(("static", 1e4))
    res = [grid_cell(eng, ef, torch, args, cfg, s, b, inputs, W, args.grid_steps)
           for s, b in cells]
    ref = {r["policy"]: r["_outs"] for r in res if r["bias"] == 0.0}
    unb = ref.get("adaptive")
    for r in res:
        base = ref.get(r["policy"], unb)
        errs = [float(np.linalg.norm(a - b) / np.linalg.norm(b)) for a, b in zip(r["_outs"], base)]
        r["output_rel_divergence_vs_unbiased"] = statistics.mean(errs)
        del r["_outs"]
    return res


def run_ours(args, cfg, bias):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2510_26730_b200 as ef
    from paper_2510_26730_b200.runtime import MoEEngine, synthetic_hidden

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    B = args.batch
    budget = budget_of(cfg, args.budget_frac)
    link_bw = measure_h2d(torch, cfg.expert_bytes)
    layer_s = measure_layer_time(torch, cfg, B)
    policy = ef.PolicyConfig(f"{args.strategy}_{args.predictor}", args.strategy,
                             predictor=args.predictor if args.strategy != "static" else "none",
                             cache_aware_routing=True)
    t_init = time.perf_counter()
    if world > 1:
        # expert parallelism: rank r owns experts [r*M/G, (r+1)*M/G)
        # of every layer, with a 40 % cache budget of its shard; each rank decodes
        # its own B tokens (weak scaling), routing blocks all-gathered and expert
        # outputs returned by all-to-all over NCCL on the engine's stream.  Home
        # copies of the shard's experts sit in the next GPU's HBM (peer tier):
        # misses are NVLink copies before they would be host copies.  The
        # residency bias needs every shard's residency before routing and is
        # not exchanged this round: EP runs unbiased.
        from paper_2510_26730_b200 import ep as EP
        ms = cfg.num_experts // world
        budget = EP.shard_budget(budget, cfg.num_experts, world, cfg.num_layers)
        bias = 0.0
        kw = dict(budget_experts=budget, policy=policy, link_bw=link_bw, layer_time_s=layer_s,
                  max_batch=B, seed=args.seed, routing_bias=0.0, timing=True, device=local,
                  ep_rank=rank, ep_world=world, ep_nccl_id=EP.nccl_group_id())
        if not args.no_peer_tier:
            kw.update(peer_device=(local + 1) % world, peer_pool_experts=cfg.num_layers * ms)
        eng = MoEEngine(cfg, **kw)
        dist.barrier()
    else:
        kw = dict(budget_experts=budget, policy=policy, link_bw=link_bw, layer_time_s=layer_s,
                  max_batch=B, seed=args.seed, routing_bias=bias, timing=True, device=local)
        eng = MoEEngine(cfg, **kw)
    init_s = time.perf_counter() - t_init

    # decode inputs: AR(1) in time with correlation rho, unit variance, in HBM
    K, W = args.steps, args.warmup
    n_in = W + 2 * K  # timed pass W..W+K, end-to-end pass on fresh inputs after it
    xs = [synthetic_hidden(cfg, args.seed + 1000 * rank, 0, B, dev)]
    for t in range(1, n_in):
        eps = synthetic_hidden(cfg, args.seed + 1000 * rank, t, B, dev)
        xs.append(args.rho * xs[-1] + math.sqrt(1 - args.rho ** 2) * eps)
    inputs = [x.clone() for x in xs]
    stream = torch.cuda.current_stream(dev)

    for t in range(W):
        eng.step(inputs[t])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    st0 = eng.stats()
    m0 = eng.metrics()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        time.sleep(0.5)  # let the sampler take its first readings
        s.record(stream)
        for t in range(W, W + K):
            eng.step(inputs[t])
        e.record(stream)
        torch.cuda.synchronize()
    dev_ms = s.elapsed_time(e)
    st1 = eng.stats()
    m1 = eng.metrics()
    if world > 1:
        tt = torch.tensor([dev_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dev_ms = float(tt.item())
    value = world * B * K / (dev_ms / 1e3)

    # expert-stall % of step: physical (device wait on copy events) and logical
    stall_ms = st1["stall_ms"] - st0["stall_ms"]
    stall_pct = 100.0 * stall_ms / dev_ms
    log_wait = m1.waiting_ns - m0.waiting_ns
    log_total = m1.total_time_ns - m0.total_time_ns
    ffn_ms = st1["ffn_ms"] - st0["ffn_ms"]
    ffn_bytes = st1["ffn_bytes"] - st0["ffn_bytes"]
    ffn_pairs = (st1["ffn_launches"] - st0["ffn_launches"]) / 2
    launches = int(st1["kernel_launches"] - st0["kernel_launches"])
    hbm_peak, peak_kind = peaks()
    achieved = ffn_bytes / (ffn_ms / 1e3) / 1e9 if ffn_ms > 0 else 0.0
    h2d_GBps = (st1["copy_bytes"] - st0["copy_bytes"]) / (dev_ms / 1e3) / 1e9

    # ---- end to end through the public API with host buffers: step_host()
    # reads each step's pinned input and writes the pinned output over PCIe
    host_in = [x.cpu().pin_memory() for x in xs]
    host_out = torch.empty(B, cfg.d_model, dtype=torch.float32).pin_memory()
    torch.cuda.synchronize()
    se, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    se.record(stream)
    for t in range(K):
        eng.step_host(host_in[W + K + t], host_out)
    ee.record(stream)
    torch.cuda.synchronize()
    e2e_ms = se.elapsed_time(ee)
    # the same with the user's own cudaMemcpy of input/output around step()
    # (queues behind an in-flight expert swap-in on the copy engine)
    buf = torch.empty(B, cfg.d_model, dtype=torch.float32, device=dev)
    host_out2 = torch.empty_like(host_out).pin_memory()
    torch.cuda.synchronize()
    se.record(stream)
    for t in range(K):
        buf.copy_(host_in[W + t], non_blocking=True)
        eng.step(buf)
        host_out2.copy_(buf, non_blocking=True)
    ee.record(stream)
    torch.cuda.synchronize()
    memcpy_ms = se.elapsed_time(ee)
    if world > 1:
        tt = torch.tensor([e2e_ms, memcpy_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms, memcpy_ms = (float(v) for v in tt.tolist())
    e2e = world * B * K / (e2e_ms / 1e3)
    finite = bool(torch.isfinite(host_out).all())

    # ---- the reference scheduler path on this run's routing (SURVEY §8d
    # D5(i)): 4 more steps recorded, replayed through OracleStepper on 1 core
    sched = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sched = replay_scheduler(eng, ef, torch, cfg, args, inputs, budget, link_bw, layer_s,
                                 policy, bias)

    grid = None
    if rank == 0 and world == 1 and not args.no_grid:
        grid = routing_grid(eng, ef, torch, args, cfg, inputs, min(W, 4))
    phys_slots = int(st1["phys_slots"])
    eng.close()
    del eng
    import gc
    gc.collect()
    torch.cuda.synchronize()

    traffic = ncu_traffic(cfg, B)
    if rank == 0:
        cpu, cpu_desc = None, "skipped (--no-cpu)"
        if not args.no_cpu:
            port = make_port(cfg, args, bias, budget)
            hin = host_inputs(cfg, args, B, W + 1 + args.cpu_steps)
            cpu = time_port(port, hin[W:], 1, args.cpu_steps)
            cpu_desc = (f"{args.cpu_steps} full {cfg.num_layers}-layer B={B} decode steps of "
                        f"the same workload after 1 warm-up step: the reference scheduler "
                        f"(OracleStepper, 1 core) + the layer arithmetic on bf16 weights "
                        f"on {cpu['threads']} OpenMP threads (oracle/cport.c); expert "
                        f"generation on first touch excluded")
            del port
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": dev_ms / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": cfg.dtype,
            "data": "synthetic (random-init weights, AR(1) hidden inputs)",
            "config": {"workload": f"{cfg.name} shape, bf16 random-init, batch-{B} decode per "
                                   f"GPU, cache budget {budget}/"
                                   f"{cfg.total_experts // world} experts per GPU "
                                   f"({100 * budget * world / cfg.total_experts:.0f}%) on "
                                   f"{world}xB200",
                       "model": cfg.name, "global_batch": B * world, "seq_len": 1,
                       "parallelism": f"ep{world} (expert parallel, NCCL all-gather + "
                                      f"all-to-all per layer)" if world > 1 else "single GPU",
                       "policy": policy.name, "routing_bias": bias, "rho": args.rho,
                       "budget_experts": budget, "physical_slots": phys_slots,
                       "link_bw_measured_GBps": link_bw / 1e9,
                       "layer_time_calibrated_us": layer_s * 1e6,
                       "l2": "expert weights streamed per step exceed the 126 MB L2",
                       "engine_init_s": round(init_s, 1)},
            "expert_stall_pct": stall_pct,
            "logical_stall_pct": 100.0 * log_wait / log_total if log_total else 0.0,
            "hit_rate": _rate(m1.hits - m0.hits, m1.misses - m0.misses),
            "copies_per_step": (st1["copies"] - st0["copies"]) / K,
            "h2d_GBps": h2d_GBps,
            "bandwidth_estimate_GBps": {"logical": m1.bandwidth_estimate / 1e9,
                                        "physical": st1["bw_physical_Bps"] / 1e9,
                                        "physical_transfers": int(st1["bw_physical_transfers"]),
                                        "what": "EWMA (alpha 0.25) of the scheduler's logical "
                                                "transfers / of the copy engine's measured "
                                                "expert copies (copy-stream events)"},
            "host_decision_us_per_layer": 1e3 * (st1["host_decision_ms"] - st0["host_decision_ms"])
            / (K * cfg.num_layers),
            "gate_wait_us_per_layer": 1e3 * (st1["gate_wait_ms"] - st0["gate_wait_ms"])
            / (K * cfg.num_layers),
            "ffn_us_per_layer": 1e3 * ffn_ms / (K * cfg.num_layers),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak,
                         "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
                         "kernel": ("decode_layer_kernel (persistent layer: routed + shared "
                                    "expert gate/up and down units on mma.sync; window = first "
                                    "FFN unit -> last down unit)"
                                    if st1.get("layer_kernel_steps", 0) > st0.get("layer_kernel_steps", 0)
                                    else "ef_expert_ffn_decode (gate/up+SiLU GEMV, down GEMV)"),
                         "bytes_per_launch": ffn_bytes / max(ffn_pairs, 1),
                         "timing": "on-device globaltimer stamps per layer (first FFN CTA past "
                                   "its ready check -> last down-projection CTA), summed over the "
                                   "timed steps; CUDA events around the launch would include the "
                                   "host-decision wait folded into the gate/up kernel",
                         "traffic_source": traffic["source"] if traffic else
                         f"no ncu capture committed for {cfg.name} B={B}",
                         "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs"},
            "h2d_roofline": {"bound": "host link", "achieved": h2d_GBps,
                             "peak": link_bw / 1e9, "unit": "GB/s",
                             "frac": h2d_GBps / (link_bw / 1e9),
                             "what": "expert swap-ins (pinned host store -> HBM slab) over the "
                                     "timed steps; peak = pinned H2D copy measured at start"},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": B * cfg.d_model * 4,
                    "d2h_bytes_per_step": B * cfg.d_model * 4, "output_finite": finite,
                    "api": "MoEEngine.step_host(pinned_in, pinned_out) -> ef_engine_step_host",
                    "via_user_memcpy": world * B * K / (memcpy_ms / 1e3)},
            "gpu_launches": launches,
            "cpu_baseline": {"value": cpu["tokens_per_s"] if cpu else None, "unit": UNIT,
                             "cores": cpu["threads"] if cpu else None, "kind": "port",
                             "sample": cpu_desc, "blas_threads": blas_threads(),
                             "host_cores": os.cpu_count(), "detail": cpu},
            "reference_scheduler": sched,
            "clocks": clocks.summary(),
        }
        if grid:
            line["routing_grid"] = grid
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def replay_scheduler(eng, ef, torch, cfg, args, inputs, budget, link_bw, layer_s, policy, bias):
    """Record 4 steps of this engine's routing and time the reference
    scheduler restatement (OracleStepper) deciding them on one core."""
    from oracle import replay as R
    from oracle.sim import Policy
    n = 4
    eng.reset(policy, bias)
    eng.set_record_routing(2)
    for t in range(n):
        eng.step(inputs[t].clone())
    torch.cuda.synchronize()
    eng.set_record_routing(0)
    log = eng.routing_log()
    st = eng.stats()
    pol = Policy(policy.name, policy.strategy, policy.predictor, policy.interval,
                 policy.cache_aware_routing, policy.cold_start, policy.cum_threshold,
                 policy.stall_threshold, policy.overfetch_threshold, policy.min_step,
                 policy.max_step, policy.recent_window, policy.noise.decay_rate,
                 policy.prediction_cache_capacity)
    t0 = time.perf_counter()
    orc, mask_bad, sel_bad = R.replay(
        log, L=cfg.num_layers, M=cfg.num_experts, k=cfg.top_k, expert_bytes=cfg.expert_bytes,
        link_bw=link_bw, budget_experts=budget, layer_ns=round(layer_s * 1e9), policy=pol,
        tokens_per_step=[(-(t + 1),) for t in range(n)], bias=bias, emit_events=False)
    sec = time.perf_counter() - t0
    m = eng.metrics()
    same = (orc.metrics.hits, orc.metrics.misses, orc.metrics.admissions,
            orc.metrics.evictions) == (m.hits, m.misses, m.admissions, m.evictions)
    return {"us_per_layer": 1e6 * sec / (n * cfg.num_layers), "cores": 1,
            "what": "OracleStepper (restatement of moesim _Sim, engine.py:543-690) deciding "
                    f"{n} recorded steps of this engine's routing, single-threaded Python",
            "decisions_identical": bool(same and not mask_bad and not sel_bad)}


def ncu_traffic(cfg, B):
    """DRAM bytes per routed-FFN launch of this config from a committed ncu
    capture (profiles/ncu_traffic.json, keyed by config and batch)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(f"{cfg.name}/B{B}")


def main():
    args = parse()
    maybe_launch_ranks(args)
    if args.impl == "reference":
        run_reference(args, load_configs()[args.config], args.bias)
    else:
        from paper_2510_26730_b200.runtime import PRESETS
        run_ours(args, PRESETS[args.config], args.bias)


if __name__ == "__main__":
    main()
