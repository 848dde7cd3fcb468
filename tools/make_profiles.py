"""Turn the GPU-side captures in gpurun_out/ into the tracked summaries under
profiles/ (per round).  Usage:

    python tools/make_profiles.py --round r01 \
        --launches gpurun_out/launches20.csv --ffn gpurun_out/prof20_ffn.ncu-rep \
        --router gpurun_out/prof20_router.ncu-rep --gemm gpurun_out/prof_gemm.ncu-rep

Writes profiles/<round>_decode_launches.csv (the ncu launch list of the
decode steps, fill/init kernels dropped), profiles/<round>_decode_launch_share.md
(per-kernel share of a decode step), profiles/<round>_ncu_<name>.txt (key
metrics of each --set full capture) and profiles/ncu_traffic.json (DRAM bytes
per launch of the decode FFN kernels, read by bench.py for roofline.traffic).
"""
import argparse
import csv
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes_read.sum.per_second", "DRAM read rate"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_static", "static smem/block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active %"),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc pipe inst %"),
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def to_bytes(v, unit):
    v = float(v)
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def summarise(rep, name, rnd):
    hdr, units, rows = raw_rows(rep)
    lines = [f"# ncu --set full summary: {name}", f"# source: {os.path.basename(rep)} "
             "(captured with --clock-control none --import-source on; cold cache, "
             "kernels serialised by ncu)", ""]
    per_kernel = []
    for r in rows:
        kname = r[hdr.index("Kernel Name")]
        lines.append(f"kernel: {kname}")
        rec = {"kernel": kname}
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                lines.append(f"  {label:28s} {r[i]} {units[i]}")
                rec[key] = (r[i], units[i])
        lines.append("")
        per_kernel.append(rec)
    path = os.path.join(PROF, f"{rnd}_ncu_{name}.txt")
    with open(path, "w") as f:
        f.write("\n".join(lines))
    return per_kernel


def launch_list(path, rnd, name="decode", command=None):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.reader(lines))
    hdr, data = rows[0], rows[1:]
    ki, gi, bi, vi = (hdr.index("Kernel Name"), hdr.index("Grid Size"), hdr.index("Block Size"),
                      hdr.index("Metric Value"))
    keep = [r for r in data if "fill_uniform" not in r[ki]]
    out = os.path.join(PROF, f"{rnd}_{name}_launches.csv")
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "grid", "block", "duration_ns"])
        for r in keep:
            w.writerow([r[0], r[ki].split("(")[0], r[gi], r[bi], r[vi]])
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in keep:
        k = r[ki].split("(")[0]
        tot[k] += float(r[vi])
        cnt[k] += 1
    all_ns = sum(tot.values())
    default_cmd = (
        "Command: `EF_PIPE_DEBUG=1 EF_FUSE=1 ncu --metrics gpu__time_duration.sum "
        "--clock-control none python tools/profile_decode.py --layers 32 --steps 3 "
        "--policy adaptive --budget-frac 0.4 --bias 10000` (Mixtral-8x7B shape, 32 layers, "
        "B=1, the bench's policy and budget).  ncu makes every launch synchronous, so the "
        "run-ahead pipeline (whose fused gate waits on the host) cannot run under it: "
        "EF_PIPE_DEBUG=1 decides each layer before enqueueing its FFN and EF_FUSE=1 keeps "
        "the gate in its own kernel.  The default pipeline has no gate_kernel launch, no "
        "combine_kernel launch (folded into the next router) and no host wait.")
    md = [f"# {rnd}: kernel share of the decode steps (ncu launch list)", "",
          command or default_cmd, "",
          "Per-launch times are cold-cache and serialised: compare shares, not absolutes.", "",
          "| kernel | launches | total us | mean us | share |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        md.append(f"| `{k}` | {cnt[k]} | {v / 1e3:.1f} | {v / cnt[k] / 1e3:.1f} | "
                  f"{v / all_ns:.1%} |")
    with open(os.path.join(PROF, f"{rnd}_{name}_launch_share.md"), "w") as f:
        f.write("\n".join(md) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--launches")
    ap.add_argument("--launch-name", default="decode")
    ap.add_argument("--launch-command")
    ap.add_argument("--ffn")
    ap.add_argument("--router")
    ap.add_argument("--gemm")
    ap.add_argument("--up", help="separate capture of the gate/up GEMV (merged into decode_ffn)")
    ap.add_argument("--down", help="separate capture of the down GEMV (merged into decode_ffn)")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        launch_list(a.launches, a.round, a.launch_name, a.launch_command)
    traffic = {}
    if a.up and a.down:
        ku = summarise(a.up, "decode_ffn_up", a.round)
        kd = summarise(a.down, "decode_ffn_down", a.round)
        a.ffn = None
        ks = ku + kd
        src = f"{os.path.basename(a.up)} + {os.path.basename(a.down)}"
    elif a.ffn:
        ks = summarise(a.ffn, "decode_ffn", a.round)
        src = os.path.basename(a.ffn)
    else:
        ks = []
    if ks:
        up = [k for k in ks if "XGather" in k["kernel"]]
        dn = [k for k in ks if "XAct" in k["kernel"]]
        if up and dn:
            def dram(k):
                return sum(to_bytes(*k[m]) for m in ("dram__bytes_read.sum",
                                                      "dram__bytes_write.sum"))
            traffic = {
                "kernel": "ef_expert_ffn_decode (gate/up GEMV + down GEMV), Mixtral-8x7B, "
                          "B=1, 2 experts",
                "dram_bytes_up": dram(up[0]), "dram_bytes_down": dram(dn[0]),
                "dram_bytes_per_launch": dram(up[0]) + dram(dn[0]),
                "algorithmic_bytes_per_launch": 2 * 3 * 4096 * 14336 * 2,
                "source": src, "round": a.round,
            }
            with open(os.path.join(PROF, "ncu_traffic.json"), "w") as f:
                json.dump(traffic, f, indent=1)
    if a.router:
        summarise(a.router, "router_route", a.round)
    if a.gemm:
        summarise(a.gemm, "prefill_grouped_gemm", a.round)
    print("wrote", sorted(os.listdir(PROF)))


if __name__ == "__main__":
    main()
