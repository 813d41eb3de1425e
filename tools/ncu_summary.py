"""Summarise an ncu launch list of ONE bench step into per-kernel-category shares.

    python tools/ncu_summary.py gpurun_out/r01_launches.csv --round r01 [--config bc100 --dtype bf16]

Input: `ncu --profile-from-start off --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv` over `bench.py --ncu-step`
(tools/ncu_round.sh).  ncu serialises launches and flushes caches before each
one, so the absolute times are cold-cache; the SHARES are what the bench's
event-timed profile must agree with.  Writes profiles/<round>_launches.md and
profiles/<round>_traffic.json (per-category DRAM bytes per launch, read by
bench.py for roofline.traffic).
"""
from __future__ import annotations

import argparse
import csv
import json
import os
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# kernel-name fragment -> category (the names bench.py / dpb_block_profile use)
CATEGORIES = [
    ("Tc3x3WgradHalo", "conv3x3_wgrad"), ("Tc3x3Wgrad", "conv3x3_wgrad"),
    ("Tc3x3DgradHalo", "conv3x3_dgrad"), ("Tc3x3Dgrad", "conv3x3_dgrad"),
    ("Tc3x3FwdHalo", "conv3x3_fwd"), ("Tc3x3Fwd", "conv3x3_fwd"), ("Conv3x3Fwd", "conv3x3_fwd"),
    ("Tc1x1Dgrad", "conv1x1_dgrad"), ("Tc1x1Wgrad", "conv1x1_wgrad"),
    ("Dgrad1x1", "conv1x1_dgrad"), ("Wgrad1x1", "conv1x1_wgrad"),
    ("StemConvGemm", "model: stem"), ("StemWgradGemm", "model: stem"), ("TransWgradGemm", "model: transition GEMMs"),
    ("k_zsplit_reduce", "conv1x1_fwd"), ("k_stem", "model: stem"), ("k_trans_pool", "model: transition fwd"), ("k_gemm", "model: transition GEMMs"),
    ("TransGemm", "model: transition GEMMs"), ("k_pool_bnb_", "model: transition/head BN bwd"),
    ("k_bnb_", "model: transition/head BN bwd"), ("k_head", "model: head"), ("k_loss", "model: head"),
    ("k_running", "model: running stats"), ("k_sgd", "optimizer (SGD)"),
    ("Fwd1x1", "conv1x1_fwd"), ("Tc1x1Fwd", "conv1x1_fwd"),
    ("Conv3x3Dgrad", "conv3x3_dgrad"), ("Conv3x3Wgrad", "conv3x3_wgrad"),
    ("Conv1x1Dgrad", "conv1x1_dgrad"), ("Conv1x1Wgrad", "conv1x1_wgrad"), ("Conv1x1Fwd", "conv1x1_fwd"),
    ("k_finalize", "finalize"), ("k_reduce_w", "reduce_wgrad"),
    ("k_bn_apply_accumulate", "bn_apply_accumulate"), ("k_channel_partials", "channel_stats"),
    ("k_running_update", "running_update"),
    ("k_pretile", "pack"), ("k_nhwc", "pack"), ("k_nchw", "pack"),
]


def category(name: str) -> str:
    for frag, cat in CATEGORIES:
        if frag in name:
            return cat
    return "other (torch copy)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--round", default="r01")
    ap.add_argument("--config", default="bc100")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--what", default="model", choices=["model", "blocks"],
                    help="what the captured step covered (bench.py --ncu-what)")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles"))
    args = ap.parse_args()

    launches = {}  # id -> dict(name, metrics)
    with open(args.csv) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for row in csv.DictReader(lines):
        rec = launches.setdefault(row["ID"], {"name": row["Kernel Name"]})
        v = float(row["Metric Value"].replace(",", ""))
        unit = row["Metric Unit"]
        if row["Metric Name"] == "gpu__time_duration.sum":
            v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)  # -> us
            rec["us"] = v
        else:
            v *= {"byte": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}.get(unit, 1)
            rec[row["Metric Name"]] = v
    cats = defaultdict(lambda: {"launches": 0, "us": 0.0, "dram_bytes": 0.0, "kernels": set()})
    for rec in launches.values():
        c = cats[category(rec["name"])]
        c["launches"] += 1
        c["us"] += rec.get("us", 0.0)
        c["dram_bytes"] += rec.get("dram__bytes_read.sum", 0.0) + rec.get("dram__bytes_write.sum", 0.0)
        c["kernels"].add(rec["name"].split("(")[0].replace("void ", ""))
    total_us = sum(c["us"] for c in cats.values())
    total_launches = sum(c["launches"] for c in cats.values())

    os.makedirs(args.out, exist_ok=True)
    if args.what == "model":
        title = "one whole-network training step"
        src = ("`bash tools/ncu_round.sh` on one B200 (`ncu --profile-from-start off --metrics "
               "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none` over "
               "`python bench.py --ncu-step --ncu-what model --no-cpu-baseline`, which replays ONE CUDA-graph "
               "training step (stem, dense blocks, transitions, head, loss, backward) plus the SGD update between "
               "cudaProfilerStart/Stop).")
    else:
        title = "one dense-blocks training step"
        src = ("one B200 (`ncu --profile-from-start off --metrics "
               "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none` over "
               f"`python bench.py --ncu-step --ncu-what blocks --config {args.config} --no-cpu-baseline "
               "--no-naive`, which replays ONE step of every dense block, forward and backward, between "
               "cudaProfilerStart/Stop).")
    md = [f"# {args.round}: ncu launch list of {title} ({args.config}, {args.dtype}, batch 64)",
          "",
          "Source: " + src + "  ncu serialises launches and flushes caches before each: times are "
          "cold-cache and sum above the graph-timed step; compare SHARES with bench.py `kernels`.",
          "",
          f"Launches in the step: {total_launches}; serialised kernel time {total_us / 1e3:.3f} ms.",
          "",
          "| category | launches | total ms | share | mean us/launch | DRAM MB/launch | kernels |",
          "|---|---:|---:|---:|---:|---:|---|"]
    traffic = {}
    for name, c in sorted(cats.items(), key=lambda kv: -kv[1]["us"]):
        per = c["dram_bytes"] / max(c["launches"], 1)
        traffic[name] = {"launches": c["launches"], "dram_bytes_per_launch": per,
                         "us_per_launch": c["us"] / max(c["launches"], 1), "share": c["us"] / total_us}
        md.append(f"| {name} | {c['launches']} | {c['us'] / 1e3:.3f} | {100 * c['us'] / total_us:.1f}% | "
                  f"{c['us'] / max(c['launches'], 1):.2f} | {per / 1e6:.3f} | "
                  f"{', '.join(sorted(c['kernels']))} |")
    open(os.path.join(args.out, f"{args.round}_launches.md"), "w").write("\n".join(md) + "\n")
    json.dump({"config": args.config, "dtype": args.dtype, "batch": 64, "source": os.path.basename(args.csv),
               "categories": traffic},
              open(os.path.join(args.out, f"{args.round}_traffic.json"), "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
