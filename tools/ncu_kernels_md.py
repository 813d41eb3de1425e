"""profiles/<round>_kernels.md from the --set full captures of tools/ncu_round.sh.

r01: the block-1, layer-15 launches of BC-100; r02: DenseNet-264-k32 block 3
(and block 1 for the 3x3 forward, the stem dW).  Algorithmic
bytes per launch follow DESIGN.md §4 (the LaunchScope formulas); achieved
GB/s = algorithmic bytes / ncu duration (cold cache, serialised: a lower
bound on the in-graph rate)."""
import csv
import json
import os
import subprocess
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def block_kernels(M, c, bk, k):
    """capture name, role, algorithmic bytes (fp32 storage), FLOPs of one launch."""
    return [
        ("Fwd1x1", f"conv1x1_fwd (v2 TMA engine), c={c}", M * (4 * c + 4 * bk), 2 * M * c * bk),
        ("Tc3x3FwdTaps", "conv3x3_fwd (halo, all-taps GEMM)", M * (4 * bk + 4 * k), 2 * M * 9 * bk * k),
        ("Tc3x3FwdHalo", "conv3x3_fwd (halo, per-tap)", M * (4 * bk + 4 * k), 2 * M * 9 * bk * k),
        ("Tc3x3DgradHalo", "conv3x3_dgrad (halo)", M * (4 * k + 8 * bk), 2 * M * 9 * bk * k),
        ("Dgrad1x1", f"conv1x1_dgrad (v2, epilogue ring + TMA store), c={c}", M * (8 * bk + 8 * c),
         2 * M * c * bk),
        ("Wgrad1x1", f"conv1x1_wgrad (v2, split-K in TMEM), c={c}", M * (8 * bk + 4 * c), 2 * M * c * bk),
        ("Tc3x3WgradHalo", "conv3x3_wgrad (halo)", M * (4 * k + 4 * bk), 2 * M * 9 * bk * k),
        ("k_bn_apply_accumulate4", f"bn_apply_accumulate (BN_a bwd + concat acc), c={c}", M * 16 * c, 0),
    ]


if R == "r01":  # BC-100, block 1, layer 15
    TITLE = "BC-100, block 1, layer 15"
    SHAPE = "M = 65,536 pixels, c = 204, bk = 48, k = 12"
    KERNELS = [kk for kk in block_kernels(65536, 204, 48, 12) if kk[0] != "Tc3x3FwdHalo"]
else:  # r02: DenseNet-264-k32 at batch 64 (the SPECS of tools/ncu_round.sh in round 2)
    TITLE = "DenseNet-264-k32, batch 64: block 3 (14x14) layers 30 / 33; block 1 (56x56) layer 3 for the 3x3 forward"
    SHAPE = ("block 3: M = 12,544, bk = 128, k = 32, c = 1,216 (forward, layer 30) / 1,312 (backward, layer 33); "
             "block 1: M = 200,704; the ImageNet stem dW: 802,816 pixels x 64 x 147")
    b3f = {kk[0]: kk for kk in block_kernels(12544, 1216, 128, 32)}
    b3b = {kk[0]: kk for kk in block_kernels(12544, 1312, 128, 32)}
    b1 = {kk[0]: kk for kk in block_kernels(200704, 64 + 3 * 32, 128, 32)}
    M1 = 802816  # stem conv output pixels (64 x 112 x 112)
    KERNELS = [b3f["Fwd1x1"], b1["Tc3x3FwdHalo"], b3b["Tc3x3DgradHalo"], b3b["Dgrad1x1"], b3b["Wgrad1x1"],
               b3b["Tc3x3WgradHalo"], b3b["k_bn_apply_accumulate4"],
               ("StemConvGemm", "ImageNet stem conv 7x7/2 (tcgen05, space-to-depth operands, fp16x3)",
                M1 * 64 * 4 + 64 * 3 * 224 * 224 * 4, 2 * M1 * 64 * 147),
               ("StemWgradGemm", "ImageNet stem dW (tcgen05, BN-backward apply in the producer)",
                M1 * (4 * 64 + 4 * 64) + 64 * 3 * 224 * 224 * 4, 2 * M1 * 64 * 147)]
KEYS = {"dur": "gpu__time_duration.sum", "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum",
        "dram": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "tensor": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "warps": "sm__warps_active.avg.pct_of_peak_sustained_active", "regs": "launch__registers_per_thread",
        "l2hit": "lts__t_sector_hit_rate.pct", "grid": "Grid Size", "block": "Block Size"}
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
hbm = float(peaks["hbm_gbs"])


def num(v, unit):
    x = float(v.replace(",", ""))
    scale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
             "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    return x * scale.get(unit, 1)


rows = []
for name, role, abytes, aflops in KERNELS:
    rep = os.path.join(ROOT, "gpurun_out", f"{R}_{name}.ncu-rep")
    if not os.path.exists(rep):
        continue
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    t = list(csv.reader(out.splitlines()))
    hdr, units, r = t[0], t[1], t[2]
    g = {key: (r[hdr.index(m)], units[hdr.index(m)]) for key, m in KEYS.items() if m in hdr}
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                st.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    st.sort(reverse=True)
    dur = num(*g["dur"])
    traffic = num(*g["rd"]) + num(*g["wr"])
    rows.append((role, g["grid"][0], g["block"][0], dur * 1e6, abytes / 1e6, traffic / 1e6,
                 abytes / dur / 1e9, abytes / dur / 1e9 / hbm, float(g["dram"][0]), float(g["tensor"][0]),
                 aflops / dur / 1e12, float(g["warps"][0]), g["regs"][0], float(g["l2hit"][0]),
                 ", ".join(f"{n} {int(v)}" for v, n in st[:3])))

md = [f"# {R}: `ncu --set full` of every conv kernel type and the BN apply ({TITLE})", "",
      "Captured by `bash tools/ncu_round.sh` (one B200; each ncu run follows the same command run "
      f"plainly).  Each row is ONE launch: {SHAPE}, fp32 arena, tensor cores.  ncu times are cold-cache "
      "and serialised; the in-graph step overlaps kernels "
      "(two streams, PDL).  Algorithmic bytes: DESIGN.md §4.  Peak HBM: "
      f"{hbm:.1f} GB/s (MEASURED_PEAKS.json).", "",
      "| kernel | grid x block | us | alg. MB | DRAM MB | alg. GB/s | frac of HBM | DRAM % (ncu) | "
      "tensor pipe % | alg. TFLOP/s | warps active % | regs | L2 hit % | top stalls |",
      "|---|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---|"]
for (role, grid, block, us, amb, dmb, gbs, frac, dram, tensor, tf, warps, regs, l2, stalls) in rows:
    md.append(f"| {role} | {grid} x {block} | {us:.1f} | {amb:.1f} | {dmb:.1f} | {gbs:.0f} | {frac:.3f} | "
              f"{dram:.1f} | {tensor:.2f} | {tf:.2f} | {warps:.1f} | {regs} | {l2:.1f} | {stalls} |")
if R != "r01":
    md += ["", "Reading (DenseNet-264-k32): every dense-block kernel is HBM- or latency-bound (intensity "
           "44 FLOP/B against a ridge of 254).  At 14x14 and batch 64 a layer has 98 pixel tiles: the "
           "persistent 1x1 kernels run one or two tiles per CTA, and their per-SM operand intake (features "
           "+ the streamed W1 image) is the limit (fwd 0.26, dgrad 0.37, wgrad 0.25 of HBM).  The 3x3 halo "
           "kernels run one CTA per SM; the forward's producer warps now build K chunk kb+1 while "
           "two issuer warps drive chunk kb's MMAs (mbarrier hand-off), the dgrad splits its 128 "
           "output columns over two CTAs per tile under two waves.  The BN_a apply + accumulate "
           "streams near HBM speed.  The stem runs on the tensor cores (space-to-depth operands)."]
md += [] if R != "r01" else ["", "Reading: every kernel is HBM/latency-bound (intensity 18-66 FLOP/B against a bf16 ridge of "
       "254 FLOP/B).  So the tensor pipe idles by construction: at the HBM roofline these shapes reach "
       "at most 7-26 % tensor-pipe utilisation.  The gap to the roofline is per-tile latency (the 3x3 halo "
       "kernels: produce, issue and epilogue in sequence at two CTAs per SM) and ramp/tail effects of "
       "short launches (3.5 tiles per SM), not bandwidth."]
open(os.path.join(ROOT, "profiles", f"{R}_kernels.md"), "w").write("\n".join(md) + "\n")
print("\n".join(md))
