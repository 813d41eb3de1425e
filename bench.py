"""Benchmark of the memory-efficient dense-block hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config bc100|cfg1|d121|d264k32|d264k48]

One step = one whole training step of the configuration (BASELINE.json
configs[1] by default: DenseNet-BC-100, k=12, batch 64 per GPU, 3x32x32
input): stem, dense blocks, transitions, head, softmax cross-entropy, forward
+ backward and the momentum-SGD update, on synthetic inputs resident in HBM,
through libdpb.so (bf16 tensor-core GEMMs, fp32 arena and gradients), CUDA-
graph captured.  The dense blocks alone (the hot path) are reported beside it
under "dense_blocks".  ImageNet-shaped configs, whose 7x7/2 stem is not built,
time the dense blocks only.  Prints ONE JSON line on rank 0; see DESIGN.md §5
for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BATCH = 64
METRIC = "DenseNet train images/sec"


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


def block_shapes(config: str, batch: int):
    from paper_1707_06990_b200.model import CONFIGS
    cfg = CONFIGS[config]
    stem_stride = 4 if cfg.in_shape[1] >= 224 else 1   # ImageNet 7x7/2 + maxpool geometry (F4)
    return [(s.n, s.h, s.w, s.c0, s.m, s.k, s.bk) for s in cfg.block_shapes(batch, stem_stride)]


def algorithmic_per_image(shapes, S=2):
    """F = sum_l HW [6 c bk + 54 bk k],  B = sum_l HW (22 c + 16 bk + 6 k)."""
    F = B = 0.0
    for (n, h, w, c0, m, k, bk) in shapes:
        hw = h * w
        for l in range(m):
            c = c0 + l * k
            F += hw * (3 * 2 * c * bk + 3 * 2 * 9 * bk * k)
            B += hw * (22 * c + 16 * bk + 6 * k)
    return F, B


def committed_traffic(kernel: str, config: str, dtype: str):
    """DRAM bytes per launch of `kernel` from the committed ncu launch list of one
    bench step (profiles/r*_traffic.json, tools/ncu_summary.py), or None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")), reverse=True):
        try:
            d = json.load(open(path))
        except (OSError, ValueError):
            continue
        if d.get("config") == config and d.get("dtype") == dtype and kernel in d.get("categories", {}):
            return d["categories"][kernel]["dram_bytes_per_launch"]
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={device_index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        sms.sort()
        return {"sm_mhz": sms[len(sms) // 2] if sms else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms)}


def cpu_runner(config: str):
    """The reference CPU workload matching the GPU arm: its whole training step
    (GraphPlan::step_trace, one image per process) for CIFAR-type networks,
    else one image of every dense block (fwd+bwd)."""
    from oracle import cpu_bench as CB
    from paper_1707_06990_b200.model import CONFIGS
    cfg = CONFIGS[config]
    if cfg.in_shape[1] < 64 and CB.kind() == "reference":
        net = (tuple(cfg.block_sizes), cfg.growth_rate, cfg.compression, cfg.num_classes, cfg.c0,
               tuple(cfg.in_shape))
        return CB.CpuModelRunner(net, batch=1), f"1 image, {config} full training step (GraphPlan::step_trace)"
    return CB.CpuRunner(block_shapes(config, 1)), f"1 image of each {config} dense block (fwd+bwd, f32)"


def measure_naive_block(shape, dtype):
    """The reference's Naive strategy on the device (paper_1707_06990_b200.naive,
    unfused per-op kernels, every intermediate kept): one fwd+bwd of `shape`,
    its allocator peak and held bytes against the efficient arena of the same
    block.  Outside the timed region; a memory comparison, not a speed claim."""
    import torch
    import paper_1707_06990_b200 as P
    from paper_1707_06990_b200.naive import NaiveBlock
    g = torch.Generator(device="cpu").manual_seed(5)
    p = (torch.randn(shape.param_elems, generator=g) * 0.1 + 0.5).cuda()
    x = torch.randn((shape.n, shape.c0, shape.h, shape.w), generator=g).cuda()
    acc = torch.randn((shape.n, shape.c_out, shape.h, shape.w), generator=g).cuda()
    grads = torch.empty_like(p)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    nb = NaiveBlock(shape, "naive")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    nb.forward(x, p)
    nb.backward(p, acc, grads)
    e1.record()
    torch.cuda.synchronize()
    out = {"block": [shape.n, shape.h, shape.w, shape.c0, shape.m, shape.k, shape.bk],
           "accounted_bytes": nb.retained_bytes() + 4 * x.numel(),
           "held_bytes": torch.cuda.memory_allocated() - base + 4 * x.numel(),
           "allocator_peak_bytes": torch.cuda.max_memory_allocated() - base + 4 * x.numel(),
           "efficient_arena_bytes": P.block_memory(shape, dtype)[0],
           "ms": e0.elapsed_time(e1),
           "note": "Naive strategy on the device, unfused per-op kernels, fp32; bytes include the block input"}
    out["efficient_over_held"] = out["efficient_arena_bytes"] / out["held_bytes"]
    del nb
    torch.cuda.empty_cache()
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import cpu_bench as CB
    runner, what = cpu_runner(args.config)
    shapes = block_shapes(args.config, 1)
    for i in range(args.warmup):
        runner.step(seed=i)
    imgs = secs = 0.0
    t_budget = time.perf_counter()
    steps = 0
    for i in range(args.steps):
        n, s = runner.step(seed=100 + i)
        imgs += n
        secs += s
        steps += 1
        if time.perf_counter() - t_budget > args.ref_budget_s:
            break
    runner.close()
    value = imgs / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": args.warmup, "ms_per_step": 1000 * secs / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {what}, reference CPU", "global_batch": runner.procs,
                   "per_process_batch": 1,
                   "shapes": shapes},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": runner.procs, "kind": CB.kind(),
                         "sample": f"{steps} steps x {runner.procs} processes x {what}, {CB.cpu_model()}"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="bc100")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch kernels directly (no CUDA graph)")
    ap.add_argument("--cpu-budget-s", type=float, default=25.0)
    ap.add_argument("--ref-budget-s", type=float, default=180.0)
    ap.add_argument("--no-naive", action="store_true",
                    help="skip the measured Naive store-everything block (memory comparison)")
    ap.add_argument("--ncu-what", default="blocks", choices=["blocks", "model"],
                    help="with --ncu-step: the dense blocks alone or the whole network step")
    ap.add_argument("--ncu-step", action="store_true",
                    help="after warm-up, run ONE step inside cudaProfilerStart/Stop and exit "
                         "(for `ncu --profile-from-start off`; prints no bench line)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1707_06990_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    hbm_peak, bf16_peak, bf16_sust, peak_src = load_peaks()
    shapes = block_shapes(args.config, BATCH)
    stream = torch.cuda.Stream(device=dev)
    g = torch.Generator(device="cpu").manual_seed(1234 + rank)

    from paper_1707_06990_b200.dp import GradientBuckets
    buckets = GradientBuckets([P.BlockShape(*s).param_elems for s in shapes], device=dev)
    blocks = []
    with torch.cuda.stream(stream):
        for s in shapes:
            shp = P.BlockShape(*s)
            plan = P.BlockPlan(shp, dtype=args.dtype, layout="nhwc", device=local, stream=stream)
            params = torch.randn(shp.param_elems, generator=g) * 0.1
            for l, o in enumerate(shp.param_offsets()):
                c = shp.c_in(l)
                params[o:o + c] += 1.0
                gb = o + 2 * c + shp.bk * c
                params[gb:gb + shp.bk] += 1.0
            blocks.append(dict(
                shape=shp, plan=plan, params=params.to(dev),
                running=shp.initial_running(dev),
                x=torch.randn(shp.pixels, shp.c0, generator=g).to(dev),
                gup=torch.randn(shp.pixels, shp.c_out, generator=g).to(dev),
                acc=torch.empty(shp.pixels, shp.c_out, device=dev),
                grads=buckets.view(len(blocks))))   # block grads are views of one flat buffer

    def step():
        for b in blocks:
            b["plan"].forward(b["x"], b["params"], b["running"], True)
        for b in reversed(blocks):
            b["acc"].copy_(b["gup"])          # consumer BN backward writes the block-output grad
            b["plan"].backward(b["params"], b["acc"], b["grads"])

    def reduce_grads():
        # data-parallel gradient allreduce (per-GPU BN); outside the
        # CUDA graph: one NCCL allreduce of the flat fp32 buffer, scaled by 1/P
        if world > 1:
            buckets.reduce_all()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
            reduce_grads()
    torch.cuda.synchronize(dev)
    launches_per_step = sum(b["plan"].launch_count for b in blocks)  # last backward only
    # count forward+backward launches of one step precisely
    with torch.cuda.stream(stream):
        fwd_launches = 0
        for b in blocks:
            b["plan"].forward(b["x"], b["params"], b["running"], True)
            fwd_launches += b["plan"].launch_count
        bwd_launches = 0
        for b in reversed(blocks):
            b["acc"].copy_(b["gup"])
            b["plan"].backward(b["params"], b["acc"], b["grads"])
            bwd_launches += b["plan"].launch_count
    launches_per_step = fwd_launches + bwd_launches
    torch.cuda.synchronize(dev)

    # ---- capture one step as a CUDA graph (launch overhead off the host) -----
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            step()
        with torch.cuda.stream(stream):
            for _ in range(2):
                graph.replay()
        torch.cuda.synchronize(dev)

    def timed_step():
        if graph is not None:
            graph.replay()
        else:
            step()
        reduce_grads()

    def ncu_step_and_exit(fn, what):
        torch.cuda.synchronize(dev)
        torch.cuda.profiler.start()
        with torch.cuda.stream(stream):
            fn()
        torch.cuda.synchronize(dev)
        torch.cuda.profiler.stop()
        print(json.dumps({"ncu_step": what, "launches_per_step": launches_per_step}), flush=True)
        return 0

    if args.ncu_step and args.ncu_what == "blocks":
        return ncu_step_and_exit(timed_step, "dense blocks")

    def time_steps(fn):
        """K steps of fn between barriers + syncs, CUDA events on `stream`, nvidia-smi
        clocks sampled during the region; returns (ms per step, max over ranks; clocks)."""
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        clocks = ClockSampler(local)
        time.sleep(0.3)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            t0.record(stream)
            for _ in range(args.steps):
                fn()
            t1.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        ms = t0.elapsed_time(t1)
        clk = clocks.stop()
        if world > 1:
            tt = torch.tensor([ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        return ms / args.steps, clk

    # ---- dense blocks alone (the hot path) --------------------------------------
    blocks_ms, blocks_clk = time_steps(timed_step)
    blocks_value = BATCH * world / (blocks_ms / 1000.0)

    # ---- the whole network (headline for CIFAR-type configs: the 3x3 stem) -------
    from paper_1707_06990_b200.model import CONFIGS, ModelPlan
    cfg = CONFIGS[args.config]
    whole = cfg.in_shape[1] < 64
    mplan = None
    if whole:
        mplan = ModelPlan(cfg, BATCH, dtype=args.dtype, device=local, stream=stream)
        m_params = mplan.init_params(seed=1234 + rank, device=dev)
        m_run = mplan.initial_running(dev)
        m_x = torch.randn(BATCH, *cfg.in_shape, generator=g).to(dev)
        m_labels = (torch.arange(BATCH, dtype=torch.int32) % cfg.num_classes).to(dev)
        m_grads = torch.empty(mplan.param_elems, device=dev)
        m_vel = torch.zeros(mplan.param_elems, device=dev)
        m_loss = torch.zeros(1, device=dev)
        from paper_1707_06990_b200.ops import sgd_step

        def model_step():
            mplan.step(m_x, m_labels, m_params, m_run, m_grads, m_loss)

        def model_reduce():
            if world > 1:   # DP allreduce of the flat gradients (per-GPU BN), outside the graph
                dist.all_reduce(m_grads)
                m_grads.mul_(1.0 / world)
            # momentum SGD + weight decay on the averaged gradients (train.hpp:43-70)
            sgd_step(m_params, m_grads, m_vel, lr=0.1, momentum=0.9, weight_decay=1e-4, stream=stream)

        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                model_step()
                model_reduce()
        torch.cuda.synchronize(dev)
        m_graph = None
        if not args.no_graph:
            m_graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(m_graph, stream=stream):
                model_step()
            with torch.cuda.stream(stream):
                for _ in range(2):
                    m_graph.replay()
            torch.cuda.synchronize(dev)

        def model_timed():
            if m_graph is not None:
                m_graph.replay()
            else:
                model_step()
            model_reduce()

        if args.ncu_step:
            return ncu_step_and_exit(model_timed, "whole network")
        ms_per_step, clk = time_steps(model_timed)
        value = BATCH * world / (ms_per_step / 1000.0)
        # block launches + stem / transitions / head kernels of dpb_model_step + SGD
        launches_per_step += 11 + 9 * (len(cfg.block_sizes) - 1) + 1
    else:
        ms_per_step, clk, value = blocks_ms, blocks_clk, blocks_value

    # ---- per-kernel roofline (separate profiled pass, events on `stream`) -----
    for b in blocks:
        b["plan"].profile(True)
    with torch.cuda.stream(stream):
        for _ in range(2):
            for b in blocks:
                b["plan"].forward(b["x"], b["params"], b["running"], True)
            for b in reversed(blocks):
                b["acc"].copy_(b["gup"])
                b["plan"].backward(b["params"], b["acc"], b["grads"])
    torch.cuda.synchronize(dev)
    cats = {}
    for b in blocks:
        for name, st in b["plan"].profile_read().items():
            c = cats.setdefault(name, {"launches": 0, "total_ms": 0.0, "bytes": 0.0, "flops": 0.0})
            for key in c:
                c[key] += st[key]
        b["plan"].profile(False)
    prof_total = sum(c["total_ms"] for c in cats.values())
    # dominant kernel among the categories that move algorithmic HBM bytes
    # (SURVEY 8(d) model); BN-statistic folds (finalize) carry none and are
    # reported beside it
    dom_name, dom = max(((k, v) for k, v in cats.items() if v["bytes"] > 0),
                        key=lambda kv: kv[1]["total_ms"])
    avg_ms = dom["total_ms"] / dom["launches"]
    bytes_per_launch = dom["bytes"] / dom["launches"]
    flops_per_launch = dom["flops"] / dom["launches"]
    ridge = bf16_peak * 1e12 / (hbm_peak * 1e9)
    intensity = flops_per_launch / max(bytes_per_launch, 1.0)
    if intensity < ridge:
        roof = {"bound": "hbm", "achieved": bytes_per_launch / (avg_ms * 1e-3) / 1e9, "peak": hbm_peak,
                "unit": "GB/s"}
    else:
        roof = {"bound": "tensor", "achieved": flops_per_launch / (avg_ms * 1e-3) / 1e12,
                "peak": bf16_sust, "unit": "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = committed_traffic(dom_name, args.config, args.dtype)
    roof["kernel"] = dom_name
    roof["kernel_share_of_step"] = dom["total_ms"] / prof_total
    roof["excluded_zero_byte_kernels"] = {k: round(v["total_ms"] / prof_total, 4)
                                          for k, v in cats.items() if v["bytes"] <= 0}
    roof["peak_source"] = peak_src
    roof["timing"] = ("profiled pass: every launch bracketed by CUDA events on its stream, the backward "
                      "on one stream; in the timed step the weight-gradient kernels (conv*_wgrad, "
                      "reduce_wgrad) run on a side stream overlapping the data-gradient chain, and the "
                      "1x1 wgrad is sized to half the SMs for that overlap")
    F_img, B_img = algorithmic_per_image(shapes)
    t_roof = max(F_img / (bf16_peak * 1e12), B_img / (hbm_peak * 1e9))
    # SURVEY 8(d) byte / FLOP model of the dense blocks: measured against the
    # dense-blocks-only rate (the network's stem / transitions / head are outside it)
    step_roof = {"scope": "dense blocks (SURVEY 8(d) model)",
                 "algorithmic_gflop_per_img": F_img / 1e9, "algorithmic_mb_per_img": B_img / 1e6,
                 "ceiling_img_per_s_per_gpu": 1.0 / t_roof,
                 "frac": (blocks_value / world) * t_roof}
    kernels = {k: {"launches": v["launches"], "ms": round(v["total_ms"] / 2, 4),
                   "GB/s": round(v["bytes"] / max(v["total_ms"], 1e-9) / 1e6, 1),
                   "TFLOP/s": round(v["flops"] / max(v["total_ms"], 1e-9) / 1e9, 2)}
               for k, v in sorted(cats.items(), key=lambda kv: -kv[1]["total_ms"])}

    # ---- end to end through the public API with host buffers --------------------
    if whole:
        # ModelPlan.step per step: H2D of the images and labels from pinned host
        # memory, the training step, the DP allreduce (N > 1), D2H of the flat
        # fp32 gradients and the loss
        x_h = torch.randn(BATCH, *cfg.in_shape, generator=g).pin_memory()
        l_h = (torch.arange(BATCH, dtype=torch.int32) % cfg.num_classes).pin_memory()
        grads_h = torch.empty(mplan.param_elems).pin_memory()
        loss_h = torch.empty(1).pin_memory()
        e_x = torch.empty_like(m_x)
        e_l = torch.empty_like(m_labels)

        def e2e_step():
            e_x.copy_(x_h, non_blocking=True)
            e_l.copy_(l_h, non_blocking=True)
            mplan.step(e_x, e_l, m_params, m_run, m_grads, m_loss)
            model_reduce()
            grads_h.copy_(m_grads, non_blocking=True)
            loss_h.copy_(m_loss, non_blocking=True)

        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                e2e_step()
        torch.cuda.synchronize(dev)
        ek = max(3, min(args.steps, 10))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(ek):
                e2e_step()
            e1.record(stream)
        torch.cuda.synchronize(dev)
        ems = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([ems], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        e2e = {"value": BATCH * world * ek / (ems / 1000.0), "unit": "images/s",
               "h2d_bytes_per_step": x_h.numel() * 4 + l_h.numel() * 4,
               "d2h_bytes_per_step": grads_h.numel() * 4 + 4, "steps": ek,
               "path": "ModelPlan.step (dpb_model_step): pinned host images/labels -> training step -> "
                       "host gradients and loss"}
    else:
        # HostBlockChain: per step, H2D of every block's input and upstream gradient
        # from pinned host memory (copy stream, per-block events), the block
        # forwards/backwards, the DP allreduce (N > 1) and the D2H of the flat fp32
        # gradients, all inside the timed region.
        from paper_1707_06990_b200.host import HostBlockChain
        chain = HostBlockChain([b["shape"] for b in blocks], [b["params"] for b in blocks],
                               [b["running"] for b in blocks], dtype=args.dtype, layout="nchw",
                               device=dev, stream=stream, group=None)
        x_h = [torch.randn(b["shape"].n, b["shape"].c0, b["shape"].h, b["shape"].w, generator=g).pin_memory()
               for b in blocks]
        g_h = [torch.randn(b["shape"].n, b["shape"].c_out, b["shape"].h, b["shape"].w, generator=g).pin_memory()
               for b in blocks]
        for _ in range(args.warmup):
            chain.step(x_h, g_h)
        torch.cuda.synchronize(dev)
        ek = max(3, min(args.steps, 10))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
        for _ in range(ek):
            chain.step(x_h, g_h)
        with torch.cuda.stream(stream):
            e1.record(stream)
        torch.cuda.synchronize(dev)
        ems = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([ems], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        e2e = {"value": BATCH * world * ek / (ems / 1000.0), "unit": "images/s",
               "h2d_bytes_per_step": chain.h2d_bytes(), "d2h_bytes_per_step": chain.d2h_bytes(), "steps": ek,
               "path": "HostBlockChain.step: dpb_block_forward/backward (NCHW), pinned host buffers, "
                       "H2D on a copy stream overlapping compute"}
        chain.close()


    # ---- memory: efficient arena vs naive store-everything ---------------------
    eff = sum(P.block_memory(b["shape"], args.dtype)[0] for b in blocks)
    naive = sum(P.block_memory(b["shape"], "fp32")[1] for b in blocks)
    naive_measured = None
    if rank == 0 and world == 1 and not args.no_naive and P.block_memory(blocks[0]["shape"], "fp32")[1] < 40e9:
        naive_measured = measure_naive_block(blocks[0]["shape"], args.dtype)

    # ---- CPU baseline (rank 0, N=1 only) ---------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import cpu_bench as CB
            runner, what = cpu_runner(args.config)
            runner.step(seed=1)        # warm (spawn + page-in)
            imgs, secs, n = 0, 0.0, 0
            while secs < args.cpu_budget_s and n < 5:
                a, s = runner.step(seed=10 + n)
                imgs += a
                secs += s
                n += 1
            runner.close()
            cpu = {"value": imgs / secs, "unit": "images/s", "cores": runner.procs, "kind": CB.kind(),
                   "sample": f"{n} steps x {runner.procs} processes x {what}, {CB.cpu_model()}"}
        except Exception as exc:  # the baseline is reported, never the target
            cpu = {"value": None, "unit": "images/s", "cores": 0, "kind": "port", "sample": f"failed: {exc}"}

    if rank == 0:
        S = 2 if args.dtype == "bf16" else 4
        ws_bytes = sum(P.plan_arena(b["shape"], args.dtype, "nhwc")["total_bytes"] for b in blocks)
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": (f"DenseNet-{args.config} full training step: stem, dense blocks, transitions, "
                                    f"head, softmax-xent, fwd+bwd, momentum-SGD update" if whole else
                                    f"DenseNet-{args.config} dense blocks, fwd+bwd (the {cfg.in_shape[1]}px "
                                    f"7x7/2 stem is not built)"),
                       "model": args.config, "global_batch": BATCH * world,
                       "per_gpu_batch": BATCH, "blocks": [list(s) for s in shapes],
                       "parallelism": f"dp{world}",
                       "cuda_graph": graph is not None,
                       "l2": f"working set {ws_bytes / 1e6:.0f} MB > 126 MB L2 (no explicit flush)"},
            "dense_blocks": {"value": blocks_value, "unit": "images/s", "ms_per_step": blocks_ms,
                             "note": "the dense blocks alone (the hot path), graph-captured"},
            "roofline": roof, "step_roofline": step_roof, "kernels": kernels,
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "memory": {"efficient_arena_bytes": eff, "naive_bytes": naive,
                       "ratio": eff / naive, "naive_measured": naive_measured},
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    for b in blocks:
        b["plan"].close()
    if mplan is not None:
        mplan.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
