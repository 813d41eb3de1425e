"""Benchmark of the memory-efficient DenseNet training step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config d264k32|d264k48|d121|bc100|cfg1|...]

One step = one whole training step of the configuration, by default
BASELINE.json configs[3]: DenseNet-264 (k=32, 33M parameters) at 3x224x224,
batch 64 per GPU, ImageNet stem (7x7/2 conv, BN, ReLU, 3x3/2 max-pool), four
dense blocks at 56/28/14/7, transitions, head, softmax cross-entropy, forward
+ backward, the DP gradient allreduce (N > 1) and the momentum-SGD update —
through the public C ABI (ModelPlan -> dpb_model_step, replayed as a CUDA
graph; bf16 tensor-core GEMMs, fp32 arena and gradients) on synthetic inputs
resident in HBM.  The dense blocks alone (the hot path) are timed and
profiled beside it ("dense_blocks", "roofline", "kernels").  Prints ONE JSON
line on rank 0; DESIGN.md §5 documents every field.
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
DEFAULT_CONFIG = "d264k32"   # BASELINE.json configs[3]: DenseNet-264 (k=32, 33M params), 224x224


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
    return [(s.n, s.h, s.w, s.c0, s.m, s.k, s.bk) for s in cfg.block_shapes(batch)]


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


def reference_config(config: str):
    """The configuration the reference itself runs for `config`: the
    ImageNet-stem networks at the reference's own geometry (its 3x3/1 stem on
    3x56x56 gives the same dense blocks, transitions and head as the 7x7/2 +
    max-pool stem on 224x224)."""
    from paper_1707_06990_b200.model import CONFIGS
    name = config + "@56" if CONFIGS[config].stem == "imagenet" else config
    return name, CONFIGS[name]


def cpu_runner(config: str):
    """The reference CPU workload matching the GPU arm: its whole training
    step (GraphPlan::step_trace, the reference's public API), one image per
    process, one process per host core (the reference is single-threaded)."""
    from oracle import cpu_bench as CB
    name, cfg = reference_config(config)
    net = (tuple(cfg.block_sizes), cfg.growth_rate, cfg.compression, cfg.num_classes, cfg.c0, tuple(cfg.in_shape))
    geo = "x".join(str(v) for v in cfg.in_shape)
    return CB.CpuModelRunner(net, batch=1), f"1 image, {name} ({geo}) full training step (GraphPlan::step_trace)"


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
    # the reference is CPU code with no warm-up effects beyond page-in; one
    # untimed step keeps the whole arm within minutes at DenseNet-264 scale
    for i in range(min(args.warmup, 1)):
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
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch kernels directly (no CUDA graph)")
    ap.add_argument("--ref-budget-s", type=float, default=240.0)
    ap.add_argument("--no-blocks", action="store_true", help="skip the dense-blocks-only timing and profile")
    ap.add_argument("--no-naive", action="store_true", help="skip the naive store-everything memory replay")
    ap.add_argument("--ncu-what", default="model", choices=["blocks", "model"],
                    help="with --ncu-step: the dense blocks alone or the whole network step")
    ap.add_argument("--ncu-step", action="store_true",
                    help="after warm-up, run ONE step inside cudaProfilerStart/Stop and exit "
                         "(for `ncu --profile-from-start off`; prints no bench line)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_1707_06990_b200 as P
    from paper_1707_06990_b200.model import CONFIGS, ModelPlan
    from paper_1707_06990_b200.ops import sgd_step

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    hbm_peak, bf16_peak, bf16_sust, peak_src = load_peaks()
    cfg = CONFIGS[args.config]
    shapes = block_shapes(args.config, BATCH)
    stream = torch.cuda.Stream(device=dev)
    g = torch.Generator(device="cpu").manual_seed(1234 + rank)

    def time_steps(fn, k):
        """k steps of fn between barriers + syncs, CUDA events on `stream`,
        nvidia-smi clocks sampled during the region; (ms per step, max over ranks; clocks)."""
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        clocks = ClockSampler(local)
        time.sleep(0.3)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            t0.record(stream)
            for _ in range(k):
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
        return ms / k, clk

    # ---- the whole training step through the public API (ModelPlan) ------------
    free0 = torch.cuda.mem_get_info(dev)[0]
    mplan = ModelPlan(cfg, BATCH, dtype=args.dtype, device=local, stream=stream)
    torch.cuda.synchronize(dev)
    model_alloc_bytes = free0 - torch.cuda.mem_get_info(dev)[0]
    m_params = mplan.init_params(seed=7, device=dev)          # GraphPlan::build's init (rng replay)
    m_run = mplan.initial_running(dev)
    m_x = torch.randn(BATCH, *cfg.in_shape, generator=g).to(dev)
    m_labels = (torch.arange(BATCH, dtype=torch.int32) % cfg.num_classes).to(dev)
    m_grads = torch.empty(mplan.param_elems, device=dev)
    m_vel = torch.zeros(mplan.param_elems, device=dev)
    m_loss = torch.zeros(1, device=dev)

    comm = None
    if world > 1:
        # libdpb's NCCL communicator: dpb_model_step averages the gradients per
        # block bucket on its communication stream, overlapped with the backward
        # of the blocks below (per-GPU BN), inside the step's graph
        from paper_1707_06990_b200.dp import DpComm
        comm = DpComm(rank, world, local)
        mplan.set_comm(comm)

    def model_update():
        # momentum SGD + weight decay (train.hpp:43-70) on the averaged gradients
        sgd_step(m_params, m_grads, m_vel, lr=0.1, momentum=0.9, weight_decay=1e-4, stream=stream)

    def model_step():
        mplan.step(m_x, m_labels, m_params, m_run, m_grads, m_loss)   # graph-replayed by libdpb
        model_update()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            model_step()
    torch.cuda.synchronize(dev)
    mplan.sync()
    if args.ncu_step and args.ncu_what == "model":
        torch.cuda.synchronize(dev)
        torch.cuda.profiler.start()
        with torch.cuda.stream(stream):
            model_step()
        torch.cuda.synchronize(dev)
        torch.cuda.profiler.stop()
        print(json.dumps({"ncu_step": "whole network"}), flush=True)
        return 0
    ms_per_step, clk = time_steps(model_step, args.steps)
    value = BATCH * world / (ms_per_step / 1000.0)
    mplan.sync()
    launches_per_step = mplan.launch_count() + 1  # + SGD

    # ---- end to end with host buffers: pinned images + labels in, loss out -------
    x_h = torch.randn(BATCH, *cfg.in_shape, generator=g).pin_memory()
    l_h = (torch.arange(BATCH, dtype=torch.int32) % cfg.num_classes).pin_memory()
    loss_h = torch.empty(1).pin_memory()
    e_x = torch.empty_like(m_x)
    e_l = torch.empty_like(m_labels)

    copy_stream = torch.cuda.Stream(dev)
    copied = torch.cuda.Event()
    first = [False]  # the timed region's first copy starts after its start event

    def e2e_step():
        if first[0]:
            copy_stream.wait_stream(torch.cuda.current_stream(dev))
            first[0] = False
        # the batch's host-to-device copy runs on its own stream as soon as the
        # previous step has read its inputs (dpb_model_wait_input), overlapping
        # that step's backward like a prefetching input pipeline; the step waits
        # for its copy
        mplan.wait_input(copy_stream)
        with torch.cuda.stream(copy_stream):
            e_x.copy_(x_h, non_blocking=True)
            e_l.copy_(l_h, non_blocking=True)
            copied.record(copy_stream)
        torch.cuda.current_stream(dev).wait_event(copied)
        mplan.step(e_x, e_l, m_params, m_run, m_grads, m_loss)
        model_update()
        loss_h.copy_(m_loss, non_blocking=True)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            e2e_step()
    torch.cuda.synchronize(dev)
    first[0] = True
    e_ms, _ = time_steps(e2e_step, args.steps)
    e2e = {"value": BATCH * world / (e_ms / 1000.0), "unit": "images/s",
           "h2d_bytes_per_step": x_h.numel() * 4 + l_h.numel() * 4, "d2h_bytes_per_step": 4,
           "steps": args.steps,
           "path": "ModelPlan.step (dpb_model_step, C ABI): pinned host images + labels -> H2D (copy stream, "
                   "after the previous step read its inputs: dpb_model_wait_input) -> training step -> DP "
                   "allreduce (N > 1) -> SGD -> D2H loss"}
    mplan.sync()
    loss_value = float(loss_h.item())

    # ---- the dense blocks alone (the hot path) + per-kernel roofline -------------
    blocks_value = blocks_ms = None
    roof = kernels = step_roof = None
    if not args.no_blocks:
        blocks = []
        with torch.cuda.stream(stream):
            for s_ in shapes:
                shp = P.BlockShape(*s_)
                plan = P.BlockPlan(shp, dtype=args.dtype, layout="nhwc", device=local, stream=stream)
                params = torch.randn(shp.param_elems, generator=g) * 0.1
                for l, o in enumerate(shp.param_offsets()):
                    c = shp.c_in(l)
                    params[o:o + c] += 1.0
                    gb = o + 2 * c + shp.bk * c
                    params[gb:gb + shp.bk] += 1.0
                blocks.append(dict(shape=shp, plan=plan, params=params.to(dev), running=shp.initial_running(dev),
                                   x=torch.randn(shp.pixels, shp.c0, generator=g).to(dev),
                                   gup=torch.randn(shp.pixels, shp.c_out, generator=g).to(dev),
                                   acc=torch.empty(shp.pixels, shp.c_out, device=dev),
                                   grads=torch.empty(shp.param_elems, device=dev)))

        def blocks_step():
            for b in blocks:
                b["plan"].forward(b["x"], b["params"], b["running"], True)
            for b in reversed(blocks):
                b["acc"].copy_(b["gup"])      # the consumer BN backward writes the block-output grad
                b["plan"].backward(b["params"], b["acc"], b["grads"])

        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                blocks_step()
        torch.cuda.synchronize(dev)
        graph = None
        if not args.no_graph:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                blocks_step()
        if args.ncu_step:
            torch.cuda.synchronize(dev)
            torch.cuda.profiler.start()
            with torch.cuda.stream(stream):
                graph.replay() if graph is not None else blocks_step()
            torch.cuda.synchronize(dev)
            torch.cuda.profiler.stop()
            print(json.dumps({"ncu_step": "dense blocks"}), flush=True)
            return 0
        blocks_ms, _ = time_steps(lambda: graph.replay() if graph is not None else blocks_step(), args.steps)
        blocks_value = BATCH * world / (blocks_ms / 1000.0)

        # profiled pass: every launch bracketed by CUDA events on its stream
        for b in blocks:
            b["plan"].profile(True)
        with torch.cuda.stream(stream):
            for _ in range(2):
                blocks_step()
        torch.cuda.synchronize(dev)
        cats = {}
        for b in blocks:
            for name, st in b["plan"].profile_read().items():
                c = cats.setdefault(name, {"launches": 0, "total_ms": 0.0, "bytes": 0.0, "flops": 0.0,
                                           "bytes_8d": 0.0})
                for key in c:
                    c[key] += st[key]
            b["plan"].profile(False)
            b["plan"].close()
        prof_total = sum(c["total_ms"] for c in cats.values())
        # dominant kernel: the largest share of the profiled pass, every category counted
        dom_name, dom = max(cats.items(), key=lambda kv: kv[1]["total_ms"])
        avg_s = dom["total_ms"] / dom["launches"] * 1e-3
        b8 = dom["bytes_8d"] / dom["launches"]
        b32 = dom["bytes"] / dom["launches"]
        fl = dom["flops"] / dom["launches"]
        ridge = bf16_peak * 1e12 / (hbm_peak * 1e9)
        if fl / max(b8, 1.0) < ridge:
            roof = {"bound": "hbm", "achieved": b8 / avg_s / 1e9, "peak": hbm_peak, "unit": "GB/s"}
            roof["frac"] = roof["achieved"] / roof["peak"]
            roof["achieved_fp32_storage"] = b32 / avg_s / 1e9
            roof["frac_fp32_storage"] = roof["achieved_fp32_storage"] / hbm_peak
        else:
            roof = {"bound": "tensor", "achieved": fl / avg_s / 1e12, "peak": bf16_sust, "unit": "TFLOP/s"}
            roof["frac"] = roof["achieved"] / roof["peak"]
        roof.update({
            "kernel": dom_name, "launches_per_pass": dom["launches"] // 2, "avg_launch_us": avg_s * 1e6,
            "algorithmic_bytes_per_launch_8d": b8, "algorithmic_bytes_per_launch_fp32_storage": b32,
            "traffic": committed_traffic(dom_name, args.config, args.dtype),
            "kernel_share_of_pass": dom["total_ms"] / prof_total, "peak_source": peak_src,
            "bytes_model": "achieved/frac: SURVEY 8(d) algorithmic bytes (2-byte activations, fp32 gradients); "
                           "*_fp32_storage: the same traffic with this build's fp32 feature storage "
                           "(DESIGN.md 2: bf16 storage breaks the 2e-2 gradient bound)",
            "timing": "profiled pass of the dense blocks: CUDA events around every launch on its stream, "
                      "backward on one stream"})
        F_img, B_img = algorithmic_per_image(shapes)
        t_roof = max(F_img / (bf16_peak * 1e12), B_img / (hbm_peak * 1e9))
        step_roof = {"scope": "dense blocks (SURVEY 8(d) model)",
                     "algorithmic_gflop_per_img": F_img / 1e9, "algorithmic_mb_per_img": B_img / 1e6,
                     "ceiling_img_per_s_per_gpu": 1.0 / t_roof,
                     "frac_dense_blocks": (blocks_value / world) * t_roof,
                     "frac_whole_step": (value / world) * t_roof}
        kernels = {k: {"launches": v["launches"] // 2, "ms": round(v["total_ms"] / 2, 4),
                       "share": round(v["total_ms"] / prof_total, 4),
                       "GB/s_8d": round(v["bytes_8d"] / max(v["total_ms"], 1e-9) / 1e6, 1),
                       "GB/s_fp32_storage": round(v["bytes"] / max(v["total_ms"], 1e-9) / 1e6, 1),
                       "TFLOP/s": round(v["flops"] / max(v["total_ms"], 1e-9) / 1e9, 2)}
                   for k, v in sorted(cats.items(), key=lambda kv: -kv[1]["total_ms"])}
        del blocks
        torch.cuda.empty_cache()

    # ---- memory: the efficient step's device footprint vs naive store-everything --
    mem = mplan.memory()
    peaks = {st: P.predict_peak_elements(cfg, st, BATCH, cfg.in_shape[0], shapes[0][1], shapes[0][2])
             for st in ("naive", "shared-all")}
    feat_elems = {st: sum(v for k, v in d.items() if k != "params") for st, d in peaks.items()}
    memory = {
        "efficient_activation_bytes": mem["activation_bytes"],
        "efficient_total_allocated_bytes": mem["total_bytes"],
        "efficient_allocated_measured_bytes": model_alloc_bytes,
        "efficient_by_arena": mem["by_arena"],
        "reference_peak_model_bytes_fp32": {st: 4 * v for st, v in feat_elems.items()},
        "note": ("efficient: libdpb's device allocations for the whole step (tracked per arena; "
                 "'measured' = cudaMemGetInfo delta around ModelPlan creation); reference_peak_model: "
                 "predict_peak_elements (peak_model.hpp:37-158) feature arenas at this batch, fp32 — the "
                 "reference's own geometry for the stem")}
    if rank == 0 and world == 1 and not args.no_naive:
        from paper_1707_06990_b200.naive import naive_network_replay
        memory["naive_measured"] = naive_network_replay(cfg, BATCH, dev)
        memory["ratio_efficient_over_naive"] = (mem["activation_bytes"] /
                                                memory["naive_measured"]["allocator_peak_bytes"])

    # ---- CPU baseline (rank 0, N=1 only): the reference on the host cores --------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import cpu_bench as CB
            runner, what = cpu_runner(args.config)
            a, secs = runner.step(seed=10)
            runner.close()
            cpu = {"value": a / secs, "unit": "images/s", "cores": runner.procs, "kind": CB.kind(),
                   "sample": f"1 step x {runner.procs} processes x {what}, {CB.cpu_model()}"}
        except Exception as exc:  # the baseline is reported, never the target
            cpu = {"value": None, "unit": "images/s", "cores": 0, "kind": "port", "sample": f"failed: {exc}"}

    if rank == 0:
        ref_name, _ = reference_config(args.config)
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (random-init weights, GraphPlan::build "
                                                               "Rng replay; Gaussian images)",
            "config": {"workload": (f"DenseNet-{args.config} whole training step at {'x'.join(map(str, cfg.in_shape))}"
                                    f" ({cfg.stem} stem, dense blocks, transitions, head, softmax-xent, fwd+bwd, "
                                    f"momentum-SGD update), batch {BATCH} per GPU"),
                       "model": args.config, "global_batch": BATCH * world, "per_gpu_batch": BATCH,
                       "blocks": [list(s_) for s_ in shapes], "parallelism": f"dp{world}",
                       "reference_geometry": ref_name, "loss": loss_value,
                       "cuda_graph": not args.no_graph,
                       "dp": ("libdpb NCCL allreduce (ncclAvg) per block bucket on a communication stream, "
                              "overlapped with backward, inside the step's CUDA graph" if world > 1 else None),
                       "l2": "inputs and working set (GBs of arena) far larger than the 126 MB L2; no flush"},
            "dense_blocks": {"value": blocks_value, "unit": "images/s", "ms_per_step": blocks_ms,
                             "note": "the dense blocks alone (the hot path), graph-captured"},
            "roofline": roof, "step_roofline": step_roof, "kernels": kernels,
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "memory": memory, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    mplan.close()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
