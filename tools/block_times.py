"""Per-block timing of the BC-100 dense blocks (graph-captured fwd+bwd of each
block alone, bf16 NHWC), against the block's HBM floor (SURVEY 8(d) bytes)
and a launch-count floor.  Usage: python tools/block_times.py [config]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1707_06990_b200 as P  # noqa: E402
from bench import algorithmic_per_image, block_shapes, load_peaks  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "bc100"
hbm, _, _, _ = load_peaks()
rows = []
for s in block_shapes(cfg, 64):
    shp = P.BlockShape(*s)
    plan = P.BlockPlan(shp, dtype="bf16", layout="nhwc")
    p = torch.randn(shp.param_elems, device="cuda") * 0.1 + 0.5
    x = torch.randn(shp.pixels, shp.c0, device="cuda")
    acc0 = torch.randn(shp.pixels, shp.c_out, device="cuda")
    acc = acc0.clone()
    g = torch.empty(shp.param_elems, device="cuda")
    run = shp.initial_running()
    st = torch.cuda.Stream()
    plan.set_stream(st)
    with torch.cuda.stream(st):
        for _ in range(3):
            plan.forward(x, p, run, True)
            plan.backward(p, acc, g)
    torch.cuda.synchronize()
    res = {}
    for what in ("fwd", "bwd", "both"):
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=st):
            if what in ("fwd", "both"):
                plan.forward(x, p, run, True)
            if what in ("bwd", "both"):
                plan.backward(p, acc, g)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        with torch.cuda.stream(st):
            for _ in range(3):
                graph.replay()
            e0.record(st)
            for _ in range(n):
                graph.replay()
            e1.record(st)
        torch.cuda.synchronize()
        res[what] = e0.elapsed_time(e1) / n
    # per-category kernel time (events around every launch, serialised; relative only)
    plan.set_stream(None)
    plan.profile(True)
    plan.forward(x, p, run, True)
    plan.backward(p, acc, g)
    torch.cuda.synchronize()
    prof = plan.profile_read()
    plan.profile(False)
    cats = {k: round(v["total_ms"] * 1e3 / max(1, v["launches"]), 1) for k, v in prof.items() if v["launches"]}
    _, B = algorithmic_per_image([s])
    floor_ms = B * shp.n / (hbm * 1e9) * 1e3
    rows.append({"block": s, "fwd_ms": round(res["fwd"], 4), "bwd_ms": round(res["bwd"], 4),
                 "step_ms": round(res["both"], 4), "hbm_floor_ms": round(floor_ms, 4),
                 "frac": round(floor_ms / res["both"], 3), "launches": plan.launch_count, "us_per_launch": cats})
    plan.close()
for r in rows:
    print(json.dumps(r))
