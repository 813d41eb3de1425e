"""Debug: per-phase CTA timing of the halo 3x3 dgrad (dpb_debug_phase_clocks).
Needs a build with the stamps compiled in: rm -rf paper_1707_06990_b200/_build &&
DPB_PHASE_CLOCKS=1 python -m paper_1707_06990_b200.build (the default build has none).
Run with DPB_NO_FORK=1: the backward is then serial and its last halo launch
is layer 0's 3x3 dgrad (BC-100 block-1 geometry).  `python tools/phase_clocks_bwd.py wgrad`
stamps the 3x3 wgrad instead."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1707_06990_b200 as P  # noqa: E402
from paper_1707_06990_b200._lib import lib  # noqa: E402

assert os.environ.get("DPB_NO_FORK"), "run with DPB_NO_FORK=1"
L = lib()
f = L.dpb_debug_phase_clocks
f.argtypes = [C.c_int, C.c_void_p, C.c_int]
shp = P.BlockShape(*[int(v) for v in os.environ.get("SHAPE", "64,32,32,24,4,12,48").split(",")])
plan = P.BlockPlan(shp, dtype="bf16", layout="nhwc")
p = torch.randn(shp.param_elems, device="cuda") * 0.1 + 0.5
x = torch.randn(shp.pixels, shp.c0, device="cuda")
acc = torch.randn(shp.pixels, shp.c_out, device="cuda")
g = torch.empty(shp.param_elems, device="cuda")
run = shp.initial_running()
for _ in range(2):
    plan.forward(x, p, run, True)
    plan.backward(p, acc.clone(), g)
torch.cuda.synchronize()
plan.forward(x, p, run, True)
torch.cuda.synchronize()
WHICH = 2 if len(sys.argv) > 1 and sys.argv[1] == "wgrad" else 1
f(WHICH, None, 0)
plan.backward(p, acc.clone(), g)
torch.cuda.synchronize()
f(0, None, 0)
buf = np.zeros((4096, 9), dtype=np.int64)
f(-1, C.c_void_p(buf.ctypes.data), 4096)
b = buf[(buf[:, 0] != 0) & (buf[:, 8] != 0)]
if len(b) == 0:
    print("no stamps (build with DPB_PHASE_CLOCKS=1)")
    sys.exit(0)
ph = np.diff(b, axis=1)
for i, name in enumerate(["prologue+alloc", "produce", "issue", "mma wait", "epilogue loop", "epi barrier", "col sums", "dealloc"]):
    print(f"{name:18s} mean {ph[:, i].mean():8.0f}  p50 {np.median(ph[:, i]):8.0f}  max {ph[:, i].max():8.0f}")
print("CTA lifetime mean", (b[:, 8] - b[:, 0]).mean())
kbb = np.zeros((4096, 8, 4), dtype=np.int64)
f(-1, C.c_void_p(kbb.ctypes.data), -4096)
kbb = kbb[(buf[:, 0] != 0) & (buf[:, 8] != 0)]
base = b[:, 1][:, None]
for kb in range(8):
    k = kbb[:, kb, :]
    if not k[:, 0].any():
        break
    rel = (k - base).mean(axis=0)
    print(f"kb {kb}: stage free {rel[0]:7.0f}  produced {rel[1]:7.0f}  barrier {rel[2]:7.0f}  issued {rel[3]:7.0f}")
